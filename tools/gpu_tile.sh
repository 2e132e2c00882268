for t in 0 6400 12800 25600 51200; do
  PCLAB_TRSV_TUNE=$t timeout 300 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/sleep.log 2>&1
done
