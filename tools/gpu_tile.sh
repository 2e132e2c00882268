for env in "PCLAB_LANES=8" "PCLAB_LANES=32" "PCLAB_LANES=4"; do
  env $env timeout 300 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/lanes.log 2>&1
done
