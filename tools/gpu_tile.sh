for env in "PCLAB_X=1" "PCLAB_LIB=build/var/libpclab_pap5.so"; do
  env $env timeout 300 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/pap5.log 2>&1
done
