for env in "PCLAB_LIB=build/var/lib_7_0.so" "PCLAB_LIB=build/var/lib_8_0.so PCLAB_TRSV_DEPTH=6" "PCLAB_LIB=build/var/lib_8_1.so PCLAB_TRSV_DEPTH=6"; do
  env $env timeout 300 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/pf0.log 2>&1
done
