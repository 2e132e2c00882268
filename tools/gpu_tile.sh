# developer probe: sweep timing on configs[2]
for env in "PCLAB_X=0" "PCLAB_TRSV_TUNE=2" "PCLAB_TRSV_DEPTH=2.5" "PCLAB_TRSV_DEPTH=5"; do
  env $env timeout 300 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/exp9.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q > gpurun_out/t9.log 2>&1
