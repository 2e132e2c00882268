for env in "PCLAB_PADP=1" "PCLAB_PADP=0"; do
  env $env timeout 300 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/padp.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/tk6.log 2>&1
