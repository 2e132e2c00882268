for env in "PCLAB_TMAW=1" "PCLAB_TMAW=0"; do
  env $env timeout 300 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/tmaw.log 2>&1
done
PCLAB_TMAW=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/ttmaw.log 2>&1
