for env in "PCLAB_SMP=0" "PCLAB_SMP=1" "PCLAB_SMP=1 PCLAB_TRSV_DEPTH=4" "PCLAB_SMP=1 PCLAB_TRSV_TUNE=2"; do
  env $env timeout 300 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/smp.log 2>&1
done
PCLAB_SMP=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/tsmp.log 2>&1
