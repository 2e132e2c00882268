for env in "PCLAB_LANES=16" "PCLAB_LANES=8"; do
  env $env timeout 300 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/lg8.log 2>&1
done
PCLAB_LANES=8 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/tlg8.log 2>&1
