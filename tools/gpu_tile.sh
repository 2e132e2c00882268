for env in "PCLAB_PADZ=1" "PCLAB_PADZ=0"; do
  env $env timeout 300 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/padz.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_variants.py -x -q > gpurun_out/tk7.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bk7.log 2>&1
