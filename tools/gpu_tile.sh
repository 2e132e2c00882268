timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bk4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/tk4.log 2>&1
