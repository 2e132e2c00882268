timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/tall3.log 2>&1; echo RC $? >> gpurun_out/tall3.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b6.log 2>&1
