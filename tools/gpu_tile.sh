timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bk5.log 2>&1
