timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/tall5.log 2>&1; echo RC $? >> gpurun_out/tall5.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b8.log 2>&1
timeout 600 python bench.py --bw-elasticity > gpurun_out/bwe2.log 2>&1
