timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/tall4.log 2>&1; echo RC $? >> gpurun_out/tall4.log
timeout 300 python tools/trsv_time.py elasticity_q1_118 > gpurun_out/t7.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b7.log 2>&1
