timeout 600 python -m pytest tests/test_gpu_variants.py -x -q -k ic0 > gpurun_out/tm.log 2>&1; echo RC $? >> gpurun_out/tm.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "ic0 or config" > gpurun_out/tm2.log 2>&1; echo RC $? >> gpurun_out/tm2.log
timeout 300 python tools/gnn_time.py elasticity_q1_118 > gpurun_out/gm.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/bm.log 2>&1
