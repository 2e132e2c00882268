timeout 300 python tools/gnn_time.py elasticity_q1_118 > gpurun_out/ic0m2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "ic0 or config or fixture or acceptance or pcg" > gpurun_out/tic02.log 2>&1
