timeout 300 python tools/gnn_time.py elasticity_q1_118 > gpurun_out/gnn_time.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "gnn or config1" > gpurun_out/tgnn.log 2>&1
