timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_fullsize.py -x -q > gpurun_out/tpad.log 2>&1; echo RC $? >> gpurun_out/tpad.log
timeout 300 python tools/trsv_time.py elasticity_q1_118 > gpurun_out/tpadt.log 2>&1
