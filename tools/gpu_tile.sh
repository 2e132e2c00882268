for i in 1 2; do timeout 300 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/hp.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q > gpurun_out/thp.log 2>&1; echo RC $? >> gpurun_out/thp.log
