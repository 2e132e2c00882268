timeout 1200 python -m pytest tests/test_gpu_variants.py -q > gpurun_out/tv2.log 2>&1; echo RC $? >> gpurun_out/tv2.log
