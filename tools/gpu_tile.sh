timeout 300 python tools/trsv_time.py diffusion_fv_256 >> gpurun_out/rr2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/trr.log 2>&1; echo RC $? >> gpurun_out/trr.log
