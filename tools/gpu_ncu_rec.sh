mkdir -p gpurun_out/ncurec; rm -f gpurun_out/ncurec/*
python tools/run_kernels.py diffusion_fv_256 0 1 > gpurun_out/ncurec/rk.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:"rec_trsv_kernel" \
      -s 2 -c 2 -o gpurun_out/ncurec/rec python tools/run_kernels.py diffusion_fv_256 0 1 > gpurun_out/ncurec/ncu.log 2>&1
tail -2 gpurun_out/ncurec/ncu.log
