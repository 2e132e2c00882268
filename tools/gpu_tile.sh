python tools/run_kernels.py elasticity_q1_118 0 1 > gpurun_out/rk2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"ic0|gather_kernel|invd_kernel|row_stats" -c 6 -o gpurun_out/ic0prof python tools/run_kernels.py elasticity_q1_118 0 1 > gpurun_out/ncu_ic0.log 2>&1
