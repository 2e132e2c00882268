# Round profile, part 2: ncu --set full of the dominant kernels (after the
# same command exited 0 without ncu). Kernel order in run_kernels: levelling,
# IC(0) masks + block kernel, GNN edge/node kernels, stand-alone sweeps,
# then the PCG loop (padded sweeps, product).
python tools/run_kernels.py elasticity_q1_118 0 1 gnnic > gpurun_out/rk.log 2>&1 && \
  ncu --set full --clock-control none --import-source on \
      -k regex:"bsr_trsv_kernel|k_spmv_bsr_pap4|edge_kernel|ic0_block_kernel|ic0_masks" -c 12 \
      -o gpurun_out/full python tools/run_kernels.py elasticity_q1_118 0 1 gnnic > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out/
