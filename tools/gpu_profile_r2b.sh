# Round-2 ncu of the GNN kernels (configs[2]) and of the configs[4] 256^3
# product / sweeps (kernel-name filters that skip the set-up kernels)
set -x
mkdir -p gpurun_out/r2
python tools/run_kernels.py elasticity_q1_118 0 1 gnnic > gpurun_out/r2/rkg.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on \
      -k regex:"edge_kernel|node_kernel|features_kernel|node_proj_kernel" -c 10 \
      -o /tmp/gnn python tools/run_kernels.py elasticity_q1_118 0 1 gnnic > gpurun_out/r2/ncu_gnn.log 2>&1 && \
  ncu -i /tmp/gnn.ncu-rep --page raw --csv > gpurun_out/r2/gnn_raw.csv
python tools/run_kernels.py diffusion_fv_256 0 1 > gpurun_out/r2/rk2.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:"spmv_tile|rr_trsv" -c 5 \
      -o /tmp/diff python tools/run_kernels.py diffusion_fv_256 0 1 > gpurun_out/r2/ncu_diff.log 2>&1 && \
  ncu -i /tmp/diff.ncu-rep --page raw --csv > gpurun_out/r2/diff_raw.csv
