# Round-2 profile refresh (one gpurun call): bench line (+ CPU reference),
# reference arm, bandwidth sweeps, the ncu launch list of the bench command,
# ncu --set full of the configs[2] loop kernels, of the GNN kernels and of
# the configs[4] 256^3 sweep / product (each ncu run after the same command
# exited 0 without ncu); raw pages exported to CSV on the box.
set -x
mkdir -p gpurun_out/r2
python bench.py > gpurun_out/r2/bench.log 2> gpurun_out/r2/bench.err
python bench.py --impl reference > gpurun_out/r2/bench_ref.log 2> gpurun_out/r2/bench_ref.err
python bench.py --bw-elasticity > gpurun_out/r2/bw_el.log 2> gpurun_out/r2/bw_el.err
python bench.py --bw-sweep > gpurun_out/r2/bw_sweep.log 2> gpurun_out/r2/bw_sweep.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/r2/b1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
      --log-file gpurun_out/r2/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra \
      > gpurun_out/r2/ncu_launch.log 2>&1
python tools/run_kernels.py elasticity_q1_118 0 1 > gpurun_out/r2/rk.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:"bsr_trsv_kernel|k_spmv_bsr_pap4|k_axpy4|k_dot_z4" \
      -s 2 -c 6 -o /tmp/loop python tools/run_kernels.py elasticity_q1_118 0 1 > gpurun_out/r2/ncu_loop.log 2>&1 && \
  ncu -i /tmp/loop.ncu-rep --page raw --csv > gpurun_out/r2/loop_raw.csv
python tools/run_kernels.py elasticity_q1_118 0 1 gnnic > gpurun_out/r2/rkg.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on \
      -k regex:"edge_kernel|node_kernel|features_kernel|node_proj|ic0_block_kernel|level_queue|radix" -c 14 \
      -o /tmp/gnn python tools/run_kernels.py elasticity_q1_118 0 1 gnnic > gpurun_out/r2/ncu_gnn.log 2>&1 && \
  ncu -i /tmp/gnn.ncu-rep --page raw --csv > gpurun_out/r2/gnn_raw.csv
python tools/run_kernels.py diffusion_fv_256 0 1 > gpurun_out/r2/rk2.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:"tile|rr_trsv" -c 5 \
      -o /tmp/diff python tools/run_kernels.py diffusion_fv_256 0 1 > gpurun_out/r2/ncu_diff.log 2>&1 && \
  ncu -i /tmp/diff.ncu-rep --page raw --csv > gpurun_out/r2/diff_raw.csv
ls -la gpurun_out/r2/
