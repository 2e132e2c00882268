# Round profile: bench line, configs[4] bandwidth sweep, ncu launch list of
# the bench command and ncu --set full of the dominant kernels (each ncu run
# only after the same command exited 0 without ncu).
set -x
python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
python bench.py --bw-sweep > gpurun_out/bw_sweep.log 2> gpurun_out/bw_sweep.err
python tools/run_kernels.py elasticity_q1_118 0 1 gnnic > gpurun_out/rk.log 2>&1 && \
  ncu --set full --clock-control none --import-source on \
      -k regex:"bsr_trsv_kernel|k_spmv_bsr_pap|edge_kernel|node_kernel|ic0_kernel|features_kernel" -c 14 \
      -o gpurun_out/full python tools/run_kernels.py elasticity_q1_118 0 1 gnnic > gpurun_out/ncu_full.log 2>&1
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/b1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
