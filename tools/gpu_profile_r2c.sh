# Final round-2 profile refresh (one gpurun call, after the sweep / GNN changes):
# full GPU suite, smoke, the bench line and the reference arm, bandwidth sweeps,
# the ncu launch list of the bench command, ncu --set full of the configs[2]
# loop kernels, of the GNN kernels and of the configs[4] 256^3 product / sweeps
# (each ncu run after the same command exited 0 without ncu), traces of both sweeps.
export PYTHONUNBUFFERED=1
O=gpurun_out/r2c
mkdir -p $O; rm -f $O/*
python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo "tests exit $?" >> $O/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
python bench.py > $O/bench.log 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
python bench.py --impl reference > $O/bench_ref.log 2> $O/bench_ref.err
python bench.py --bw-elasticity > $O/bw_el.log 2> $O/bw_el.err
python bench.py --bw-sweep > $O/bw_sweep.log 2> $O/bw_sweep.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra > $O/b1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
      --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extra > $O/ncu_launch.log 2>&1
python tools/run_kernels.py elasticity_q1_118 0 1 > $O/rk.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:"bss_trsv_kernel|k_spmv_bsr_pap4|k_axpy4|k_dot_z4" \
      -s 2 -c 6 -o /tmp/loop python tools/run_kernels.py elasticity_q1_118 0 1 > $O/ncu_loop.log 2>&1 && \
  ncu -i /tmp/loop.ncu-rep --page raw --csv > $O/loop_raw.csv
python tools/run_kernels.py elasticity_q1_118 0 1 gnnic > $O/rkg.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on \
      -k regex:"edge_kernel|node_kernel|features_kernel|node_proj_kernel" -c 10 \
      -o /tmp/gnn python tools/run_kernels.py elasticity_q1_118 0 1 gnnic > $O/ncu_gnn.log 2>&1 && \
  ncu -i /tmp/gnn.ncu-rep --page raw --csv > $O/gnn_raw.csv
python tools/run_kernels.py diffusion_fv_256 0 1 > $O/rk2.log 2>&1 && \
  ncu -f --set full --clock-control none --import-source on -k regex:"spmv_tile|rec_trsv" -c 5 \
      -o /tmp/diff python tools/run_kernels.py diffusion_fv_256 0 1 > $O/ncu_diff.log 2>&1 && \
  ncu -i /tmp/diff.ncu-rep --page raw --csv > $O/diff_raw.csv
TRACE_WORKLOADS="elasticity_q1_118 diffusion_fv_256" bash tools/gpu_trace.sh > $O/trace.log 2>&1
build/pingpong2 > $O/pingpong2.log 2>&1
tail -2 $O/gputests.log; cat $O/smoke.log; cat $O/bench.log
