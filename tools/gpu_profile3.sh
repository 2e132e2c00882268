# Round profile refresh: bench line (+ CPU reference), reference arm,
# elasticity bandwidth, ncu launch list of the bench command, ncu --set full
# of the configs[2] loop kernels and of the configs[4] 256^3 row-tile product
# and entry-lane sweeps (each ncu run after the same command exited 0
# without ncu); raw pages exported to CSV on the box.
set -x
python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err
python bench.py --bw-elasticity > gpurun_out/bw_el.log 2> gpurun_out/bw_el.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/b1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/run_kernels.py elasticity_q1_118 0 1 > gpurun_out/rk.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"bsr_trsv_kernel|k_spmv_bsr_pap4" -s 2 -c 3 \
      -o /tmp/loop python tools/run_kernels.py elasticity_q1_118 0 1 > gpurun_out/ncu_loop.log 2>&1 && \
  ncu -i /tmp/loop.ncu-rep --page raw --csv > gpurun_out/loop_raw.csv
python tools/run_kernels.py diffusion_fv_256 0 1 > gpurun_out/rk2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"tile|rr_trsv" -c 5 \
      -o /tmp/diff python tools/run_kernels.py diffusion_fv_256 0 1 > gpurun_out/ncu_diff.log 2>&1 && \
  ncu -i /tmp/diff.ncu-rep --page raw --csv > gpurun_out/diff_raw.csv
ls -la gpurun_out/
