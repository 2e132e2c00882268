# Round profile: bench line (+ CPU reference), reference arm, bandwidth
# sweeps, ncu launch list of the bench command, ncu --set full of the loop
# kernels (each ncu run after the same command exited 0 without ncu).
set -x
python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err
python bench.py --bw-sweep > gpurun_out/bw_sweep.log 2> gpurun_out/bw_sweep.err
python bench.py --bw-elasticity > gpurun_out/bw_el.log 2> gpurun_out/bw_el.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/b1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/run_kernels.py elasticity_q1_118 0 1 > gpurun_out/rk.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"bsr_trsv_kernel|k_spmv_bsr_pap4" -s 2 -c 3 \
      -o gpurun_out/loop python tools/run_kernels.py elasticity_q1_118 0 1 > gpurun_out/ncu_loop.log 2>&1
