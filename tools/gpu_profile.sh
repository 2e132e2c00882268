# Round profile, part 1: bench line (+ CPU reference), reference arm,
# configs[4] bandwidth sweep, ncu launch list of the bench command.
set -x
python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err
python bench.py --bw-sweep > gpurun_out/bw_sweep.log 2> gpurun_out/bw_sweep.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/b1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
