python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/b1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
