timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/tfinal.log 2>&1; echo RC $? >> gpurun_out/tfinal.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo RC $? >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/b1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
