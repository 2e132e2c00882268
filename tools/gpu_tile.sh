timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/tall2.log 2>&1; echo RC $? >> gpurun_out/tall2.log
for env in "PCLAB_RAX=1" "PCLAB_RAX=0"; do
  env $env timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/brax2_$env.log 2>&1
done
