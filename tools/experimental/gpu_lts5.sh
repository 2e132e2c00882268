export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
rm -f gpurun_out/lts5_*.log
timeout 200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/lts5_parity.log 2>&1
echo "parity exit $?" >> gpurun_out/lts5_parity.log
for cfg in "PCLAB_LTS_STAGES=4" "PCLAB_LTS_STAGES=3" "PCLAB_LTS_STAGES=6" "PCLAB_LTS_HELPERS=1" "PCLAB_LTS_HELPERS=3" "PCLAB_LTS_OPT=4"; do
  env $cfg timeout 60 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/lts5_ab.log 2>&1
  echo "exit $?" >> gpurun_out/lts5_ab.log
done
timeout 120 python tools/lts_trace.py > gpurun_out/lts5_trace.log 2>&1
