export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
rm -f gpurun_out/lts4_*.log
timeout 200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/lts4_parity.log 2>&1
echo "parity exit $?" >> gpurun_out/lts4_parity.log
for cfg in "PCLAB_LTS_OPT=2" "PCLAB_LTS_OPT=6" "PCLAB_LTS_OPT=7" "PCLAB_LTS_OPT=2 PCLAB_LTS_STAGES=4" "PCLAB_LTS_OPT=2 PCLAB_LTS_STAGES=5" "PCLAB_LTS_OPT=6 PCLAB_LTS_STAGES=5"; do
  env $cfg timeout 60 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/lts4_ab.log 2>&1
  echo "exit $?" >> gpurun_out/lts4_ab.log
done
PCLAB_LTS_OPT=2 PCLAB_LTS_STAGES=5 timeout 120 python tools/lts_trace.py > gpurun_out/lts4_trace.log 2>&1
