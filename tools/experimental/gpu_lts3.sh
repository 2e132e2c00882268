export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
rm -f gpurun_out/lts3_*.log
for cfg in "PCLAB_LTS_OPT=0" "PCLAB_LTS_OPT=1" "PCLAB_LTS_OPT=2" "PCLAB_LTS_OPT=3" "PCLAB_LTS_OPT=3 PCLAB_LTS_STAGES=4" "PCLAB_LTS_OPT=3 PCLAB_LTS_STAGES=6"; do
  env $cfg timeout 60 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/lts3_ab.log 2>&1
  echo "exit $?" >> gpurun_out/lts3_ab.log
done
PCLAB_LTS_OPT=3 timeout 120 python tools/lts_trace.py > gpurun_out/lts3_trace.log 2>&1
