# lts (line-tile sweep): parity tests, then A/B timings
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
rm -f gpurun_out/lts_*.log
PCLAB_LTS_VERBOSE=1 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s > gpurun_out/lts_parity.log 2>&1
echo "parity exit $?" >> gpurun_out/lts_parity.log
for cfg in "PCLAB_LTS=0 PCLAB_BST=0" "PCLAB_LTS=1 PCLAB_LTS_PRE=0" "PCLAB_LTS=1 PCLAB_LTS_VERBOSE=1" "PCLAB_LTS=1 PCLAB_LTS_STAGES=2" "PCLAB_LTS=1 PCLAB_LTS_STAGES=4" "PCLAB_LTS=1 PCLAB_LTS_WINDOW=32" "PCLAB_LTS=1 PCLAB_LTS_WINDOW=8"; do
  env $cfg timeout 60 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/lts_ab.log 2>&1
  echo "exit $?" >> gpurun_out/lts_ab.log
done
