# bst (TMA-staged sweep) first run: parity tests, then A/B timings
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/bst_parity.log 2>&1
echo "parity exit $?" >> gpurun_out/bst_parity.log
for cfg in "PCLAB_BST=0" "PCLAB_BST=1 PCLAB_BST_STAGES=2" "PCLAB_BST=1 PCLAB_BST_STAGES=3" "PCLAB_BST=1 PCLAB_BST_STAGES=4"; do
  env $cfg timeout 300 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/bst_ab.log 2>&1
  echo "exit $?" >> gpurun_out/bst_ab.log
done
