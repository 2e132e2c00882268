for d in 4 16; do
  echo "DEPTH=$d"
  PCLAB_TRSV_DEPTH=$d timeout 120 python tools/prof_stages.py elasticity_q1_40 0 30 2>&1 | grep -E "trsv|pcg\[ic0"
  PCLAB_TRSV_DEPTH=$d PCLAB_TRSV_TRACE=gpurun_out/tr$d python tools/run_kernels.py elasticity_q1_40 0 1 > /dev/null 2>&1; python tools/trace_trsv.py gpurun_out/tr$d | grep -E "items|per item|deltas|L1:|L2:|L3:"
done
