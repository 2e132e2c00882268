for cfg in "32 4" "32 8" "16 4"; do
  set -- $cfg
  echo "LANES=$1 DEPTH=$2"
  PCLAB_SWEEP=0 PCLAB_LANES=$1 PCLAB_TRSV_DEPTH=$2 timeout 300 python tools/prof_stages.py elasticity_q1_118 0 10 2>&1 | grep -E "trsv"
done
PCLAB_SWEEP=0 timeout 300 python tools/prof_stages.py elasticity_q1_40 0 10 2>&1 | grep -E "trsv"
PCLAB_SWEEP=0 python tools/gpu_probe.py 2>&1 | grep -E " its |ERR|bitexact" | tail -6
