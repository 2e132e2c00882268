T="python tools/trsv_time.py elasticity_q1_118"
timeout 120 $T
PCLAB_CHAIN=1 timeout 120 $T
