# developer A/B: sweep knobs on configs[2]
T="python tools/trsv_time.py elasticity_q1_118"
PCLAB_FUSE=0 $T
PCLAB_FUSE=0 PCLAB_TRSV_DEPTH=2 $T
PCLAB_FUSE=0 PCLAB_TRSV_TRACE=/tmp/tr118 python tools/run_kernels.py elasticity_q1_118 0 1
python tools/trace_trsv.py /tmp/tr118
