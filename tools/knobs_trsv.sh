# developer A/B: sweep knobs on configs[2] + a trace
T="python tools/trsv_time.py elasticity_q1_118"
for d in 2 3 4; do PCLAB_TRSV_DEPTH=$d $T; done
PCLAB_TRSV_TRACE=/tmp/tr118 python tools/run_kernels.py elasticity_q1_118 0 1
python tools/trace_trsv.py /tmp/tr118
