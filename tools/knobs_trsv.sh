T="python tools/trsv_time.py elasticity_q1_118"
$T
python tools/prof_stages.py elasticity_q1_118 0 3 2>&1 | grep -E "spmv|trsv"
