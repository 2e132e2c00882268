for i in 1 2; do timeout 300 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/pfl.log 2>&1; done
