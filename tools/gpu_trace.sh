export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/tr
PCLAB_LIB=$PWD/build/var_trace/libpclab_b200.so timeout 300 python tools/bss_trace.py elasticity_q1_118 > gpurun_out/tr/lower.log 2>&1
PCLAB_LIB=$PWD/build/var_trace/libpclab_b200.so timeout 300 python tools/bss_trace.py elasticity_q1_118 upper > gpurun_out/tr/upper.log 2>&1
cat gpurun_out/tr/lower.log gpurun_out/tr/upper.log
