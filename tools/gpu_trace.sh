export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/tr
for w in ${TRACE_WORKLOADS:-elasticity_q1_118}; do
  PCLAB_LIB=$PWD/build/var_trace/libpclab_b200.so timeout 300 python tools/bss_trace.py $w > gpurun_out/tr/${w}_lower.log 2>&1
  PCLAB_LIB=$PWD/build/var_trace/libpclab_b200.so timeout 300 python tools/bss_trace.py $w upper > gpurun_out/tr/${w}_upper.log 2>&1
  cat gpurun_out/tr/${w}_lower.log gpurun_out/tr/${w}_upper.log
done
