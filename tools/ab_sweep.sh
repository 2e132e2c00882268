# A/B of compile-time sweep variants (build/var_*/libpclab_b200.so via PCLAB_LIB)
export PYTHONUNBUFFERED=1
for lib in paper_2412_07127_b200/libpclab_b200.so build/var_*/libpclab_b200.so; do
  echo "== $lib" >> gpurun_out/ab.log
  PCLAB_LIB=$PWD/$lib timeout 300 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/ab.log 2>&1
done
