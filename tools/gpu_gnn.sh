export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/gnn; rm -f gpurun_out/gnn/*
build/tanh_check > gpurun_out/gnn/tanh.log 2>&1; echo "exit $?" >> gpurun_out/gnn/tanh.log; cat gpurun_out/gnn/tanh.log
for lib in paper_2412_07127_b200/libpclab_b200.so build/var_libm/libpclab_b200.so; do
  echo "== $lib" >> gpurun_out/gnn/time.log
  PCLAB_LIB=$PWD/$lib timeout 300 python tools/gnn_time.py elasticity_q1_118 2>&1 | grep gnnic | tail -2 >> gpurun_out/gnn/time.log
  PCLAB_LIB=$PWD/$lib timeout 300 python tools/gnn_time.py diffusion_fv_256 2>&1 | grep gnnic | tail -2 >> gpurun_out/gnn/time.log
done
cat gpurun_out/gnn/time.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gnn/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gnn/tests.log
tail -4 gpurun_out/gnn/tests.log
