python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err
python tools/run_kernels.py elasticity_q1_118 0 1 > gpurun_out/rk.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"bsr_trsv_kernel|k_spmv_bsr_pap4" -s 2 -c 3 \
      -o gpurun_out/loop python tools/run_kernels.py elasticity_q1_118 0 1 > gpurun_out/ncu_loop.log 2>&1
