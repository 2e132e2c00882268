# developer probe: staggered polls + ncu full of the dominant kernels
for env in "PCLAB_POLL=0" "PCLAB_POLL=1" "PCLAB_POLL=1 PCLAB_TRSV_TUNE=20480" "PCLAB_POLL=1 PCLAB_TRSV_TUNE=51200"; do
  env $env timeout 300 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/exp10.log 2>&1
done
python tools/run_kernels.py elasticity_q1_118 0 1 gnnic > gpurun_out/rk.log 2>&1 && \
  ncu --set full --clock-control none --import-source on \
      -k regex:"bsr_trsv_kernel|k_spmv_bsr_pap|edge_kernel|node_kernel|ic0_kernel|features_kernel" -c 14 \
      -o gpurun_out/full python tools/run_kernels.py elasticity_q1_118 0 1 gnnic > gpurun_out/ncu_full.log 2>&1
