export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
rm -f gpurun_out/lts2_*.log
for cfg in "PCLAB_LTS=1 PCLAB_LTS_NOWAIT=1" "PCLAB_LTS=1"; do
  env $cfg timeout 60 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/lts2_ab.log 2>&1
  echo "exit $?" >> gpurun_out/lts2_ab.log
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lts_trsv -c 2 -o gpurun_out/lts2_ncu -f python tools/run_kernels.py elasticity_q1_118 0 1 > gpurun_out/lts2_ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/lts2_ncu.log
