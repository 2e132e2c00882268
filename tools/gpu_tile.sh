for env in "PCLAB_VGRID=4" "PCLAB_VGRID=8" "PCLAB_VGRID=2"; do
  env $env timeout 300 python tools/trsv_time.py elasticity_q1_118 >> gpurun_out/vg.log 2>&1
done
