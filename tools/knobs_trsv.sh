T="python tools/trsv_time.py diffusion_fv_256"
timeout 200 $T
PCLAB_LANES=4 timeout 200 $T
PCLAB_LANES=2 timeout 200 $T
PCLAB_RR=0 PCLAB_LANES=4 timeout 200 $T
timeout 200 python tools/trsv_time.py poisson3d_7pt_32
