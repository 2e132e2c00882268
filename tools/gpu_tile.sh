timeout 900 python bench.py --bw-elasticity > gpurun_out/bwe.log 2> gpurun_out/bwe.err
