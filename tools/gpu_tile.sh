python bench.py > gpurun_out/bench2.log 2> gpurun_out/bench2.err
python bench.py --bw-elasticity > gpurun_out/bw_el2.log 2> gpurun_out/bw_el2.err
