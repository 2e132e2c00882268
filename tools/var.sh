python tools/solve_var.py elasticity_q1_118 4 2>&1 | grep run
echo eager; PCLAB_PCG_GRAPH=0 python tools/solve_var.py elasticity_q1_118 4 2>&1 | grep run
echo pairs1; PCLAB_GRAPH_PAIRS=1 python tools/solve_var.py elasticity_q1_118 4 2>&1 | grep run
