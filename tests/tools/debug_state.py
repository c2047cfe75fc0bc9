import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import synth
from paper_2001_08707_b200.device import to_device, make_solver
p = synth.make_problem("c1", L=8, nz=4)
g = make_solver(to_device(p))
print("init", g.coefficients())
for n in range(3):
    st = g.update()
    print(n, st, g.coefficients())
