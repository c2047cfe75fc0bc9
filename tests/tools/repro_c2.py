import sys; sys.path.insert(0, '/root/repo')
import synth, numpy as np
from paper_2001_08707_b200.device import to_device, make_solver
L = int(sys.argv[1]) if len(sys.argv) > 1 else 20
p = synth.make_problem('c2', L=L)
g = make_solver(to_device(p))
for i in range(3):
    print(i, g.update(), flush=True)
print(g.residuals()[:3])
