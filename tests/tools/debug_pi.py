import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import oracle, synth
from paper_2001_08707_b200.device import to_device, make_solver
p = synth.make_problem(sys.argv[1] if len(sys.argv) > 1 else "c1")
g = make_solver(to_device(p))
o = oracle.Oracle(p.method, p.b, p.z, left=p.left, full_x=p.full_x, tol=p.tol, itermax=p.itermax,
                  flags=oracle.FLAG_NO_SWITCH)
gn = make_solver(to_device(p), flags=1)
for n in range(3):
    gn.update(); o.step(p.op)
    pig, act, ret = gn.shift_state()
    print(n, "pi gpu", pig[:4], "\n   pi orc", o.pi()[:4])
    print("   res", gn.residuals()[:3], o.residuals()[:3])
    print("   coef", {k: v for k, v in gn.coefficients().items() if k in ("alpha", "beta", "rho", "z_seed", "seed_index")}, o.scalars())
