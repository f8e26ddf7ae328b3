"""CPU (this container): the compiled reference's own GMRES on an icosphere mesh, for the
iteration-count comparison of BASELINE.md's config-3 plan.  Slow: ~10-30 s per matvec."""
import sys, os, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from checkers import Ref
from paper_1803_09948_b200.workloads import icosphere_patches
sub, prec, out = int(sys.argv[1]), sys.argv[2] != "0", sys.argv[3]
k, order = 4.0, 12
R = Ref()
t0 = time.time()
sysr = R.bie(icosphere_patches(sub), 1, k, mode=2, use_tree=True, order=order, ncrit=64, theta=0.4, kd_max=1.0, leaf_cap=-1.0)
t_build = time.time() - t0
rhs = sysr.rhs((0, 0, 1))
t0 = time.time()
sol, rep = sysr.gmres(rhs, rtol=1e-4, restart=30, max_iterations=1000, precondition=prec)
json.dump({"triangles": 20 * 4 ** sub, "unknowns": int(sysr.n), "k": k, "order": order, "block_jacobi": prec,
           "iterations": int(rep["iterations"]), "converged": bool(rep["converged"]),
           "final_residual": float(rep["final_residual"]), "build_s": t_build, "solve_s": time.time() - t0,
           "threads": os.cpu_count(), "residuals": [float(v) for v in rep["residuals"]]}, open(out, "w"))
