import sys, os, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.workloads import icosphere_patches, patch_samples
sub, k, order = int(sys.argv[1]), 4.0, 12
g = np.load(os.path.join(ROOT, "tests", "golden", "solver.npz"))
tables = {key: g["bie_rule_" + key] for key in ("sample_ref", "far_weight", "near_pts", "near_basis", "self_npts", "self_pts", "self_basis")}
patches = icosphere_patches(sub); xyz = patch_samples(patches, tables["sample_ref"])
op = HfmmCuda(k=k, order=order, ncrit=64, theta=0.4, kd_max=1.0, leaf_cap=-1.0)
op.set_points(xyz); op.build_corrections(patches, tables, fetch=False)
rhs = np.exp(1j * k * xyz[:, 2])
for restart, prec in ((30, True), (30, False), (100, True), (300, True)):
    x, rep = op.gmres(rhs, rtol=1e-4, restart=restart, max_iterations=600, precondition=prec)
    r = rep["residuals"]
    print(restart, prec, rep["iterations"], rep["converged"], "%.3e" % rep["final_residual"], ["%.2e" % v for v in r[[9, 29, 59, 99, 199, 299, 399, 599][:sum(i < len(r) for i in [9, 29, 59, 99, 199, 299, 399, 599])]]], flush=True)
