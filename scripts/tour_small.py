"""GPU: a small tour of every kernel family (matvec at two orders and both batch layouts, complex k,
corrections, GMRES, field evaluation) at sizes that finish in a second (compute-sanitizer is closed on
the GPU pool; this is the small-case run to bisect a bad access with)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.workloads import charges, icosphere_patches, patch_samples, plummer_points, sphere_points

rng = np.random.default_rng(5)
for layout in ("group", "class"):
    os.environ["HFMM_BATCHING"] = layout
    for order, k in ((6, 3.0), (13, 5.0), (8, 4.0 + 0.7j)):
        n = 3000
        xyz = plummer_points(n, 3) if order == 6 else sphere_points(n, 3)
        op = HfmmCuda(k=k, order=order, ncrit=24)
        op.set_points(xyz)
        y = op.matvec(charges(n, 1))
        assert np.isfinite(y).all()
        print("matvec", layout, order, k, float(np.linalg.norm(y)), flush=True)
del os.environ["HFMM_BATCHING"]

g = np.load(os.path.join(ROOT, "tests", "golden", "solver.npz"))
tables = {key: g["bie_rule_" + key] for key in ("sample_ref", "far_weight", "near_pts", "near_basis", "self_npts", "self_pts", "self_basis")}
patches = icosphere_patches(1)
xyz = patch_samples(patches, tables["sample_ref"])
op = HfmmCuda(k=2.0, order=8, ncrit=24)
op.set_points(xyz)
nnz = op.build_corrections(patches, tables, mode=2, fetch=False)
rhs = np.exp(2.0j * xyz[:, 2])
x, rep = op.gmres(rhs, rtol=1e-3, restart=10, max_iterations=20, precondition=True)
print("corrections nnz", nnz, "gmres", rep, flush=True)
f = op.evaluate_field(x, np.array([[0.0, 0.0, 4.0], [3.0, 1.0, 0.5]]))
print("field", f, flush=True)
print("TOUR OK")
