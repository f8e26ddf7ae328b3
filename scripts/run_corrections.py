"""GPU box: time the device correction builders against the compiled reference's
build_system (use_tree = false: patch blocks + near corrections only) on icosphere meshes."""
import os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from checkers import Ref, RefBie, have_ref
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.workloads import icosphere_patches

level = int(sys.argv[1]) if len(sys.argv) > 1 else 4
basis = int(sys.argv[2]) if len(sys.argv) > 2 else 2
k = float(sys.argv[3]) if len(sys.argv) > 3 else 5.0
g2 = np.load(os.path.join(ROOT, "tests", "golden", "corrections_order2.npz" if basis == 2 else "solver.npz"))
pre = "rule_" if basis == 2 else "bie_rule_"
tables = {key: g2[pre + key] for key in ("sample_ref", "far_weight", "near_pts", "near_basis", "self_npts", "self_pts", "self_basis")}
patches = icosphere_patches(level)
out = {"patches": len(patches), "basis_order": basis, "unknowns": len(patches) * len(tables["far_weight"])}
ref = None
if have_ref():
    R = Ref()
    t0 = time.time()
    ref = RefBie(R, patches, basis, k, 2, False, 8, 64, 0.4, 1.0, -1.0, os.cpu_count())
    out["reference_seconds"] = time.time() - t0
    out["reference_threads"] = os.cpu_count()
    want = ref.corrections()
    xyz = ref.samples()[0]
else:
    from checkers import Oracle
    want = Oracle().build_corrections(patches, tables, k)
    xyz = want["xyz"]
op = HfmmCuda(k=k, order=8, ncrit=64)
op.set_points(xyz)
for rep in range(2):
    t0 = time.time()
    nnz = op.build_corrections(patches, tables, fetch=False)
    out["device_seconds"] = time.time() - t0
out["near_nnz"] = nnz
got = op.build_corrections(patches, tables)
out["lists_equal"] = bool(np.array_equal(got["near_source"], want["near_source"]) and np.array_equal(got["near_offset"], want["near_offset"]))
out["max_rel_diff"] = max(float(np.abs(got[key] - want[key]).max() / np.abs(want[key]).max()) for key in ("patch_block", "block_lu", "near_delta"))
print(json.dumps(out))
