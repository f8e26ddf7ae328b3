"""GPU: device GMRES on an icosphere (k = 4, P = 12, restart 30, no preconditioner) against the residual history of
the reference's own solve of the same system, produced on host cores by scripts/ref_bie_cpu.py.

    python scripts/cmp_bie_history.py [subdivisions] [reference.json]
defaults: 4 subdivisions (5,120 triangles), profiles/r01_reference_gmres_5120tri_plain.json;
7 subdivisions = BASELINE config 3 (327,680 triangles), profiles/r02_reference_gmres_cfg3_full.json"""
import sys, os, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.workloads import icosphere_patches, patch_samples
sub = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ref = json.load(open(sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "r01_reference_gmres_5120tri_plain.json")))
g = np.load(os.path.join(ROOT, "tests", "golden", "solver.npz"))
tables = {key: g["bie_rule_" + key] for key in ("sample_ref", "far_weight", "near_pts", "near_basis", "self_npts", "self_pts", "self_basis")}
patches = icosphere_patches(sub); xyz = patch_samples(patches, tables["sample_ref"])
k = 4.0
op = HfmmCuda(k=k, order=12, ncrit=64, theta=0.4, kd_max=1.0, leaf_cap=-1.0)
op.set_points(xyz); op.build_corrections(patches, tables, fetch=False)
rhs = np.exp(1j * k * xyz[:, 2])
out = {"triangles": len(patches), "unknowns": len(xyz)}
for restart in ((30, 1000) if sub <= 5 else (30,)):
    x, rep = op.gmres(rhs, rtol=1e-4, restart=restart, max_iterations=1000, precondition=False)
    r = rep["residuals"]
    out[f"restart_{restart}"] = {"iterations": rep["iterations"], "final_residual": rep["final_residual"]}
    if restart == 30:
        rr = np.array(ref["residuals"])
        m = min(len(r), len(rr))
        rel = np.abs(r[:m] - rr[:m]) / rr[:m]
        out["reference_iterations"] = ref["iterations"]
        out["device_residuals"] = [float(v) for v in r]
        out["history_rel_diff_first_10"] = float(rel[:10].max())
        out["history_rel_diff_first_20"] = float(rel[:20].max())
        out["history_rel_diff_first_30"] = float(rel[:30].max())
        out["history_rel_diff_first_60"] = float(rel[:60].max())
        out["history_rel_diff_first_90"] = float(rel[:90].max())
        out["history_rel_diff_all"] = float(rel.max())
        out["residual_at_ref_stop"] = float(r[ref["iterations"] - 1]) if len(r) >= ref["iterations"] else None
print(json.dumps(out))
