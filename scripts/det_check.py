"""GPU: HFMM_FLAG_DETERMINISTIC — reproducibility (default mode for contrast), cost at cfg 2, GMRES histories."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.api import HFMM_FLAG_DETERMINISTIC, HFMM_FLAG_PHASE_TIMERS
from paper_1803_09948_b200.workloads import CONFIGS, charges, icosphere_patches, make_points, patch_samples

cfg = CONFIGS["cfg2"]
xyz, q = make_points(cfg, cfg.n), charges(cfg.n, cfg.seed)
for flags, name in ((0, "default"), (HFMM_FLAG_DETERMINISTIC, "deterministic")):
    op = HfmmCuda(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max, leaf_cap=cfg.leaf_cap, flags=flags)
    t0 = time.perf_counter(); op.set_points(xyz); ts = time.perf_counter() - t0
    ys = [op.matvec(q) for _ in range(3)]
    st = op.stats()
    diff = sum(int(np.count_nonzero(y != ys[0])) for y in ys[1:])
    print(f"{name}: setup {ts:.2f} s, matvec {st['matvec_seconds']*1e3:.2f} ms, launches {st['kernel_launches']}, "
          f"device {st['device_bytes']/1e9:.2f} GB, entries differing between runs: {diff}", flush=True)
    del op

g = np.load(os.path.join(ROOT, "tests", "golden", "solver.npz"))
tables = {key: g["bie_rule_" + key] for key in ("sample_ref", "far_weight", "near_pts", "near_basis", "self_npts", "self_pts", "self_basis")}
patches = icosphere_patches(4)
pts = patch_samples(patches, tables["sample_ref"])
rhs = np.exp(4.0j * pts[:, 2])
for flags, name in ((0, "default"), (HFMM_FLAG_DETERMINISTIC, "deterministic")):
    hist = []
    for _ in range(2):
        op = HfmmCuda(k=4.0, order=10, ncrit=64, flags=flags)
        op.set_points(pts)
        op.build_corrections(patches, tables, mode=2, fetch=False)
        x, rep = op.gmres(rhs, rtol=1e-4, restart=30, max_iterations=200, precondition=False)
        hist.append((rep["iterations"], rep["residuals"].copy(), x))
    same = hist[0][0] == hist[1][0] and np.array_equal(hist[0][1], hist[1][1]) and np.array_equal(hist[0][2], hist[1][2])
    print(f"GMRES {name}: iterations {hist[0][0]} / {hist[1][0]}, histories and solutions bitwise equal: {same}", flush=True)
