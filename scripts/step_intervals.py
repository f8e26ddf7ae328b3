"""GPU: intervals of the kernels INSIDE the co-resident step (no phase timers): when the near field runs
relative to M2L.   python scripts/step_intervals.py [cfg2]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.workloads import CONFIGS, charges, make_points

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = CONFIGS[name]
xyz, q = make_points(cfg, cfg.n), charges(cfg.n, cfg.seed)
op = HfmmCuda(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max, leaf_cap=cfg.leaf_cap)
op.set_points(xyz)
rows = []
for _ in range(8):
    op.matvec(q)
    st = op.stats()
    rows.append([st[f"{k}_seconds"] * 1e3 for k in ("p2p", "p2m", "m2m", "m2l", "l2l", "l2p", "matvec")])
med = np.median(np.array(rows[2:]), axis=0)
print(name, "in-step intervals (ms): " + " ".join(f"{k} {v:.3f}" for k, v in zip(("p2p", "p2m", "m2m", "m2l", "l2l", "l2p", "matvec"), med)), flush=True)
