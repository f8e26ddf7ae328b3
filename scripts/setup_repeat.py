"""GPU: repeated set_points on one handle — wall time and the handle's own setup_seconds per call."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.workloads import CONFIGS, charges, make_points

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
xyz, q = make_points(cfg, cfg.n), charges(cfg.n, cfg.seed)
op = HfmmCuda(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max, leaf_cap=cfg.leaf_cap)
for i in range(8):
    t0 = time.perf_counter()
    op.set_points(xyz)
    wall = time.perf_counter() - t0
    print(f"call {i}: wall {wall:.3f} s, setup_seconds {op.stats()['setup_seconds']:.3f}", flush=True)
    if i % 2:
        op.matvec(q)
