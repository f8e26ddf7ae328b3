"""GPU: set up one config and run `reps` matvecs (for ncu captures)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.workloads import CONFIGS, charges, make_points

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else CONFIGS[name].n
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cfg = CONFIGS[name]
xyz, q = make_points(cfg, n), charges(n, cfg.seed)
op = HfmmCuda(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max, leaf_cap=cfg.leaf_cap)
op.set_points(xyz)
for _ in range(reps):
    y = op.matvec(q)
print("done", abs(y).max())
