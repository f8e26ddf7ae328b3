"""GPU: M2L time and executed TFLOP/s of cfg 2's point set at several expansion orders (the kernel runs
8 warps x 2 CTAs per SM up to P = 12 and 16 warps x 1 CTA above)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import m2l_flops_per_pair
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.api import HFMM_FLAG_PHASE_TIMERS
from paper_1803_09948_b200.workloads import CONFIGS, charges, make_points

cfg = CONFIGS["cfg2"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.n
xyz, q = make_points(cfg, n), charges(n, cfg.seed)
for order in [int(a) for a in sys.argv[2:]] or [8, 10, 11, 12, 13, 14, 16]:
    op = HfmmCuda(k=cfg.k, order=order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max,
                  leaf_cap=cfg.leaf_cap, flags=HFMM_FLAG_PHASE_TIMERS)
    op.set_points(xyz)
    best = 1e9
    for _ in range(4):
        op.matvec(q)
        best = min(best, op.stats()["m2l_seconds"])
    st = op.stats()
    ex, _ = m2l_flops_per_pair(order)
    print(f"P={order:2d} pairs={st['m2l_pairs']} batches={st['m2l_batches']} m2l={best*1e3:7.2f} ms "
          f"{st['m2l_pairs']*ex/best*1e-12:6.2f} TFLOP/s executed ({ex} flop/pair)", flush=True)
    del op
