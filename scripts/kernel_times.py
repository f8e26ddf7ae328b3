"""GPU: per-kernel times of one configuration (serialised: HFMM_FLAG_PHASE_TIMERS), the co-resident
step time, and the error against the FP64 direct sum on sampled targets.

    python scripts/kernel_times.py [cfg2] [n] [order]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import dataclasses
import numpy as np

from checkers import Oracle, rel_l2
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.api import HFMM_FLAG_PHASE_TIMERS
from paper_1803_09948_b200.workloads import CONFIGS, charges, make_points

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = CONFIGS[name]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n
if len(sys.argv) > 3:
    cfg = dataclasses.replace(cfg, order=int(sys.argv[3]))
xyz, q = make_points(cfg, n), charges(n, cfg.seed)
rng = np.random.default_rng(1)
sample = np.sort(rng.choice(n, 2048, replace=False))
exact = Oracle().direct_sum(xyz, q, cfg.k, targets=sample)
kw = dict(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max, leaf_cap=cfg.leaf_cap)
op = HfmmCuda(flags=HFMM_FLAG_PHASE_TIMERS, **kw)
op.set_points(xyz)
y = op.matvec(q)
acc = {}
for _ in range(5):
    op.matvec(q)
    st = op.stats()
    for k in ("p2p", "p2m", "m2m", "m2l", "l2l", "l2p", "matvec"):
        acc.setdefault(k, []).append(st[f"{k}_seconds"])
t = {k: float(np.median(v)) * 1e3 for k, v in acc.items()}
err = rel_l2(y[sample], exact)
del op
op = HfmmCuda(**kw)
op.set_points(xyz)
tt = []
for _ in range(6):
    op.matvec(q)
    tt.append(op.stats()["matvec_seconds"])
step = float(np.median(tt[1:])) * 1e3
rot = sum((j + 1) ** 2 + j ** 2 for j in range(cfg.order + 1))
coax = sum((cfg.order + 1 - abs(m)) ** 2 for m in range(-cfg.order, cfg.order + 1))
flop = 2 * (4 * rot + 4 * coax)
print(f"{name} n={n} P={cfg.order}: pairs {st['m2l_pairs']} batches {st['m2l_batches']} "
      f"(fill {st['m2l_pairs'] / max(st['m2l_batches'], 1):.1f}) | " +
      " ".join(f"{k} {v:.3f}" for k, v in t.items()) +
      f" ms | step {step:.3f} ms | M2L {st['m2l_pairs'] * flop / t['m2l'] * 1e-9:.2f} TFLOP/s executed | err {err:.3e}",
      flush=True)
