"""GPU: near-field kernel variants (HFMM_P2P_MODE) — kernel-alone time and accuracy.

    python scripts/p2p_variants.py [cfg2] [n]

Accuracy: (i) a near-only problem (gate closed, everything is P2P) against the FP64 direct sum,
(ii) the full matvec of the configuration against the FP64 direct sum on 2,048 sampled targets."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

from checkers import Oracle, rel_l2
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.api import HFMM_FLAG_PHASE_TIMERS
from paper_1803_09948_b200.workloads import CONFIGS, charges, make_points, sphere_points

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = CONFIGS[name]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n
modes = [int(m) for m in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, 1, 2, 3]
xyz, q = make_points(cfg, n), charges(n, cfg.seed)
orc = Oracle()
rng = np.random.default_rng(1)
sample = np.sort(rng.choice(n, 2048, replace=False))
exact = orc.direct_sum(xyz, q, cfg.k, targets=sample)
# near-only: small leaves (cap) so that R' stays bounded, no far field
n2 = 20000
xyz2, q2 = 0.5 * sphere_points(n2, 9), charges(n2, 9)   # k * box diagonal = 3.5: bounded R'
exact2 = orc.direct_sum(xyz2, q2, 2.0)
for mode in modes:
    os.environ["HFMM_P2P_MODE"] = str(mode)
    op = HfmmCuda(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max,
                  leaf_cap=cfg.leaf_cap, flags=HFMM_FLAG_PHASE_TIMERS)
    op.set_points(xyz)
    y = op.matvec(q)
    ts = []
    for _ in range(5):
        op.matvec(q)
        ts.append(op.stats()["p2p_seconds"])
    st = op.stats()
    t = float(np.median(ts))
    err = rel_l2(y[sample], exact)
    del op
    # the whole step with the near field co-resident under M2L (default flags)
    opc = HfmmCuda(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max, leaf_cap=cfg.leaf_cap)
    opc.set_points(xyz)
    tt = []
    for _ in range(6):
        opc.matvec(q)
        tt.append(opc.stats()["matvec_seconds"])
    step = float(np.median(tt[1:]))
    del opc
    op2 = HfmmCuda(k=2.0, order=4, ncrit=50, theta=0.4, kd_max=1e-9, leaf_cap=0.0)
    op2.set_points(xyz2)
    y2 = op2.matvec(q2)
    st2 = op2.stats()
    err2 = rel_l2(y2, exact2)
    del op2
    print(f"mode {mode} (ran {st['p2p_mode']}, r2max {st['near_r2_max']:.3f}): step {step*1e3:.3f} ms  p2p {t*1e3:.3f} ms  "
          f"{st['p2p_body_pairs']*24/t*1e-12:.2f} TFLOP/s  matvec err {err:.3e} | near-only (mode {st2['p2p_mode']}, "
          f"r2max {st2['near_r2_max']:.2f}, m2l {st2['m2l_pairs']}) err {err2:.3e}", flush=True)
