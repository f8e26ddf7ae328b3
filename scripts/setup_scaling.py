"""GPU: setup (tree + lists + tables) time and one matvec at larger configs, device vs host builder."""
import sys, os, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from checkers import Oracle, rel_l2
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.api import HFMM_FLAG_HOST_TREE
from paper_1803_09948_b200.workloads import CONFIGS, make_points, charges
cases = [("cfg2", 1048576), ("cfg5_per_gpu", 4194304), ("cfg4", 4194304)]
if len(sys.argv) > 1:
    cases = [(sys.argv[1], int(sys.argv[2]))]
for name, n in cases:
    cfg = CONFIGS[name]; xyz = make_points(cfg, n); q = charges(n, cfg.seed)
    for fl in (0, HFMM_FLAG_HOST_TREE):
        if fl and n > 2_000_000: continue
        op = HfmmCuda(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max, leaf_cap=cfg.leaf_cap, flags=fl)
        t0 = time.time(); op.set_points(xyz); dt = time.time() - t0
        y = op.matvec(q); y = op.matvec(q); st = op.stats()
        gb = st["device_bytes"] / 1e9
        print(name, n, "host" if fl else "device", f"setup {dt:.2f}s cells {st['n_cells']} m2l {st['m2l_pairs']} p2p_body {st['p2p_body_pairs']:.3e} classes {st['m2l_shift_classes']} {gb:.2f} GB; matvec {st['matvec_seconds']*1e3:.1f} ms (p2p {st['p2p_seconds']*1e3:.1f} m2l {st['m2l_seconds']*1e3:.1f} p2m {st['p2m_seconds']*1e3:.1f} l2p {st['l2p_seconds']*1e3:.1f})", flush=True)
        if not fl:
            tg = np.random.default_rng(0).choice(n, 512, replace=False)
            print("   rel_l2 vs FP64 direct sum (512 targets):", f"{rel_l2(y[tg], Oracle().direct_sum(xyz, q, cfg.k, tg)):.3e}", flush=True)
        del op
