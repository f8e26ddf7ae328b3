"""GPU: setup cost of one rank of an R-rank job against the single-domain setup of the same point set
(per-rank pair lists: census + pruned walk).   python scripts/setup_per_rank.py [n] [ranks] [rank]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.workloads import CONFIGS, make_points

cfg = CONFIGS["cfg5"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8 * 1048576
ranks = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rank = int(sys.argv[3]) if len(sys.argv) > 3 else ranks // 2
xyz = make_points(cfg, n)
kw = dict(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max, leaf_cap=cfg.leaf_cap)
for world, r in ((1, 0), (ranks, rank)):
    for rep in range(2):
        op = HfmmCuda(**kw)
        op.set_partition(r, world)
        t0 = time.perf_counter()
        op.set_points(xyz)
        t1 = time.perf_counter()
        masks = op.exchange_masks() if world > 1 else None
        t2 = time.perf_counter()
        st = op.stats()
        stored = sum(len(op.pairs(w)) for w in (0, 1)) if rep == 1 else 0
        if rep == 1:
            print(f"n={n} world={world} rank={r}: set_points {t1 - t0:.3f} s, exchange masks {t2 - t1:.3f} s, "
                  f"device bytes {st['device_bytes'] / 2**30:.2f} GiB, stored pairs {stored} of "
                  f"{st['m2l_pairs'] + st['p2p_pairs']} global", flush=True)
        del op
