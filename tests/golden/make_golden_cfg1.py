"""Generates tests/golden/cfg1.npz: BASELINE.json configs[0] exactly (16,384 points on the unit sphere,
k = 1, P = 10, ncrit = 64, theta = 0.4; kd_max = 1 and leaf cap kd_max/|k| as the reference's solver path)
evaluated by the UNMODIFIED compiled reference (oracle/_ref/libhfmm_ref.so): its potentials and its tree /
list counts.  The points and charges are not stored — workloads.make_points / charges regenerate them from
the seed.  Run in the authoring container only:  python tests/golden/make_golden_cfg1.py"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from checkers import Ref  # noqa: E402
from paper_1803_09948_b200.workloads import CONFIGS, charges, make_points  # noqa: E402

cfg = CONFIGS["cfg1"]
xyz, q = make_points(cfg), charges(cfg.n, cfg.seed)
f = Ref().fmm(xyz, cfg.k, cfg.order, ncrit=cfg.ncrit, leaf_cap=cfg.resolved_leaf_cap(), theta=cfg.theta,
              kd_max=cfg.kd_max)
y = f.matvec(q)
c = f.counts()
np.savez_compressed(os.path.join(HERE, "cfg1.npz"), potentials=y, xyz_checksum=np.float64(np.abs(xyz).sum()),
                    q_checksum=np.float64(np.abs(q).sum()), tasks=np.int64(f.tasks()),
                    **{k: np.int64(v) for k, v in c.items()})
print({k: int(v) for k, v in c.items()}, "tasks", f.tasks(), "|y|", float(np.abs(y).sum()))
