import sys, os, json
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.api import HFMM_FLAG_NEAR_FIRST
from paper_1803_09948_b200.workloads import CONFIGS, charges, make_points
cfg = CONFIGS["cfg2"]; n = cfg.n
xyz, q = make_points(cfg, n), charges(n, cfg.seed)
q_dev = torch.from_numpy(np.stack([q.real, q.imag], 1).astype(np.float32)).cuda(); out = torch.empty_like(q_dev)
for flags in (0, HFMM_FLAG_NEAR_FIRST):
    op = HfmmCuda(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max, leaf_cap=cfg.leaf_cap, flags=flags)
    op.set_points(xyz)
    for _ in range(3): op.matvec_device(q_dev.data_ptr(), out.data_ptr())
    op.sync(); op.timer_record(0)
    for _ in range(10): op.matvec_device(q_dev.data_ptr(), out.data_ptr())
    op.timer_record(1); ms = op.timer_elapsed_ms(0, 1) / 10
    st = op.stats()
    print("flags", flags, "ms/step %.3f" % ms, "m2l %.2f p2p %.2f" % (st["m2l_seconds"] * 1e3, st["p2p_seconds"] * 1e3), flush=True)
    del op
