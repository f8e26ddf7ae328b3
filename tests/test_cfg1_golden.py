"""CPU: the oracle restatement reproduces the compiled reference's BASELINE configs[0] run (tests/golden/cfg1.npz)."""
import os

import numpy as np

from checkers import rel_l2
from paper_1803_09948_b200.workloads import CONFIGS, charges, make_points


def test_oracle_matches_reference_fixture_at_config_1(oracle):
    cfg = CONFIGS["cfg1"]
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "cfg1.npz"))
    xyz, q = make_points(cfg), charges(cfg.n, cfg.seed)
    assert np.abs(xyz).sum() == float(g["xyz_checksum"])
    f = oracle.fmm(xyz, cfg.k, cfg.order, ncrit=cfg.ncrit, leaf_cap=cfg.resolved_leaf_cap(), theta=cfg.theta,
                   kd_max=cfg.kd_max)
    c = f.counts()
    for key in ("cells", "leaves", "m2l_pairs", "p2p_pairs", "p2p_body_pairs", "max_level"):
        assert c[key] == int(g[key]), key
    assert rel_l2(f.matvec(q), g["potentials"]) < 1e-12
