import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
from checkers import Ref, rel_l2
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.workloads import icosphere_patches
R = Ref()
for sub in (1, 2, 3):
    patches = icosphere_patches(sub); k = 4.0
    sysr = R.bie(patches, 1, k, mode=2, use_tree=True, order=12, ncrit=64, theta=0.4, kd_max=1.0, leaf_cap=-1.0)
    xyz, fw = sysr.samples(); corr = sysr.corrections()
    rng = np.random.default_rng(sub); x = rng.standard_normal(sysr.n) + 1j * rng.standard_normal(sysr.n)
    y_ref = sysr.apply(x)
    op = HfmmCuda(k=k, order=12, ncrit=64, theta=0.4, kd_max=1.0, leaf_cap=-1.0)
    op.set_points(xyz); op.set_corrections(sysr.ni, far_weight=fw, **corr)
    y = op.matvec(x)
    # split: plain FMM part only
    op2 = HfmmCuda(k=k, order=12, ncrit=64, theta=0.4, kd_max=1.0, leaf_cap=-1.0); op2.set_points(xyz)
    yp = op2.matvec(x * fw)
    print(sub, sysr.n, "operator rel err %.2e" % rel_l2(y, y_ref), " |plain|/|y| = %.1f" % (np.linalg.norm(yp) / np.linalg.norm(y_ref)))
