import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
from checkers import Oracle, rel_l2
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.api import HFMM_FLAG_HOST_TREE
from paper_1803_09948_b200.workloads import sphere_points, plummer_points, charges
O = Oracle()
for name, xyz, k, P in (("sphere", sphere_points(20000, 2), 4.0, 12), ("plummer", plummer_points(15000, 3), 8.0, 14), ("ck", sphere_points(8000, 4), 2.0 + 0.4j, 10)):
    q = charges(len(xyz), 7)
    ys = []
    for flags in (0, HFMM_FLAG_HOST_TREE):
        op = HfmmCuda(k=k, order=P, flags=flags); op.set_points(xyz); ys.append(op.matvec(q)); st = op.stats()
        print(name, "flags", flags, "batches", st["m2l_batches"], "classes", st["m2l_shift_classes"], "pairs", st["m2l_pairs"])
    tg = np.random.default_rng(0).choice(len(xyz), 512, replace=False)
    ex = O.direct_sum(xyz, q, k, tg)
    print(name, "device-vs-host builder %.2e" % rel_l2(ys[0], ys[1]), "vs direct %.2e %.2e" % (rel_l2(ys[0][tg], ex), rel_l2(ys[1][tg], ex)))
