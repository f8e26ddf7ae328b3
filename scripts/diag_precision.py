"""GPU diagnostic: where does the FP32 error of the matvec come from? (near / multipoles / locals)"""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from checkers import Oracle, rel_l2
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.workloads import charges, sphere_points

O = Oracle()
for (n, k, order, ncrit, cap) in [(4096, 1.0, 8, 32, -1.0), (6000, 4.0, 12, 64, -1.0), (4096, 2.0, 10, 64, -1.0)]:
    xyz, q = sphere_points(n, 5), charges(n, 5)
    cap_res = cap if cap >= 0 else 1.0 / k
    op = HfmmCuda(k=k, order=order, ncrit=ncrit, leaf_cap=cap)
    op.set_points(xyz)
    y = op.matvec(q)
    f = O.fmm(xyz, k, order, ncrit=ncrit, leaf_cap=cap_res)
    yr = f.matvec(q)
    print(f"n={n} k={k} P={order}: total rel_l2={rel_l2(y, yr):.3e}  stats levels={op.stats()['max_level']}")
    key = lambda c: [tuple(r) for r in c[:, :4].tolist()]
    mine = {kk: i for i, kk in enumerate(key(op.cells()))}
    perm = np.array([mine[kk] for kk in key(f.cells())])
    lvl = f.cells()[:, 0]
    leaf = f.cells()[:, 7] == 0
    for which, name in ((0, "multipole"), (1, "local")):
        a = op.expansions(which)[perm]; b = f.expansions(which, order)
        used = np.abs(a).sum(axis=1) > 0
        for L in sorted(set(lvl[used])):
            sel = used & (lvl == L)
            for lf in (True, False):
                s2 = sel & (leaf == lf)
                if not s2.any(): continue
                err = np.linalg.norm(a[s2] - b[s2], axis=1) / np.linalg.norm(b[s2], axis=1)
                # per-degree error
                pern = []
                for nn in range(order + 1):
                    sl = slice(nn * nn, (nn + 1) ** 2)
                    pern.append(np.linalg.norm(a[s2][:, sl] - b[s2][:, sl]) / max(np.linalg.norm(b[s2][:, sl]), 1e-300))
                print(f"  {name} L{L} leaf={lf}: cells={s2.sum()} max={err.max():.2e} mean={err.mean():.2e} per-n=" + " ".join(f"{v:.0e}" for v in pern))
    # near-only
    op2 = HfmmCuda(k=k, order=2, ncrit=ncrit, kd_max=1e-9, leaf_cap=0.0)
    op2.set_points(xyz)
    print(f"  near-only vs direct: {rel_l2(op2.matvec(q), O.direct_sum(xyz, q, k)):.3e}")
