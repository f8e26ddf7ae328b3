import sys
import os; ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'tests'))
import numpy as np
from checkers import Oracle, Ref
from paper_1803_09948_b200.workloads import icosphere_patches
oracle, ref = Oracle(), Ref()
k, order = 3.0, 10
sysr = ref.bie(icosphere_patches(2), 1, k, mode=2, use_tree=False)
xyz, fw = sysr.samples(); corr = sysr.corrections()
fr = ref.fmm(xyz, k, order, ncrit=16, leaf_cap=1.0 / k, theta=0.4, kd_max=1.0, threads=8)
minv = lambda u: oracle.block_lu_solve(sysr.ni, corr["block_lu"], corr["block_piv"], u)
rng = np.random.default_rng(1)
for direction in [(0.36, 0.48, 0.8), (0.6, 0.0, 0.8), (0.48, 0.6, 0.64), (1/3**.5,)*3, (0.8, 0.6, 0.0)]:
    rhs = sysr.rhs(direction)
    res = []
    for mode in ("f64", "f32p2p", "noise1e-7", "noise3e-7", "in32"):
        def A(u):
            v = minv(u)
            if mode == "in32": v = v.astype(np.complex64).astype(np.complex128)
            y = oracle.apply_corrections(sysr.ni, corr["patch_block"], corr["near_offset"], corr["near_source"], corr["near_delta"], v, fr.matvec(v * fw, f32_p2p=(mode == "f32p2p")))
            if mode.startswith("noise"):
                eps = float(mode[5:])
                y = y + eps * np.linalg.norm(y) / np.sqrt(len(y)) * (rng.standard_normal(len(y)) + 1j * rng.standard_normal(len(y))) / np.sqrt(2)
            return y
        _, rep = oracle.gmres(A, rhs, rtol=1e-4, restart=30, max_iterations=300)
        res.append((mode, rep["iterations"], f"{rep['residuals'][-2]:.3e}"))
    print(direction, res, flush=True)
