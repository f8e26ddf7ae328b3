"""960-unknown restarted GMRES: iteration counts and residual tails of device / same-operator / FP64 runs"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from checkers import Oracle, Ref
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.api import HFMM_FLAG_DETERMINISTIC
from paper_1803_09948_b200.workloads import icosphere_patches

oracle = Oracle()
k, order = 3.0, 10
sysr = Ref().bie(icosphere_patches(2), 1, k, mode=2, use_tree=False)
xyz, fw = sysr.samples(); corr = sysr.corrections()
f = oracle.fmm(xyz, k, order, ncrit=16, leaf_cap=1.0 / k, theta=0.4, kd_max=1.0)
minv = lambda u: oracle.block_lu_solve(sysr.ni, corr["block_lu"], corr["block_piv"], u)
def z_cpu(u):
    v = minv(u)
    return oracle.apply_corrections(sysr.ni, corr["patch_block"], corr["near_offset"], corr["near_source"], corr["near_delta"], v, f.matvec(v * fw))
for flags in (HFMM_FLAG_DETERMINISTIC, 0):
    op = HfmmCuda(k=k, order=order, ncrit=16, flags=flags); op.set_points(xyz); op.set_corrections(sysr.ni, far_weight=fw, **corr)
    for direction in [(0.36, 0.48, 0.8), (0.6, 0.0, 0.8), (0.48, 0.6, 0.64), (1/3**.5,)*3, (0.8, 0.6, 0.0)]:
        rhs = sysr.rhs(direction)
        _, rd = op.gmres(rhs, rtol=1e-4, restart=30, max_iterations=300)
        _, rs = oracle.gmres(lambda u: op.matvec(minv(u)), rhs, rtol=1e-4, restart=30, max_iterations=300)
        _, rc = oracle.gmres(z_cpu, rhs, rtol=1e-4, restart=30, max_iterations=300)
        print(f"flags={flags} dir={direction}: device {rd['iterations']} same-op {rs['iterations']} fp64 {rc['iterations']}")
        print("   device tail", " ".join(f"{v:.3e}" for v in rd["residuals"][-6:]))
        print("   fp64   tail", " ".join(f"{v:.3e}" for v in rc["residuals"][-6:]))
