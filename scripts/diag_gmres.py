import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from checkers import Oracle, Ref, rel_l2
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.workloads import icosphere_patches
oracle = Oracle()
k, order = 3.0, 10
sysr = Ref().bie(icosphere_patches(2), 1, k, mode=2, use_tree=False)
xyz, fw = sysr.samples(); corr = sysr.corrections(); rhs = sysr.rhs((0, 0, 1))
op = HfmmCuda(k=k, order=order, ncrit=16); op.set_points(xyz); op.set_corrections(sysr.ni, far_weight=fw, **corr)
f = oracle.fmm(xyz, k, order, ncrit=16, leaf_cap=1.0 / k, theta=0.4, kd_max=1.0)
def A(v): return oracle.apply_corrections(sysr.ni, corr["patch_block"], corr["near_offset"], corr["near_source"], corr["near_delta"], v, f.matvec(v * fw))
def z(u): return A(oracle.block_lu_solve(sysr.ni, corr["block_lu"], corr["block_piv"], u))
rng = np.random.default_rng(0)
xr = rng.standard_normal(sysr.n) + 1j * rng.standard_normal(sysr.n)
print("apply rel err random x:", rel_l2(op.matvec(xr), A(xr)), " rhs:", rel_l2(op.matvec(rhs), A(rhs)))
print("dense ref apply vs oracle tree apply:", rel_l2(sysr.apply(xr), A(xr)))
print("|fmm part| vs |corr part|:", np.linalg.norm(f.matvec(xr*fw)), np.linalg.norm(A(xr) - f.matvec(xr*fw)))
for restart in (30, 300):
    xg, rg = op.gmres(rhs, rtol=1e-4, restart=restart, max_iterations=300)
    u, ro = oracle.gmres(z, rhs, rtol=1e-4, restart=restart, max_iterations=300)
    print("restart", restart, "gpu it", rg["iterations"], "cpu it", ro["iterations"], "final", rg["final_residual"], ro["final_residual"])
    m = min(len(rg["residuals"]), len(ro["residuals"]))
    idx = list(range(0, m, 5))
    print("  gpu:", " ".join(f"{rg['residuals'][i]:.2e}" for i in idx))
    print("  cpu:", " ".join(f"{ro['residuals'][i]:.2e}" for i in idx))
# oracle GMRES (FP64 Krylov) over the GPU operator
def zg(u): return op.matvec(oracle.block_lu_solve(sysr.ni, corr["block_lu"], corr["block_piv"], u))
for restart in (30,):
    u, rm = oracle.gmres(zg, rhs, rtol=1e-4, restart=restart, max_iterations=300)
    print("FP64 Krylov over GPU operator: it", rm["iterations"], " ".join(f"{rm['residuals'][i]:.2e}" for i in range(0, len(rm['residuals']), 5)))
# oracle GMRES over oracle operator perturbed at 3e-7
def zp(u):
    y = z(u); return y + 3e-7*np.linalg.norm(y)/np.sqrt(len(y))*(rng.standard_normal(len(y))+1j*rng.standard_normal(len(y)))/np.sqrt(2)
u, rp = oracle.gmres(zp, rhs, rtol=1e-4, restart=30, max_iterations=300)
print("FP64 Krylov over CPU operator + 3e-7 noise: it", rp["iterations"])
