"""GPU + compiled reference: where do the extra GMRES iterations on the lat-long sphere come from?
FP64 Krylov over the FP64 operator / over the device operator / over the FP64 operator with noise, and the
device solver."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from checkers import Oracle, Ref, rel_l2
from paper_1803_09948_b200 import HfmmCuda

seg, rings, k, order = int(sys.argv[1]) if len(sys.argv) > 1 else 16, int(sys.argv[2]) if len(sys.argv) > 2 else 10, 4.0, 10
ref, oracle = Ref(), Oracle()
patches = ref.sphere_mesh(1.0, seg, rings)
sysr = ref.bie(patches, 1, k, mode=2, use_tree=True, order=order, ncrit=32, theta=0.4, kd_max=1.0)
xyz, fw = sysr.samples(); corr = sysr.corrections(); rhs = sysr.rhs((0, 0, 1))
op = HfmmCuda(k=k, order=order, ncrit=32, theta=0.4); op.set_points(xyz); op.set_corrections(sysr.ni, far_weight=fw, **corr)
print("unknowns", len(rhs), "apply err", rel_l2(op.matvec(rhs), sysr.apply(rhs)))
minv = lambda u: oracle.block_lu_solve(sysr.ni, corr["block_lu"], corr["block_piv"], u)
rng = np.random.default_rng(0)
for pre in (True, False):
    P = minv if pre else (lambda u: u)
    z64 = lambda u: sysr.apply(P(u))
    zg = lambda u: op.matvec(P(u))
    def zn(u, eps=1.5e-7):
        y = z64(u); return y + eps * np.linalg.norm(y) / np.sqrt(len(y)) * (rng.standard_normal(len(y)) + 1j * rng.standard_normal(len(y))) / np.sqrt(2)
    def z32in(u):   # FP64 operator applied to the FP32-rounded operand
        return z64(u.astype(np.complex64).astype(np.complex128))
    _, r_ref = sysr.gmres(rhs, rtol=1e-4, restart=30, max_iterations=300, precondition=pre)
    _, r64 = oracle.gmres(z64, rhs, rtol=1e-4, restart=30, max_iterations=300)
    _, rg = oracle.gmres(zg, rhs, rtol=1e-4, restart=30, max_iterations=300)
    _, rn = oracle.gmres(zn, rhs, rtol=1e-4, restart=30, max_iterations=300)
    _, r32 = oracle.gmres(z32in, rhs, rtol=1e-4, restart=30, max_iterations=300)
    _, rd = op.gmres(rhs, rtol=1e-4, restart=30, max_iterations=300, precondition=pre)
    print(f"precondition={pre}: reference {r_ref['iterations']} | FP64 Krylov: FP64 op {r64['iterations']}, device op {rg['iterations']}, "
          f"FP64 op + 1.5e-7 noise {rn['iterations']}, FP64 op on FP32 operand {r32['iterations']} | device solver {rd['iterations']}")
    print("   residuals device :", " ".join(f"{v:.1e}" for v in rd["residuals"][::4]))
    print("   residuals fp64   :", " ".join(f"{v:.1e}" for v in r64["residuals"][::4]))

# ---- which stage carries the perturbation?  FP64 Krylov (oracle.gmres) over hybrid operators -------------
from paper_1803_09948_b200.api import HFMM_FLAG_DETERMINISTIC
fr = ref.fmm(xyz, k, order, ncrit=32, leaf_cap=1.0 / k, theta=0.4, kd_max=1.0)
opd = HfmmCuda(k=k, order=order, ncrit=32, theta=0.4, flags=HFMM_FLAG_DETERMINISTIC); opd.set_points(xyz)
opd.set_corrections(sysr.ni, far_weight=fw, **corr)
plain = HfmmCuda(k=k, order=order, ncrit=32, theta=0.4, flags=HFMM_FLAG_DETERMINISTIC); plain.set_points(xyz)
plain.set_corrections(sysr.ni, far_weight=fw)
corr64 = lambda v, y: oracle.apply_corrections(sysr.ni, corr["patch_block"], corr["near_offset"], corr["near_source"], corr["near_delta"], v, y)
ops = {
    "A all FP64": lambda v: corr64(v, fr.matvec(v * fw)),
    "B reference FMM with its f32 P2P + FP64 corrections": lambda v: corr64(v, fr.matvec(v * fw, f32_p2p=True)),
    "C device FMM + FP64 corrections": lambda v: corr64(v, plain.matvec(v)),
    "D FP64 FMM + device corrections": lambda v: fr.matvec(v * fw) + (opd.matvec(v) - plain.matvec(v)),
    "E device": lambda v: opd.matvec(v),
}
for pre in (True, False):
    P = minv if pre else (lambda u: u)
    out = []
    for name, A in ops.items():
        _, r = oracle.gmres(lambda u: A(P(u)), rhs, rtol=1e-4, restart=30, max_iterations=300)
        out.append(f"{name}: {r['iterations']}")
    print(f"precondition={pre}  " + " | ".join(out))
