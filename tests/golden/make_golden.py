"""Generates tests/golden/*.npz from the UNMODIFIED reference compiled into
oracle/_ref/libhfmm_ref.so (see oracle/Makefile).  Run in the authoring container only
(/root/reference must exist):   python tests/golden/make_golden.py

The reference ships no golden vectors; these files pin our oracle and the CUDA path
to what the reference itself computes on small seeded inputs.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from checkers import Ref  # noqa: E402
from paper_1803_09948_b200.workloads import charges, icosphere_patches, plummer_points, sphere_points  # noqa: E402

R = Ref()


def special():
    zs = np.array([1e-3, 0.04, 0.3, 0.49, 0.5, 0.9, 3.7, 12.5, 31.0])
    jn = np.stack([R.sph_jn(28, z) for z in zs])
    hn = np.stack([R.sph_hn(28, z) for z in zs])
    dirs = np.array([[0.3, -0.2, 0.5], [0, 0, 1.0], [0, 0, -2.0], [1.0, 0, 0], [-0.4, 0.4, 0.1],
                     [0, 0, 0]])
    ynm = np.stack([R.ynm(12, d) for d in dirs])
    w3 = [(a, b, c, d, e, -d - e) for a in range(0, 7) for b in range(0, 7)
          for c in range(abs(a - b), a + b + 1, 1) for d in (-a, 0, a) for e in (-b, 0, b)
          if abs(-d - e) <= c]
    w3 = np.array(w3[:600])
    w3v = np.array([R.wigner3j(*t) for t in w3])
    np.savez_compressed(os.path.join(HERE, "special.npz"), zs=zs, jn=jn, hn=hn, dirs=dirs, ynm=ynm,
                        w3_args=w3, w3_vals=w3v)


def translations():
    k, P = 1.7, 5
    shifts = np.array([[0.3, -0.5, 0.4], [0, 0, 0.7], [0, 0, -0.7], [0.5, 0, 0], [-0.2, 0.2, 0.2],
                       [0.125, 0.125, -0.125]])
    sing = np.stack([R.translation_matrix(k, t, P, 1) for t in shifts])
    reg = np.stack([R.translation_matrix(k, t, P, 0) for t in shifts])
    rng = np.random.default_rng(3)
    pts = rng.uniform(-0.1, 0.1, (17, 3))
    q = rng.uniform(-1, 1, 17) + 1j * rng.uniform(-1, 1, 17)
    center = np.array([0.01, -0.02, 0.03])
    M = R.p2m(pts, q, center, k, 8)
    far = np.array([[1.2, 0.4, -0.8], [-2.0, 0.1, 0.3]])
    mv = np.array([R.eval_expansion(0, 8, M, center, p, k) for p in far])
    # complex wavenumber (attenuation): dense matrices for the factored-table composition test
    kc, Pc = 3.0 + 0.8j, 7
    cshifts = np.array([[0.21, -0.33, 0.27], [0, 0, 0.31], [0, 0, -0.31], [0.2, 0, 0],
                        [0.0625, -0.0625, 0.0625], [0.3, 0.1, -0.2]])
    ckinds = np.array([0, 0, 1, 1, 0, 1])            # 0: singular (M2L), 1: regular (M2M / L2L)
    cT = np.stack([R.translation_matrix(kc, t, Pc, 1 if kind == 0 else 0) for t, kind in zip(cshifts, ckinds)])
    np.savez_compressed(os.path.join(HERE, "translations.npz"), k=k, order=P, shifts=shifts,
                        singular=sing, regular=reg, p2m_pts=pts, p2m_q=q, p2m_center=center,
                        p2m_order=8, p2m_coeff=M, eval_points=far, eval_multipole=mv,
                        complex_k=kc, complex_order=Pc, complex_shifts=cshifts, complex_kinds=ckinds,
                        complex_T=cT)


def fmm_cases():
    out = {}
    cases = {
        # the reference's own pipeline test shape (tests/test_fmm.cpp:941-961): 1000 pts, k=2, P=10
        "pipeline": dict(xyz=np.random.default_rng(7).uniform(-1, 1, (1000, 3)), k=2.0, order=10,
                         ncrit=20, leaf_cap=0.5, theta=0.5, kd_max=1.0),
        "sphere": dict(xyz=sphere_points(1500, 4), k=4.0, order=8, ncrit=32, leaf_cap=0.25,
                       theta=0.4, kd_max=1.0),
        "plummer": dict(xyz=plummer_points(1200, 5, 0.05), k=8.0, order=6, ncrit=16,
                        leaf_cap=0.125, theta=0.35, kd_max=1.0),
        "gate_off": dict(xyz=sphere_points(800, 6), k=1.0, order=6, ncrit=24, leaf_cap=0.0,
                         theta=0.4, kd_max=0.0),
    }
    for name, c in cases.items():
        n = c["xyz"].shape[0]
        q = charges(n, 100 + len(name))
        f = R.fmm(c["xyz"], c["k"], c["order"], ncrit=c["ncrit"], leaf_cap=c["leaf_cap"],
                  theta=c["theta"], kd_max=c["kd_max"], threads=1)
        y = f.matvec(q)
        y32 = f.matvec(q, f32_p2p=True)
        cnt = f.counts()
        out.update({f"{name}_xyz": c["xyz"], f"{name}_q": q, f"{name}_y": y, f"{name}_y_f32p2p": y32,
                    f"{name}_direct": R.direct_sum(c["xyz"], q, c["k"]),
                    f"{name}_cells": f.cells(), f"{name}_order": f.body_order(),
                    f"{name}_m2l": f.pair_set(0), f"{name}_p2p": f.pair_set(1),
                    f"{name}_params": np.array([c["k"], c["order"], c["ncrit"], c["leaf_cap"],
                                                c["theta"], c["kd_max"]]),
                    f"{name}_counts": np.array([cnt[k] for k in sorted(cnt)])})
    np.savez_compressed(os.path.join(HERE, "fmm.npz"), **out)


def fmm_complex_wavenumber():
    # k = k_r + i k_i (attenuation): the reference's pipeline takes a complex wavenumber throughout
    xyz = np.concatenate([sphere_points(900, 8), 0.4 * sphere_points(300, 9) + 0.05])
    k, order = 2.0 + 0.5j, 8
    q = charges(len(xyz), 77)
    f = R.fmm(xyz, k, order, ncrit=24, leaf_cap=1.0 / abs(k), theta=0.4, kd_max=1.0, threads=1)
    cnt = f.counts()
    np.savez_compressed(os.path.join(HERE, "fmm_complex_k.npz"), xyz=xyz, q=q, k=k, order=order, ncrit=24,
                        leaf_cap=1.0 / abs(k), theta=0.4, kd_max=1.0, y=f.matvec(q),
                        direct=R.direct_sum(xyz, q, k), m2l_pairs=cnt["m2l_pairs"], p2p_body_pairs=cnt["p2p_body_pairs"])


def mesh_files():
    # the reference's two mesh formats, written by the reference itself (mesh_io.cpp)
    import ctypes as C
    rc = R.lib.ref_write_sphere_mesh(C.c_double(1.0), 8, 5, os.path.join(HERE, "sphere_8x5.msh").encode(),
                                     os.path.join(HERE, "sphere_8x5.hfmm").encode())
    assert rc == 0


def gmres_and_bie():
    rng = np.random.default_rng(11)
    n = 48
    A = np.eye(n) * 4 + 0.5 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    x, rep = R.gmres(lambda v: A @ v, b, rtol=1e-6, restart=10, max_iterations=200)
    out = dict(A=A, b=b, x=x, iterations=rep["iterations"], residuals=rep["residuals"],
               final_residual=rep["final_residual"])
    # small BIE: 80 curved triangles (icosphere, 1 subdivision), order-1 basis, tree operator
    patches = icosphere_patches(1)
    k = 2.0
    sysr = R.bie(patches, 1, k, mode=2, use_tree=True, order=8, ncrit=16, theta=0.4, kd_max=1.0)
    xyz, fw = sysr.samples()
    corr = sysr.corrections()
    rhs = sysr.rhs((0, 0, 1))
    xr = rng.standard_normal(sysr.n) + 1j * rng.standard_normal(sysr.n)
    yr = sysr.apply(xr)
    sol, rep2 = sysr.gmres(rhs, rtol=1e-4, restart=30, max_iterations=200, precondition=True)
    sol0, rep0 = sysr.gmres(rhs, rtol=1e-4, restart=30, max_iterations=200, precondition=False)
    obs = np.array([[0, 0, 3.0], [2.5, 0, 0], [0, -2.0, 2.0]])
    scat = sysr.scattered(sol, obs)
    out.update(bie_patches=patches, bie_k=k, bie_xyz=xyz, bie_far_weight=fw, bie_rhs=rhs,
               bie_x=xr, bie_y=yr, bie_sol=sol, bie_iterations=rep2["iterations"],
               bie_residuals=rep2["residuals"], bie_sol_noprec=sol0,
               bie_iterations_noprec=rep0["iterations"], bie_obs=obs, bie_scattered=scat,
               bie_order=8, bie_ni=sysr.ni, **{f"bie_{k_}": v for k_, v in corr.items()})
    # inputs of the correction builders (solver.cpp:80-230): geometry.cpp's tables for the basis above
    out.update({f"bie_rule_{k_}": v for k_, v in R.correction_tables(1).items()})
    np.savez_compressed(os.path.join(HERE, "solver.npz"), **out)
    # second-order basis (6 functions per patch) on the 20-triangle icosphere: corrections only
    p2 = icosphere_patches(0)
    sys2 = R.bie(p2, 2, 1.5, mode=2, use_tree=False, order=6, ncrit=16, theta=0.4, kd_max=1.0)
    o2 = dict(patches=p2, k=1.5, xyz=sys2.samples()[0], **sys2.corrections())
    o2.update({f"rule_{k_}": v for k_, v in R.correction_tables(2).items()})
    np.savez_compressed(os.path.join(HERE, "corrections_order2.npz"), **o2)


if __name__ == "__main__" and "--complex-only" in sys.argv:
    fmm_complex_wavenumber()
    sys.exit(0)

if __name__ == "__main__":
    special()
    translations()
    fmm_cases()
    fmm_complex_wavenumber()
    mesh_files()
    gmres_and_bie()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)) // 1024, "KiB")
