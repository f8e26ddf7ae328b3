"""ctypes windows onto the two CPU checkers (TEST INFRASTRUCTURE, never imported by the product):

* ``Ref``    — oracle/_ref/libhfmm_ref.so, the unmodified reference + oracle/ref_shim.cpp
* ``Oracle`` — oracle/libhfmm_oracle.so, our plain-C restatement (oracle/hfmm_oracle.c)

Both expose the same Python surface so a test can run against either.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libhfmm_ref.so")
ORACLE_SO = os.path.join(ORACLE_DIR, "libhfmm_oracle.so")

_dp = C.POINTER(C.c_double)


def _d(a):
    return a.ctypes.data_as(_dp)


def _c128(a):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return a


def build_oracle():
    if not os.path.exists(ORACLE_SO):
        subprocess.check_call(["make", "-C", ORACLE_DIR, "oracle"], stdout=subprocess.DEVNULL)
    return ORACLE_SO


def have_ref() -> bool:
    return os.path.exists(REF_SO)


class _Fmm:
    def __init__(self, lib, prefix, handle, n):
        self.lib, self.p, self.h, self.n = lib, prefix, handle, n

    def _f(self, name):
        return getattr(self.lib, f"{self.p}_fmm_{name}")

    def counts(self):
        c = (C.c_longlong * 10)()
        self._f("counts")(self.h, c)
        keys = ["cells", "leaves", "m2l_pairs", "p2p_pairs", "p2p_body_pairs", "max_level",
                "m2l_groups", "p2p_groups", "max_m2l_list", "max_p2p_list"]
        return dict(zip(keys, [int(v) for v in c]))

    def tasks(self):
        f = self._f("tasks")
        f.restype = C.c_longlong
        return int(f(self.h))

    def starved(self):
        f = self._f("starved")
        f.restype = C.c_longlong
        return int(f(self.h))

    def cells(self):
        nc = self.counts()["cells"]
        out = np.zeros((nc, 8), dtype=np.uint32)
        self._f("cells")(self.h, out.ctypes.data_as(C.c_void_p))
        return out

    def box(self):
        out = np.zeros(4)
        self._f("box")(self.h, _d(out))
        return out

    def measure_weights(self):
        """partition.cpp:143-163: (local, remote) per body, caller order"""
        local, remote = np.zeros(self.n), np.zeros(self.n)
        getattr(self.lib, f"{self.p}_measure_weights")(self.h, _d(local), _d(remote))
        return local, remote

    def body_order(self):
        out = np.zeros(self.n, dtype=np.uint32)
        self._f("body_order")(self.h, out.ctypes.data_as(C.c_void_p))
        return out

    def plan(self, which):
        c = self.counts()
        ng = c["p2p_groups"] if which else c["m2l_groups"]
        npairs = c["p2p_pairs"] if which else c["m2l_pairs"]
        t = np.zeros(ng, dtype=np.uint32)
        off = np.zeros(ng + 1, dtype=np.uint64)
        s = np.zeros(max(npairs, 1), dtype=np.uint32)
        self._f("plan")(self.h, which, t.ctypes.data_as(C.c_void_p), off.ctypes.data_as(C.c_void_p),
                        s.ctypes.data_as(C.c_void_p))
        return t, off, s[:npairs]

    def pair_set(self, which):
        """canonical (target, source) pairs sorted, for list parity"""
        t, off, s = self.plan(which)
        tt = np.repeat(t, np.diff(off).astype(np.int64))
        return np.stack([tt, s], 1)

    def matvec(self, q, f32_p2p=False):
        q = _c128(q)
        out = np.zeros(self.n, dtype=np.complex128)
        rc = self._f("matvec")(self.h, q.ctypes.data_as(_dp), int(f32_p2p), out.ctypes.data_as(_dp))
        assert rc == 0
        return out

    def seconds(self):
        s = np.zeros(3)
        self._f("seconds")(self.h, _d(s))
        return s

    def expansions(self, which, order):
        nc = self.counts()["cells"]
        out = np.zeros((nc, (order + 1) ** 2), dtype=np.complex128)
        self._f("expansions")(self.h, which, out.ctypes.data_as(_dp))
        return out

    def close(self):
        if self.h:
            self._f("destroy")(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


MATVEC_CB = C.CFUNCTYPE(None, C.c_void_p, C.c_long, _dp, _dp)


class _Base:
    prefix = ""

    def _fn(self, name):
        return getattr(self.lib, f"{self.prefix}_{name}")

    # ---- special functions
    def sph_jn(self, nmax, z):
        raise NotImplementedError

    def ynm(self, nmax, d):
        out = np.zeros((nmax + 1) ** 2, dtype=np.complex128)
        d = np.ascontiguousarray(d, dtype=np.float64)
        self._fn("ynm")(nmax, _d(d), out.ctypes.data_as(_dp))
        return out

    def wigner3j(self, *a):
        f = self._fn("wigner3j")
        f.restype = C.c_double
        return f(*[int(v) for v in a])

    def direct_sum(self, xyz, q, k, targets=None):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        q = _c128(q)
        n = xyz.shape[0]
        if targets is None:
            nt, tp = n, None
        else:
            targets = np.ascontiguousarray(targets, dtype=np.int64)
            nt, tp = len(targets), targets.ctypes.data_as(C.c_void_p)
        out = np.zeros(nt, dtype=np.complex128)
        self._direct(n, xyz, q, k, nt, tp, out)
        return out

    def gmres(self, matvec, rhs, rtol=1e-4, restart=30, max_iterations=500):
        rhs = _c128(rhs)
        n = len(rhs)

        def cb(_user, nn, xp, yp):
            x = np.ctypeslib.as_array(xp, shape=(2 * nn,)).view(np.complex128)
            y = np.ctypeslib.as_array(yp, shape=(2 * nn,)).view(np.complex128)
            y[:] = matvec(x.copy())

        x = np.zeros(n, dtype=np.complex128)
        rep = np.zeros(5)
        res = np.zeros(max_iterations + 1)
        rc = self._fn("gmres")(MATVEC_CB(cb), None, C.c_long(n), rhs.ctypes.data_as(_dp),
                               C.c_double(rtol), restart, max_iterations, x.ctypes.data_as(_dp),
                               _d(rep), _d(res), len(res))
        assert rc == 0
        it = int(rep[0])
        return x, dict(iterations=it, converged=bool(rep[1]), breakdown=bool(rep[2]),
                       rhs_norm=rep[3], final_residual=rep[4], residuals=res[:it].copy())


class Oracle(_Base):
    prefix = "ho"

    def __init__(self):
        self.lib = C.CDLL(build_oracle())

    def build_corrections(self, patches, tables, k, mode=2, near_patch_distance=-1.0):
        return _oracle_build_corrections(self.lib, patches, tables, k, mode, near_patch_distance)

    def sph_jn(self, nmax, z):
        out = np.zeros(nmax + 1)
        self.lib.ho_sph_jn(nmax, C.c_double(z), _d(out))
        return out.astype(np.complex128)

    def sph_hn(self, nmax, z):
        out = np.zeros(nmax + 1, dtype=np.complex128)
        self.lib.ho_sph_hn(nmax, C.c_double(z), out.ctypes.data_as(_dp))
        return out

    def translation_matrix(self, k, t, order, singular):
        dim = (order + 1) ** 2
        out = np.zeros((dim, dim), dtype=np.complex128)
        t = np.ascontiguousarray(t, dtype=np.float64)
        if np.imag(k) != 0:
            self.lib.ho_translation_matrix_complex_k(C.c_double(np.real(k)), C.c_double(np.imag(k)), _d(t), order,
                                                     int(singular), out.ctypes.data_as(_dp))
        else:
            self.lib.ho_translation_matrix(C.c_double(np.real(k)), _d(t), order, int(singular), out.ctypes.data_as(_dp))
        return out

    def p2m(self, xyz, q, center, k, order):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        q = _c128(q)
        center = np.ascontiguousarray(center, dtype=np.float64)
        out = np.zeros((order + 1) ** 2, dtype=np.complex128)
        self.lib.ho_p2m(C.c_long(len(q)), _d(xyz), q.ctypes.data_as(_dp), _d(center), C.c_double(k),
                        order, out.ctypes.data_as(_dp))
        return out

    def eval_expansion(self, local, order, coeff, center, point, k):
        coeff = _c128(coeff)
        center = np.ascontiguousarray(center, dtype=np.float64)
        point = np.ascontiguousarray(point, dtype=np.float64)
        out = np.zeros(2)
        self.lib.ho_eval_expansion(int(local), order, coeff.ctypes.data_as(_dp), _d(center),
                                   _d(point), C.c_double(k), _d(out))
        return complex(out[0], out[1])

    def fmm(self, xyz, k, order, ncrit=64, leaf_cap=0.0, theta=0.4, kd_max=1.0, s=None, threads=0):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        self.lib.ho_fmm_create_complex_k.restype = C.c_void_p
        h = self.lib.ho_fmm_create_complex_k(C.c_long(xyz.shape[0]), _d(xyz), C.c_double(np.real(k)),
                                             C.c_double(np.imag(k)), order, ncrit, C.c_double(leaf_cap),
                                             C.c_double(theta), C.c_double(kd_max))
        assert h, "ho_fmm_create rejected the configuration"
        for name in ("counts", "cells", "box", "body_order", "plan", "matvec", "seconds",
                     "expansions", "destroy"):
            getattr(self.lib, f"ho_fmm_{name}").argtypes = None
        return _Fmm(_VoidLib(self.lib), "ho", C.c_void_p(h), xyz.shape[0])

    def _direct(self, n, xyz, q, k, nt, tp, out):
        if np.imag(k) != 0:
            self.lib.ho_direct_sum_complex_k(C.c_long(n), _d(xyz), q.ctypes.data_as(_dp), C.c_double(np.real(k)),
                                             C.c_double(np.imag(k)), C.c_long(nt), tp, out.ctypes.data_as(_dp))
            return
        self.lib.ho_direct_sum(C.c_long(n), _d(xyz), q.ctypes.data_as(_dp), C.c_double(np.real(k)),
                               C.c_long(nt), tp, out.ctypes.data_as(_dp))

    def apply_corrections(self, ni, patch_block, near_offset, near_source, near_delta, x, y):
        x = _c128(x)
        y = _c128(y).copy()
        n = len(x)
        pb = _c128(patch_block) if patch_block is not None else None
        nd = _c128(near_delta) if near_delta is not None and len(near_delta) else None
        no = np.ascontiguousarray(near_offset, dtype=np.uint32) if nd is not None else None
        ns = np.ascontiguousarray(near_source, dtype=np.uint32) if nd is not None else None
        vp = lambda a: a.ctypes.data_as(C.c_void_p) if a is not None else None
        self.lib.ho_apply_corrections(C.c_long(n), ni, vp(pb), vp(no), vp(ns), vp(nd),
                                      x.ctypes.data_as(_dp), y.ctypes.data_as(_dp))
        return y

    def block_lu_solve(self, ni, block_lu, block_piv, x):
        x = _c128(x).copy()
        lu = _c128(block_lu)
        piv = np.ascontiguousarray(block_piv, dtype=np.int32)
        self.lib.ho_block_lu_solve(C.c_long(len(x) // ni), ni, lu.ctypes.data_as(_dp),
                                   piv.ctypes.data_as(C.c_void_p), x.ctypes.data_as(_dp))
        return x


class _VoidLib:
    """passes the opaque handle as c_void_p to every fmm accessor"""

    def __init__(self, lib):
        self._lib = lib

    def __getattr__(self, name):
        return getattr(self._lib, name)


def update_alpha(lib, prefix, alpha, runtime, alpha_max=2.0):
    """partition.cpp:175-227 through the reference (prefix "ref") or the oracle ("ho")"""
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    r = np.ascontiguousarray(runtime, dtype=np.float64)
    out = C.c_double()
    rc = getattr(lib, f"{prefix}_update_alpha")(_d(a), _d(r), len(a), C.c_double(alpha_max), C.byref(out))
    assert rc == 0
    return out.value


def _oracle_build_corrections(lib, patches, tables, k, mode=2, near_patch_distance=-1.0):
    from paper_1803_09948_b200.api import make_correction_rules
    r, keep = make_correction_rules(patches, tables, mode, near_patch_distance)
    ni, npatch = r.basis_count, int(r.n_patches)
    n = ni * npatch
    xyz = np.zeros((n, 3))
    lib.ho_correction_samples(C.byref(r), _d(xyz))
    pb = np.zeros(npatch * ni * ni, dtype=np.complex128)
    lu = np.zeros(npatch * ni * ni if mode else 0, dtype=np.complex128)
    piv = np.zeros(npatch * ni if mode else 0, dtype=np.int32)
    vp = lambda a: a.ctypes.data_as(C.c_void_p) if a.size else None
    lib.ho_build_patch_blocks.restype = C.c_int
    rc = lib.ho_build_patch_blocks(C.byref(r), C.c_double(np.real(k)), C.c_double(np.imag(k)), vp(pb), vp(lu), vp(piv))
    assert rc == 0, "singular self block"
    off = np.zeros(n + 1, dtype=np.uint32)
    srcp = C.POINTER(C.c_uint32)()
    lib.ho_build_near_lists.restype = C.c_long
    nnz = lib.ho_build_near_lists(C.byref(r), vp(off), C.byref(srcp))
    src = np.ctypeslib.as_array(srcp, shape=(nnz,)).copy() if nnz else np.zeros(0, dtype=np.uint32)
    if nnz:
        lib.ho_free(srcp)
    dl = np.zeros(nnz, dtype=np.complex128)
    if nnz:
        lib.ho_build_near_deltas(C.byref(r), C.c_double(np.real(k)), C.c_double(np.imag(k)), vp(off), vp(src), vp(dl))
    return dict(xyz=xyz, patch_block=pb, block_lu=lu, block_piv=piv, near_offset=off, near_source=src,
                near_delta=dl)


class Ref(_Base):
    prefix = "ref"

    def correction_tables(self, basis_order, near_rule=25, self_rule=8):
        """geometry.cpp's interpolation / quadrature tables in the layout of hfmm_correction_rules"""
        L = self.lib
        ni = L.ref_geom_basis(basis_order, None, None)
        nodes, w = np.zeros((ni, 2)), np.zeros(ni)
        L.ref_geom_basis(basis_order, _d(nodes), _d(w))

        def basis_at(pts):
            out = np.zeros((len(pts), ni))
            for i, (z, e, _) in enumerate(pts):
                row = np.zeros(ni)
                L.ref_geom_basis_eval(basis_order, C.c_double(z), C.c_double(e), _d(row))
                out[i] = row
            return out

        nq = L.ref_geom_gauss_rule(near_rule, None)
        near = np.zeros((nq, 3))
        L.ref_geom_gauss_rule(near_rule, _d(near))
        self_pts, self_npts = [], []
        for j in range(ni):
            m = L.ref_geom_duffy_rule(C.c_double(nodes[j, 0]), C.c_double(nodes[j, 1]), self_rule, None)
            p = np.zeros((m, 3))
            L.ref_geom_duffy_rule(C.c_double(nodes[j, 0]), C.c_double(nodes[j, 1]), self_rule, _d(p))
            self_pts.append(p)
            self_npts.append(m)
        self_pts = np.concatenate(self_pts)
        return dict(sample_ref=nodes, far_weight=w, near_pts=near, near_basis=basis_at(near),
                    self_npts=np.array(self_npts, dtype=np.int32), self_pts=self_pts,
                    self_basis=basis_at(self_pts))

    def __init__(self):
        if not have_ref():
            raise FileNotFoundError(REF_SO)
        self.lib = C.CDLL(REF_SO)
        self.lib.ref_last_error.restype = C.c_char_p

    def err(self):
        return self.lib.ref_last_error().decode()

    def sph_jn(self, nmax, z):
        out = np.zeros(nmax + 1, dtype=np.complex128)
        self.lib.ref_sph_jn(nmax, C.c_double(z), C.c_double(0), out.ctypes.data_as(_dp))
        return out

    def sph_hn(self, nmax, z):
        out = np.zeros(nmax + 1, dtype=np.complex128)
        self.lib.ref_sph_hn(nmax, C.c_double(z), C.c_double(0), out.ctypes.data_as(_dp))
        return out

    def translation_matrix(self, k, t, order, singular):
        dim = (order + 1) ** 2
        out = np.zeros((dim, dim), dtype=np.complex128)
        t = np.ascontiguousarray(t, dtype=np.float64)
        rc = self.lib.ref_translation_matrix(C.c_double(np.real(k)), C.c_double(np.imag(k)), _d(t), order,
                                             int(singular), out.ctypes.data_as(_dp))
        assert rc == 0, self.err()
        return out

    def p2m(self, xyz, q, center, k, order):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        q = _c128(q)
        center = np.ascontiguousarray(center, dtype=np.float64)
        out = np.zeros((order + 1) ** 2, dtype=np.complex128)
        rc = self.lib.ref_p2m(C.c_long(len(q)), _d(xyz), q.ctypes.data_as(_dp), _d(center),
                              C.c_double(k), C.c_double(0), order, out.ctypes.data_as(_dp))
        assert rc == 0, self.err()
        return out

    def eval_expansion(self, local, order, coeff, center, point, k):
        coeff = _c128(coeff)
        center = np.ascontiguousarray(center, dtype=np.float64)
        point = np.ascontiguousarray(point, dtype=np.float64)
        out = np.zeros(2)
        rc = self.lib.ref_eval_expansion(int(local), order, coeff.ctypes.data_as(_dp), _d(center),
                                         _d(point), C.c_double(k), C.c_double(0), _d(out))
        assert rc == 0, self.err()
        return complex(out[0], out[1])

    def fmm(self, xyz, k, order, ncrit=64, leaf_cap=0.0, theta=0.4, kd_max=1.0, s=None, threads=0):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        h = C.c_void_p()
        threads = threads or (os.cpu_count() or 1)
        rc = self.lib.ref_fmm_create(C.byref(h), C.c_long(xyz.shape[0]), _d(xyz), C.c_double(np.real(k)),
                                     C.c_double(np.imag(k)), order, ncrit, C.c_double(leaf_cap),
                                     int(s or ncrit), C.c_double(theta), C.c_double(kd_max), threads)
        assert rc == 0, self.err()
        return _Fmm(self.lib, "ref", h, xyz.shape[0])

    def _direct(self, n, xyz, q, k, nt, tp, out):
        rc = self.lib.ref_direct_sum(C.c_long(n), _d(xyz), q.ctypes.data_as(_dp), C.c_double(np.real(k)),
                                     C.c_double(np.imag(k)), C.c_long(nt), tp, out.ctypes.data_as(_dp))
        assert rc == 0, self.err()

    def distributed_matvec(self, xyz, q, k, order, nranks, ncrit=64, leaf_cap=0.0, theta=0.4,
                           kd_max=1.0):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        q = _c128(q)
        out = np.zeros(len(q), dtype=np.complex128)
        let = np.zeros(nranks, dtype=np.uint64)
        rc = self.lib.ref_distributed_matvec(
            C.c_long(len(q)), _d(xyz), q.ctypes.data_as(_dp), C.c_double(k), C.c_double(0), order,
            ncrit, C.c_double(leaf_cap), ncrit, C.c_double(theta), C.c_double(kd_max), nranks,
            out.ctypes.data_as(_dp), let.ctypes.data_as(C.c_void_p))
        assert rc == 0, self.err()
        return out, let

    # ---- BIE
    def bie(self, patches, basis_order, k, mode=2, use_tree=True, order=-1, ncrit=64, theta=0.4,
            kd_max=1.0, leaf_cap=0.0, threads=0):
        return RefBie(self, patches, basis_order, k, mode, use_tree, order, ncrit, theta, kd_max,
                      leaf_cap, threads or (os.cpu_count() or 1))

    def sphere_mesh(self, radius, segments, rings):
        self.lib.ref_sphere_mesh.restype = C.c_long
        ne = self.lib.ref_sphere_mesh(C.c_double(radius), segments, rings, None)
        nodes = np.zeros((ne, 6, 3))
        self.lib.ref_sphere_mesh(C.c_double(radius), segments, rings, _d(nodes))
        return nodes

    def mie_soft_sphere(self, radius, k, obs_r_theta_phi):
        obs = np.ascontiguousarray(obs_r_theta_phi, dtype=np.float64)
        out = np.zeros(obs.shape[0], dtype=np.complex128)
        rc = self.lib.ref_mie_soft_sphere(C.c_double(radius), C.c_double(k), C.c_double(0),
                                          C.c_long(obs.shape[0]), _d(obs), out.ctypes.data_as(_dp))
        assert rc == 0, self.err()
        return out


class RefBie:
    def __init__(self, ref, patches, basis_order, k, mode, use_tree, order, ncrit, theta, kd_max,
                 leaf_cap, threads):
        self.ref, self.lib, self.k = ref, ref.lib, k
        patches = np.ascontiguousarray(patches, dtype=np.float64)
        self.h = C.c_void_p()
        rc = self.lib.ref_bie_create(C.byref(self.h), C.c_long(patches.shape[0]), _d(patches),
                                     basis_order, C.c_double(np.real(k)), C.c_double(np.imag(k)), mode, int(use_tree),
                                     order, ncrit, ncrit, C.c_double(theta), C.c_double(kd_max),
                                     C.c_double(leaf_cap), threads)
        assert rc == 0, ref.err()
        s = (C.c_longlong * 5)()
        self.lib.ref_bie_sizes(self.h, s)
        self.n, self.ni, self.nnz, self.order, self.has_lu = [int(v) for v in s]

    def samples(self):
        xyz = np.zeros((self.n, 3))
        fw = np.zeros(self.n)
        self.lib.ref_bie_samples(self.h, _d(xyz), _d(fw))
        return xyz, fw

    def corrections(self):
        npatch = self.n // self.ni
        pb = np.zeros(npatch * self.ni * self.ni, dtype=np.complex128)
        lu = np.zeros(npatch * self.ni * self.ni if self.has_lu else 0, dtype=np.complex128)
        piv = np.zeros(npatch * self.ni if self.has_lu else 0, dtype=np.int32)
        off = np.zeros(self.n + 1, dtype=np.uint32)
        src = np.zeros(self.nnz, dtype=np.uint32)
        dl = np.zeros(self.nnz, dtype=np.complex128)
        vp = lambda a: a.ctypes.data_as(C.c_void_p) if a.size else None
        self.lib.ref_bie_corrections(self.h, vp(pb), vp(lu), vp(piv), vp(off), vp(src), vp(dl))
        return dict(patch_block=pb, block_lu=lu, block_piv=piv, near_offset=off, near_source=src,
                    near_delta=dl)

    def rhs(self, direction=(0, 0, 1)):
        d = np.ascontiguousarray(direction, dtype=np.float64)
        out = np.zeros(self.n, dtype=np.complex128)
        rc = self.lib.ref_bie_rhs(self.h, _d(d), C.c_double(self.k), C.c_double(0), out.ctypes.data_as(_dp))
        assert rc == 0, self.ref.err()
        return out

    def apply(self, x):
        x = _c128(x)
        y = np.zeros(self.n, dtype=np.complex128)
        rc = self.lib.ref_bie_apply(self.h, x.ctypes.data_as(_dp), y.ctypes.data_as(_dp))
        assert rc == 0, self.ref.err()
        return y

    def gmres(self, rhs, rtol=1e-4, restart=30, max_iterations=500, precondition=True):
        rhs = _c128(rhs)
        x = np.zeros(self.n, dtype=np.complex128)
        rep = np.zeros(5)
        res = np.zeros(max_iterations + 1)
        rc = self.lib.ref_bie_gmres(self.h, rhs.ctypes.data_as(_dp), C.c_double(rtol), restart,
                                    max_iterations, int(precondition), x.ctypes.data_as(_dp),
                                    _d(rep), _d(res), len(res))
        assert rc == 0, self.ref.err()
        it = int(rep[0])
        return x, dict(iterations=it, converged=bool(rep[1]), breakdown=bool(rep[2]),
                       rhs_norm=rep[3], final_residual=rep[4], residuals=res[:it].copy())

    def scattered(self, solution, obs_xyz):
        sol = _c128(solution)
        obs = np.ascontiguousarray(obs_xyz, dtype=np.float64)
        out = np.zeros(obs.shape[0], dtype=np.complex128)
        rc = self.lib.ref_bie_scattered(self.h, sol.ctypes.data_as(_dp), C.c_long(obs.shape[0]),
                                        _d(obs), C.c_double(self.k), C.c_double(0), out.ctypes.data_as(_dp))
        assert rc == 0, self.ref.err()
        return out

    def close(self):
        if self.h:
            self.lib.ref_bie_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
