"""ctypes binding of include/hfmm_cuda.h.  No arithmetic lives here; there is no CPU fallback —
if the shared library or a CUDA device is missing every compute call raises."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libhfmm_b200.so")

HFMM_FLAG_HOST_TREE = 1 << 0
HFMM_FLAG_PHASE_TIMERS = 1 << 1
HFMM_FLAG_NEAR_FIRST = 1 << 2
HFMM_FLAG_DETERMINISTIC = 1 << 3
HFMM_FLAG_NO_HOST_FALLBACK = 1 << 4

_STATUS = {1: "config_error", 2: "singular_error", 3: "structural_error", 4: "accuracy_error",
           5: "domain_error", 6: "device_error", 9: "internal_error"}


class HfmmError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{_STATUS.get(status, status)}: {message}")
        self.status = status
        self.kind = _STATUS.get(status, str(status))


class _Config(C.Structure):
    _fields_ = [("wave_r", C.c_double), ("wave_i", C.c_double), ("order", C.c_int),
                ("ncrit", C.c_int), ("grain", C.c_int), ("theta", C.c_double),
                ("kd_max", C.c_double), ("leaf_cap", C.c_double), ("device", C.c_int),
                ("flags", C.c_int)]


class Stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in
                ("n_bodies", "n_cells", "n_leaves", "max_level", "m2l_pairs", "p2p_pairs",
                 "p2p_body_pairs", "m2l_shift_classes", "rotation_tables", "coaxial_tables",
                 "starved_cells")] + \
               [(n, C.c_double) for n in
                ("setup_seconds", "upward_seconds", "interaction_seconds", "downward_seconds",
                 "p2p_seconds", "m2l_seconds", "p2m_seconds", "m2m_seconds", "l2l_seconds",
                 "l2p_seconds", "matvec_seconds")] + \
               [("kernel_launches", C.c_uint64), ("device_bytes", C.c_uint64), ("m2l_batches", C.c_uint64),
                ("host_tree_used", C.c_uint64), ("p2p_mode", C.c_uint64), ("near_r2_max", C.c_double),
                ("tasks", C.c_uint64), ("p2p_mode_in_step", C.c_uint64)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class Partition(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("n_bodies", C.c_uint64),
                ("body_first", C.c_uint64), ("body_count", C.c_uint64),
                ("level_first", C.c_int32), ("level_last", C.c_int32),
                ("cell_first", C.c_uint32 * 22), ("cell_count", C.c_uint32 * 22),
                ("level_cell_first", C.c_uint32 * 22), ("level_cell_count", C.c_uint32 * 22),
                ("coeff_stride", C.c_uint64), ("multipole_dev", C.c_void_p),
                ("owned_m2l_pairs", C.c_uint64), ("owned_p2p_body_pairs", C.c_uint64)]


class _GmresConfig(C.Structure):
    _fields_ = [("rtol", C.c_double), ("restart", C.c_int), ("max_iterations", C.c_int),
                ("precondition", C.c_int)]


class _GmresReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("breakdown", C.c_int),
                ("rhs_norm", C.c_double), ("final_residual", C.c_double), ("seconds", C.c_double),
                ("matvec_seconds", C.c_double), ("seconds_history", C.c_void_p),
                ("matvec_seconds_history", C.c_void_p), ("history_cap", C.c_int)]


class CorrectionRules(C.Structure):
    """hfmm_correction_rules (include/hfmm_cuda.h): the inputs of the correction builders"""
    _fields_ = [("basis_count", C.c_int), ("mode", C.c_int), ("n_patches", C.c_uint64),
                ("nodes", C.c_void_p), ("sample_ref", C.c_void_p), ("far_weight", C.c_void_p),
                ("near_patch_distance", C.c_double), ("near_npts", C.c_int),
                ("near_pts", C.c_void_p), ("near_basis", C.c_void_p), ("self_npts", C.c_void_p),
                ("self_pts", C.c_void_p), ("self_basis", C.c_void_p)]


def make_correction_rules(patches, tables, mode=2, near_patch_distance=-1.0):
    """patches: (n_patches, 6, 3); tables: dict with sample_ref (ni, 2), far_weight (ni,), near_pts
    (q, 3), near_basis (q, ni), self_npts (ni,), self_pts (sum, 3), self_basis (sum, ni) — the
    reference's geometry.cpp rules.  Returns (struct, keep-alive list)."""
    f8 = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    keep = [f8(patches), f8(tables["sample_ref"]), f8(tables["far_weight"]), f8(tables["near_pts"]),
            f8(tables["near_basis"]), np.ascontiguousarray(tables["self_npts"], dtype=np.int32),
            f8(tables["self_pts"]), f8(tables["self_basis"])]
    ptr = lambda a: a.ctypes.data_as(C.c_void_p) if a.size else None
    ni = int(keep[2].shape[0])
    r = CorrectionRules(ni, int(mode), int(keep[0].shape[0]), ptr(keep[0]), ptr(keep[1]), ptr(keep[2]),
                        float(near_patch_distance), int(keep[3].shape[0]), ptr(keep[3]), ptr(keep[4]),
                        ptr(keep[5]), ptr(keep[6]), ptr(keep[7]))
    return r, keep


ALLTOALLV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p, C.POINTER(C.c_uint64))
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int)


class _HostTransport(C.Structure):
    """hfmm_host_transport (include/hfmm_cuda.h)"""
    _fields_ = [("user", C.c_void_p), ("alltoallv", ALLTOALLV_FN), ("allreduce_sum", ALLREDUCE_FN)]


def library_path() -> str:
    return _SO


def build_library(force: bool = False) -> str:
    """compile csrc/ for sm_100a in-tree (nvcc cross-compiles without a GPU)"""
    if force or not os.path.exists(_SO):
        subprocess.check_call(["make", "-C", os.path.join(_HERE, "csrc"), "-j8"],
                              stdout=subprocess.DEVNULL)
    return _SO


_lib = None


def load_library():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise FileNotFoundError(
                f"{_SO} is missing: build it with `make -C paper_1803_09948_b200/csrc` "
                "(there is no CPU fallback)")
        lib = C.CDLL(_SO)
        lib.hfmm_cuda_last_error.restype = C.c_char_p
        lib.hfmm_cuda_version.restype = C.c_char_p
        _lib = lib
    return _lib


_dp = C.POINTER(C.c_double)


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


class HfmmCuda:
    """One FMM operator on one GPU (mirror of build_tree + dual_tree_traversal + execute_plan)."""

    def __init__(self, k: float, order: int, ncrit: int = 64, theta: float = 0.4,
                 kd_max: float = 1.0, leaf_cap: float = -1.0, grain: int | None = None,
                 device: int = 0, flags: int = 0, wave_i: float = 0.0):
        self.lib = load_library()
        if np.iscomplexobj(k):        # k = k_r + i k_i (attenuation), the reference's WaveNumber
            k, wave_i = float(np.real(k)), float(np.imag(k))
        cfg = _Config(float(k), float(wave_i), int(order), int(ncrit),
                      int(grain if grain is not None else ncrit), float(theta), float(kd_max),
                      float(leaf_cap), int(device), int(flags))
        self.h = C.c_void_p()
        rc = self.lib.hfmm_cuda_create(C.byref(self.h), C.byref(cfg))
        if rc:
            raise HfmmError(rc, self.lib.hfmm_cuda_last_error(None).decode())
        self.order = order
        self.n = 0
        self.partitioned = False

    def _check(self, rc):
        if rc:
            raise HfmmError(rc, self.lib.hfmm_cuda_last_error(self.h).decode())

    def set_points(self, xyz):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        if xyz.ndim != 2 or xyz.shape[1] != 3:
            raise ValueError("xyz must be (n, 3)")
        self._check(self.lib.hfmm_cuda_set_points(self.h, xyz.ctypes.data_as(_dp),
                                                  C.c_size_t(xyz.shape[0])))
        self.n = xyz.shape[0]

    def matvec(self, q):
        q = _c128(q)
        if q.shape != (self.n,):
            raise ValueError("charge vector length mismatch")
        out = np.empty(self.n, dtype=np.complex128)
        self._check(self.lib.hfmm_cuda_matvec(self.h, q.ctypes.data_as(_dp), out.ctypes.data_as(_dp)))
        return out

    def matvec_into(self, q_ptr: int, out_ptr: int):
        """host buffers by address (pinned memory from the caller), no numpy allocation"""
        self._check(self.lib.hfmm_cuda_matvec(self.h, C.c_void_p(q_ptr), C.c_void_p(out_ptr)))

    def matvec_device(self, q_dev_ptr: int, out_dev_ptr: int):
        self._check(self.lib.hfmm_cuda_matvec_device(self.h, C.c_void_p(q_dev_ptr),
                                                     C.c_void_p(out_dev_ptr)))

    def sync(self):
        self._check(self.lib.hfmm_cuda_sync(self.h))

    # ---- multi-GPU (Morton partition; see paper_1803_09948_b200/distributed.py)
    def set_partition(self, rank: int, nranks: int):
        self._check(self.lib.hfmm_cuda_set_partition(self.h, int(rank), int(nranks)))
        self.partitioned = True

    def set_partition_alpha(self, alpha: float):
        """Morton cuts balanced by the reference's w = l + alpha r (alpha < 0: default cost model)"""
        self._check(self.lib.hfmm_cuda_set_partition_alpha(self.h, C.c_double(alpha)))

    def measure_weights(self):
        """(local, remote) work estimates per body, caller order (reference measure_weights)"""
        local, remote = np.zeros(self.n), np.zeros(self.n)
        self._check(self.lib.hfmm_cuda_measure_weights(self.h, local.ctypes.data_as(_dp), remote.ctypes.data_as(_dp)))
        return local, remote

    def exchange_masks(self):
        """(far_mask, near_mask, cell_rank) per cell: which ranks need a cell's multipole / a leaf's
        bodies (locally essential trees), and who owns it"""
        nc = self.stats()["n_cells"]
        far, near = np.zeros(nc, dtype=np.uint64), np.zeros(nc, dtype=np.uint64)
        rank = np.zeros(nc, dtype=np.int32)
        self._check(self.lib.hfmm_cuda_get_exchange_masks(self.h, far.ctypes.data_as(C.c_void_p),
                                                          near.ctypes.data_as(C.c_void_p),
                                                          rank.ctypes.data_as(C.c_void_p)))
        return far, near, rank

    def partition(self) -> Partition:
        p = Partition()
        self._check(self.lib.hfmm_cuda_get_partition(self.h, C.byref(p)))
        return p

    def dist_upward(self, q_morton_dev_ptr: int):
        self._check(self.lib.hfmm_cuda_dist_upward(self.h, C.c_void_p(q_morton_dev_ptr)))

    def dist_downward(self, out_morton_dev_ptr: int):
        self._check(self.lib.hfmm_cuda_dist_downward(self.h, C.c_void_p(out_morton_dev_ptr)))

    def timer_record(self, slot: int):
        self._check(self.lib.hfmm_cuda_timer_record(self.h, int(slot)))

    def timer_elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_double()
        self._check(self.lib.hfmm_cuda_timer_elapsed_ms(self.h, int(a), int(b), C.byref(ms)))
        return ms.value

    def flush_l2(self):
        self._check(self.lib.hfmm_cuda_flush_l2(self.h))

    def fp32_peak_tflops(self) -> float:
        v = C.c_double()
        self._check(self.lib.hfmm_cuda_fp32_peak_tflops(self.h, C.byref(v)))
        return v.value

    def stats(self) -> dict:
        s = Stats()
        self._check(self.lib.hfmm_cuda_get_stats(self.h, C.byref(s)))
        return s.as_dict()

    def cells(self):
        nc = self.stats()["n_cells"]
        out = np.zeros((nc, 8), dtype=np.uint32)
        self._check(self.lib.hfmm_cuda_get_cells(self.h, out.ctypes.data_as(C.c_void_p), C.c_size_t(nc)))
        return out

    def body_order(self):
        out = np.zeros(self.n, dtype=np.uint32)
        self._check(self.lib.hfmm_cuda_get_body_order(self.h, out.ctypes.data_as(C.c_void_p)))
        return out

    def pairs(self, which: int):
        cnt = C.c_uint64()
        self._check(self.lib.hfmm_cuda_get_pairs(self.h, which, None, C.byref(cnt)))
        out = np.zeros((cnt.value, 2), dtype=np.uint32)
        if cnt.value:
            self._check(self.lib.hfmm_cuda_get_pairs(self.h, which, out.ctypes.data_as(C.c_void_p),
                                                     C.byref(cnt)))
        return out

    def expansions(self, which: int):
        nc = self.stats()["n_cells"]
        out = np.zeros((nc, (self.order + 1) ** 2), dtype=np.complex128)
        self._check(self.lib.hfmm_cuda_get_expansions(self.h, which, out.ctypes.data_as(_dp)))
        return out

    def set_corrections(self, ni, far_weight=None, patch_block=None, near_offset=None,
                        near_source=None, near_delta=None, block_lu=None, block_piv=None):
        keep = []

        def ptr(a, dt):
            if a is None or len(a) == 0:
                return None
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a.ctypes.data_as(C.c_void_p)

        self._check(self.lib.hfmm_cuda_set_corrections(
            self.h, int(ni), ptr(far_weight, np.float64), ptr(patch_block, np.complex128),
            ptr(near_offset, np.uint32), ptr(near_source, np.uint32), ptr(near_delta, np.complex128),
            ptr(block_lu, np.complex128), ptr(block_piv, np.int32)))

    @staticmethod
    def _report(rep, res, sec, mv):
        it = rep.iterations
        return dict(iterations=it, converged=bool(rep.converged), breakdown=bool(rep.breakdown),
                    rhs_norm=rep.rhs_norm, final_residual=rep.final_residual, seconds=rep.seconds,
                    matvec_seconds=rep.matvec_seconds, residuals=res[:it].copy(),
                    seconds_history=sec[:it].copy(), matvec_seconds_history=mv[:it].copy())

    def gmres(self, rhs, rtol=1e-4, restart=30, max_iterations=500, precondition=True):
        rhs = _c128(rhs)
        if rhs.shape != (self.n,):
            raise ValueError("right-hand side length mismatch")
        x = np.zeros(self.n, dtype=np.complex128)
        cfg = _GmresConfig(rtol, restart, max_iterations, int(precondition))
        cap = max(int(max_iterations), 0) + 1
        res, sec, mv = np.zeros(cap), np.zeros(cap), np.zeros(cap)
        rep = _GmresReport(seconds_history=sec.ctypes.data, matvec_seconds_history=mv.ctypes.data, history_cap=cap)
        self._check(self.lib.hfmm_cuda_gmres(self.h, rhs.ctypes.data_as(_dp), x.ctypes.data_as(_dp),
                                             C.byref(cfg), C.byref(rep), res.ctypes.data_as(_dp),
                                             len(res)))
        return x, self._report(rep, res, sec, mv)

    def assemble_rhs(self, direction=(0.0, 0.0, 1.0), amplitude=1.0):
        """plane-wave right-hand side A exp(i k d.x) over the points of set_points (reference assemble_rhs)"""
        d = np.ascontiguousarray(direction, dtype=np.float64)
        if d.shape != (3,):
            raise ValueError("direction must have three components")
        a = np.array([np.real(amplitude), np.imag(amplitude)], dtype=np.float64)
        out = np.zeros(self.n, dtype=np.complex128)
        self._check(self.lib.hfmm_cuda_assemble_rhs(self.h, d.ctypes.data_as(_dp), a.ctypes.data_as(_dp),
                                                    out.ctypes.data_as(_dp)))
        return out

    def set_patch_diameters(self, diameters):
        d = np.ascontiguousarray(diameters, dtype=np.float64)
        self._check(self.lib.hfmm_cuda_set_patch_diameters(self.h, d.ctypes.data_as(_dp), C.c_size_t(d.shape[0])))

    # ---- the library's own data plane (csrc/comm.cu)
    @staticmethod
    def nccl_unique_id() -> bytes:
        """128 bytes from ncclGetUniqueId (rank 0 creates, the application's bootstrap distributes)"""
        buf = C.create_string_buffer(128)
        lib = load_library()
        rc = lib.hfmm_cuda_nccl_unique_id(buf)
        if rc:
            raise HfmmError(rc, lib.hfmm_cuda_last_error(None).decode())
        return buf.raw

    def comm_init_nccl(self, unique_id: bytes):
        """ncclCommInitRank over (rank, nranks) of set_partition; collective"""
        if len(unique_id) != 128:
            raise ValueError("an NCCL unique id is 128 bytes")
        self._check(self.lib.hfmm_cuda_comm_init_nccl(self.h, C.c_char_p(unique_id)))

    def comm_init_host(self, alltoallv, allreduce_sum):
        """Host-staged transport.  alltoallv(send: np.uint8[...], send_bytes: np.uint64[R], recv: np.uint8[...],
        recv_bytes: np.uint64[R]) and allreduce_sum(values: np.float64[...]) work in place on host arrays;
        an exception inside either aborts the running call with a device error."""
        nranks = int(self.partition().nranks) if self.n else None
        failure = self._transport_failure = []

        def a2a(_u, send, sbytes, recv, rbytes):
            if failure:
                return 1
            try:
                R = nranks if nranks is not None else int(self.partition().nranks)
                sb = np.ctypeslib.as_array(sbytes, shape=(R,)).copy()
                rb = np.ctypeslib.as_array(rbytes, shape=(R,)).copy()
                s_arr = np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_uint8)), shape=(max(int(sb.sum()), 1),))
                r_arr = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_uint8)), shape=(max(int(rb.sum()), 1),))
                alltoallv(s_arr[:int(sb.sum())], sb, r_arr[:int(rb.sum())], rb)
                return 0
            except BaseException as e:      # a callback must not unwind through C
                failure.append(e)
                return 1

        def red(_u, p, c):
            if failure:
                return 1
            try:
                allreduce_sum(np.ctypeslib.as_array(p, shape=(c,)))
                return 0
            except BaseException as e:
                failure.append(e)
                return 1

        self._transport = _HostTransport(None, ALLTOALLV_FN(a2a), ALLREDUCE_FN(red))   # kept alive with the handle
        self._check(self.lib.hfmm_cuda_comm_init_host(self.h, C.byref(self._transport)))

    def _raise_transport_failure(self):
        f = getattr(self, "_transport_failure", None)
        if f:
            e = f[0]
            f.clear()
            raise e

    def dist_matvec(self, q_owned_dev_ptr: int, out_owned_dev_ptr: int):
        rc = self.lib.hfmm_cuda_dist_matvec(self.h, C.c_void_p(q_owned_dev_ptr), C.c_void_p(out_owned_dev_ptr))
        self._raise_transport_failure()
        self._check(rc)

    def exchange_volume(self):
        """(halo charge bytes, remote multipole bytes) this rank receives per matvec"""
        a, b = C.c_uint64(), C.c_uint64()
        self._check(self.lib.hfmm_cuda_get_exchange_volume(self.h, C.byref(a), C.byref(b)))
        return int(a.value), int(b.value)

    def dist_solve(self, rhs_owned, rtol=1e-4, restart=30, max_iterations=500, precondition=True):
        """GMRES over Morton-sharded vectors through the handle's communicator.  rhs_owned: the owned
        Morton slice (complex128); returns the same slice of the solution and the report."""
        rhs = _c128(rhs_owned)
        if rhs.shape != (int(self.partition().body_count),):
            raise ValueError("rhs_owned must hold exactly the owned Morton slice")
        x = np.zeros(rhs.shape[0], dtype=np.complex128)
        cfg = _GmresConfig(rtol, restart, max_iterations, int(precondition))
        cap = max(int(max_iterations), 0) + 1
        res, sec, mv = np.zeros(cap), np.zeros(cap), np.zeros(cap)
        rep = _GmresReport(seconds_history=sec.ctypes.data, matvec_seconds_history=mv.ctypes.data, history_cap=cap)
        vp = lambda a: a.ctypes.data_as(_dp) if a.size else None
        rc = self.lib.hfmm_cuda_dist_solve(self.h, vp(rhs), vp(x), C.byref(cfg), C.byref(rep),
                                           res.ctypes.data_as(_dp), len(res))
        self._raise_transport_failure()
        self._check(rc)
        return x, self._report(rep, res, sec, mv)

    def evaluate_targets(self, targets, q):
        """potentials of the operator's points (strengths q) at other points: fmm_evaluate with distinct
        target and source trees (traversal.hpp:59-67)"""
        t = np.ascontiguousarray(targets, dtype=np.float64)
        q = _c128(q)
        if t.ndim != 2 or t.shape[1] != 3 or q.shape != (self.n,):
            raise ValueError("targets must be (m, 3), q must hold one strength per source")
        out = np.zeros(t.shape[0], dtype=np.complex128)
        self.lib.hfmm_cuda_evaluate_targets.argtypes = [C.c_void_p, _dp, C.c_size_t, _dp, _dp]
        self._check(self.lib.hfmm_cuda_evaluate_targets(self.h, t.ctypes.data_as(_dp), t.shape[0],
                                                        q.ctypes.data_as(_dp), out.ctypes.data_as(_dp)))
        return out

    def solve_residual(self):
        """b - Z u of the last gmres / dist_solve (complex128; all unknowns or the owned Morton slice)"""
        n = int(self.partition().body_count) if self.partitioned else self.n
        out = np.zeros(n, dtype=np.complex128)
        self.lib.hfmm_cuda_get_solve_residual.argtypes = [C.c_void_p, _dp, C.c_size_t]
        self._check(self.lib.hfmm_cuda_get_solve_residual(self.h, out.ctypes.data_as(_dp) if n else None, n))
        return out

    def build_corrections(self, patches, tables, mode=2, near_patch_distance=-1.0, fetch=True):
        """Correction arrays built on the device from the patches and the reference's rule tables
        (see make_correction_rules) and installed as this operator's corrections."""
        r, keep = make_correction_rules(patches, tables, mode, near_patch_distance)
        nnz = C.c_uint64(0)
        self._check(self.lib.hfmm_cuda_build_corrections(self.h, C.byref(r), C.byref(nnz)))
        nnz = int(nnz.value)
        if not fetch:
            return nnz
        ni, npatch = r.basis_count, int(r.n_patches)
        n = ni * npatch
        pb = np.zeros(n * ni, dtype=np.complex128)
        lu = np.zeros(n * ni if mode else 0, dtype=np.complex128)
        piv = np.zeros(n if mode else 0, dtype=np.int32)
        off = np.zeros(n + 1, dtype=np.uint32)
        src = np.zeros(nnz, dtype=np.uint32)
        dl = np.zeros(nnz, dtype=np.complex128)
        vp = lambda a: a.ctypes.data_as(C.c_void_p) if a.size else None
        self._check(self.lib.hfmm_cuda_get_corrections(self.h, vp(pb), vp(lu), vp(piv), vp(off), vp(src), vp(dl)))
        return dict(patch_block=pb, block_lu=lu, block_piv=piv, near_offset=off, near_source=src, near_delta=dl)

    def evaluate_field(self, coeff, obs):
        coeff = _c128(coeff)
        obs = np.ascontiguousarray(obs, dtype=np.float64)
        if coeff.shape != (self.n,) or obs.ndim != 2 or obs.shape[1] != 3:
            raise ValueError("coeff must have one entry per unknown and obs must be (nobs, 3)")
        out = np.zeros(obs.shape[0], dtype=np.complex128)
        self._check(self.lib.hfmm_cuda_evaluate_field(self.h, coeff.ctypes.data_as(_dp),
                                                      obs.ctypes.data_as(_dp),
                                                      C.c_size_t(obs.shape[0]), out.ctypes.data_as(_dp)))
        return out

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            self.lib.hfmm_cuda_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- host-only debug helpers (no device needed) used by the CPU-side tests -------------------
def update_alpha(alphas, runtimes, alpha_max: float = 2.0) -> float:
    """next alpha of the repartitioning loop (reference update_alpha, partition.cpp:175-227)"""
    lib = load_library()
    a = np.ascontiguousarray(alphas, dtype=np.float64)
    r = np.ascontiguousarray(runtimes, dtype=np.float64)
    out = C.c_double()
    rc = lib.hfmm_partition_update_alpha(a.ctypes.data_as(_dp), r.ctypes.data_as(_dp), len(a),
                                         C.c_double(alpha_max), C.byref(out))
    if rc:
        raise HfmmError(rc, "update_alpha: empty history or non-positive alpha_max")
    return out.value


def debug_compose_translation(order, k, t, kind, s_src=1.0, s_dst=1.0):
    lib = load_library()
    dim = (order + 1) ** 2
    out = np.zeros((dim, dim), dtype=np.complex128)
    t = np.ascontiguousarray(t, dtype=np.float64)
    rc = lib.hfmm_debug_compose_translation_ck(int(order), C.c_double(np.real(k)), C.c_double(np.imag(k)),
                                               t.ctypes.data_as(_dp), int(kind), C.c_double(s_src),
                                               C.c_double(s_dst), out.ctypes.data_as(_dp))
    if rc:
        raise HfmmError(rc, lib.hfmm_cuda_last_error(None).decode())
    return out


def debug_partition(xyz, ncrit, leaf_cap, k, theta, kd_max, nranks, n_cells=None):
    """(first[r], count[r], cell_rank, lcut) of the Morton partition, computed on the host"""
    lib = load_library()
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    first = np.zeros(nranks, dtype=np.uint32)
    count = np.zeros(nranks, dtype=np.uint32)
    cells = np.full(n_cells or 0, -2, dtype=np.int32)
    lcut = C.c_int32()
    vp = lambda a: a.ctypes.data_as(C.c_void_p) if a.size else None
    rc = lib.hfmm_debug_partition(xyz.ctypes.data_as(_dp), C.c_size_t(xyz.shape[0]), int(ncrit),
                                  C.c_double(leaf_cap), C.c_double(k), C.c_double(theta),
                                  C.c_double(kd_max), int(nranks), vp(first), vp(count), vp(cells),
                                  C.c_size_t(cells.size), C.byref(lcut))
    if rc:
        raise HfmmError(rc, lib.hfmm_cuda_last_error(None).decode())
    return first, count, cells, lcut.value


def debug_host_tree(xyz, ncrit, leaf_cap, k, theta, kd_max):
    lib = load_library()
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    n = xyz.shape[0]
    counts = (C.c_uint64 * 5)()
    args = lambda *extra: lib.hfmm_debug_host_tree(
        xyz.ctypes.data_as(_dp), C.c_size_t(n), int(ncrit), C.c_double(leaf_cap), C.c_double(k),
        C.c_double(theta), C.c_double(kd_max), counts, *extra)
    rc = args(None, C.c_size_t(0), None, None, None, C.c_size_t(0))
    if rc:
        raise HfmmError(rc, lib.hfmm_cuda_last_error(None).decode())
    nc, nl, nm2l, np2p, maxl = [int(v) for v in counts]
    cells = np.zeros((nc, 8), dtype=np.uint32)
    order = np.zeros(n, dtype=np.uint32)
    cap = max(nm2l, np2p, 1)
    m2l = np.zeros((cap, 2), dtype=np.uint32)
    p2p = np.zeros((cap, 2), dtype=np.uint32)
    vp = lambda a: a.ctypes.data_as(C.c_void_p)
    rc = args(vp(cells), C.c_size_t(nc), vp(order), vp(m2l), vp(p2p), C.c_size_t(cap))
    if rc:
        raise HfmmError(rc, lib.hfmm_cuda_last_error(None).decode())
    return dict(cells=cells, order=order, m2l=m2l[:nm2l], p2p=p2p[:np2p], n_leaves=nl, max_level=maxl)
