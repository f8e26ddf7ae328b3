"""GPU: the BIE operator tail, block-Jacobi preconditioner, device GMRES and exterior field
evaluation against the reference's fixtures (tests/golden/solver.npz) and, where the compiled
reference travelled to the box, against a live mid-size system."""
import os

import numpy as np
import pytest

from checkers import have_ref, rel_l2
from paper_1803_09948_b200 import HfmmCuda, HfmmError
from paper_1803_09948_b200.api import HFMM_FLAG_DETERMINISTIC
from paper_1803_09948_b200.workloads import icosphere_patches, sphere_points, charges

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "solver.npz"))


def _bie_operator(g, prefix="bie_", **kw):
    k, order = float(g[prefix + "k"]), int(g[prefix + "order"])
    op = HfmmCuda(k=k, order=order, ncrit=16, theta=0.4, kd_max=1.0, leaf_cap=-1.0, **kw)
    op.set_points(g[prefix + "xyz"])
    op.set_corrections(int(g[prefix + "ni"]), far_weight=g[prefix + "far_weight"],
                       patch_block=g[prefix + "patch_block"], near_offset=g[prefix + "near_offset"],
                       near_source=g[prefix + "near_source"], near_delta=g[prefix + "near_delta"],
                       block_lu=g[prefix + "block_lu"], block_piv=g[prefix + "block_piv"])
    return op


def test_apply_operator_matches_reference_fixture():
    # reference solver.cpp:314-359: FMM(x * far_weight) + blockdiag + CSR; FP32 tolerance 1e-5
    op = _bie_operator(G)
    assert rel_l2(op.matvec(G["bie_x"]), G["bie_y"]) < 1e-5


@pytest.mark.parametrize("flags", [0, 1 << 3], ids=["atomics", "deterministic"])
def test_gmres_iteration_parity_with_reference_fixture(flags):
    # north star: GMRES reaches 1e-4 in the reference's iteration count +-1 (in the default mode and
    # with HFMM_FLAG_DETERMINISTIC = 1 << 3, the reference's ordered accumulation)
    op = _bie_operator(G, flags=flags)
    for precondition, it_ref, sol_ref in ((True, int(G["bie_iterations"]), G["bie_sol"]),
                                          (False, int(G["bie_iterations_noprec"]), G["bie_sol_noprec"])):
        x, rep = op.gmres(G["bie_rhs"], rtol=1e-4, restart=30, max_iterations=200,
                          precondition=precondition)
        assert rep["converged"] and rep["final_residual"] <= 1.05e-4
        assert abs(rep["iterations"] - it_ref) <= 1, (rep["iterations"], it_ref)
        assert rel_l2(x, sol_ref) < 2e-3          # both are 1e-4-residual solutions
        assert np.all(np.diff(rep["residuals"]) <= 1e-12)   # GMRES residual estimates never grow


def test_gmres_dense_fixture_and_report():
    # plain (uncorrected) FMM operator on a point cloud: converges, true residual agrees
    n, k = 3000, 2.0
    xyz = sphere_points(n, 8)
    op = HfmmCuda(k=k, order=8, ncrit=32)
    op.set_points(xyz)
    b = charges(n, 8)
    # shifted operator I*c + A is what converges quickly; emulate with a diagonal block correction
    blocks = np.full(n, 2000.0 + 0j)   # row sums of the kernel matrix are O(n / 4 pi) ~ 240
    op.set_corrections(1, patch_block=blocks)
    x, rep = op.gmres(b, rtol=1e-5, restart=20, max_iterations=200, precondition=False)
    assert rep["converged"] and rep["iterations"] < 200
    r = b - op.matvec(x)
    assert abs(np.linalg.norm(r) / np.linalg.norm(b) - rep["final_residual"]) < 2e-6
    assert rep["rhs_norm"] == pytest.approx(np.linalg.norm(b), rel=1e-12)
    with pytest.raises(HfmmError) as e:
        op.gmres(b, rtol=2.0)
    assert e.value.kind == "config_error"       # gmres.cpp:25-31
    x0, rep0 = op.gmres(np.zeros(n), rtol=1e-4)
    assert rep0["converged"] and rep0["iterations"] == 0 and np.abs(x0).max() == 0


def test_scattered_field_matches_reference_fixture():
    op = _bie_operator(G)
    f = op.evaluate_field(G["bie_sol"], G["bie_obs"])
    assert rel_l2(f, G["bie_scattered"]) < 1e-5


def test_assemble_rhs_matches_reference_fixture():
    # reference solver.cpp:302-312, evaluated in FP64 on the device from the FP64 points
    op = _bie_operator(G)
    rhs = op.assemble_rhs((0.0, 0.0, 1.0))
    assert np.abs(rhs - G["bie_rhs"]).max() < 1e-13
    k = float(G["bie_k"])
    d = np.array([1.0, 2.0, -2.0]) / 3.0
    amp = 0.5 - 1.5j
    assert np.abs(op.assemble_rhs(d, amp) - amp * np.exp(1j * k * (G["bie_xyz"] @ d))).max() < 1e-13
    with pytest.raises(HfmmError) as e:          # "incident direction must be unit length"
        op.assemble_rhs((0.0, 0.0, 1.0001))
    assert e.value.kind == "config_error"
    # complex wavenumber: exp(i (kr + i ki) d.x)
    opc = HfmmCuda(k=2.0 + 0.3j, order=6, ncrit=16)
    opc.set_points(G["bie_xyz"])
    assert np.abs(opc.assemble_rhs(d) - np.exp(1j * (2.0 + 0.3j) * (G["bie_xyz"] @ d))).max() < 1e-13


def test_scattered_field_refuses_points_on_the_surface():
    # reference solver.cpp:399-413: singular_error within 0.1 x patch diameter of a sample
    op = _bie_operator(G)
    patches = G["bie_patches"]
    diam = 2 * np.linalg.norm(patches - patches.mean(axis=1, keepdims=True), axis=2).max(axis=1)
    far = op.evaluate_field(G["bie_sol"], G["bie_obs"])       # no geometry known: nothing to test against
    op.set_patch_diameters(diam)
    assert np.array_equal(op.evaluate_field(G["bie_sol"], G["bie_obs"]), far)
    x0 = G["bie_xyz"][17]
    near = x0 * (1.0 + 0.05 * diam[17 // 3] / np.linalg.norm(x0))
    with pytest.raises(HfmmError) as e:
        op.evaluate_field(G["bie_sol"], np.vstack([G["bie_obs"], near]))
    assert e.value.kind == "singular_error"
    ok = x0 * (1.0 + 0.5 * diam[17 // 3] / np.linalg.norm(x0))
    assert np.isfinite(op.evaluate_field(G["bie_sol"], ok[None, :])).all()
    # the device builders know the patches: the test is armed without set_patch_diameters
    tables = {key: G["bie_rule_" + key] for key in ("sample_ref", "far_weight", "near_pts", "near_basis",
                                                    "self_npts", "self_pts", "self_basis")}
    op2 = HfmmCuda(k=float(G["bie_k"]), order=int(G["bie_order"]), ncrit=16)
    op2.set_points(G["bie_xyz"])
    op2.build_corrections(patches, tables, mode=2, fetch=False)
    with pytest.raises(HfmmError) as e:
        op2.evaluate_field(G["bie_sol"], near[None, :])
    assert e.value.kind == "singular_error"
    # far away, FP64 distances: a large offset of the whole geometry leaves the field unchanged to FP32 rounding
    shift = np.array([300.0, -200.0, 100.0])
    op3 = HfmmCuda(k=float(G["bie_k"]), order=int(G["bie_order"]), ncrit=16)
    op3.set_points(G["bie_xyz"] + shift)
    op3.set_corrections(int(G["bie_ni"]), far_weight=G["bie_far_weight"])
    assert rel_l2(op3.evaluate_field(G["bie_sol"], G["bie_obs"] + shift), G["bie_scattered"]) < 1e-5


def test_solve_report_histories():
    # SolveReport::seconds / matvec_seconds, one entry per iteration (solver.hpp:106-116)
    op = _bie_operator(G)
    x, rep = op.gmres(G["bie_rhs"], rtol=1e-4, restart=30, max_iterations=200, precondition=True)
    it = rep["iterations"]
    assert len(rep["seconds_history"]) == it == len(rep["matvec_seconds_history"]) == len(rep["residuals"])
    assert np.all(np.diff(rep["seconds_history"]) > 0) and rep["seconds_history"][-1] <= rep["seconds"]
    assert np.all(rep["matvec_seconds_history"] > 0)
    # restarts add one operator application to the iteration that follows them; the exit residual one more
    assert rep["matvec_seconds_history"].sum() <= rep["matvec_seconds"] + 1e-12


@pytest.mark.skipif(not have_ref(), reason="compiled reference not on this box")
@pytest.mark.parametrize("direction", [(0.36, 0.48, 0.8), (0.0, 0.0, 1.0)], ids=["generic-wave", "wave-along-a-symmetry-axis"])
def test_midsize_system_against_oracle_gmres(oracle, direction):
    """320 curved triangles (960 unknowns): system built by the reference, GMRES run (a) on the device and
    (b) by the oracle's restatement of gmres.cpp over the oracle's FP64 FMM matvec.

    North star: the same iteration count +-1.  That holds — restarted or not — for a GENERIC right-hand
    side.  With the wave along a symmetry axis of the mesh (the icosphere's five-fold axis here, the polar
    axis of the reference's lat-long sphere in tests/test_gpu_dropin.py) the all-FP64 iteration never leaves
    the invariant subspace of that symmetry and converges early; ANY rounding at FP32 level breaks the
    symmetry, the Krylov vectors leak into the other sectors and have to be resolved there too.  The
    reference's own FP32 near-field mode (kernel::Precision::f32) does exactly the same
    (tests/test_oracle_vs_reference.py::test_symmetric_problem_iteration_count_is_not_robust_in_fp32), so
    for that degenerate case the device count is pinned against the same operator under the FP64 Krylov
    loop, and only loosely against the all-FP64 run."""
    from checkers import Ref

    k, order = 3.0, 10
    sysr = Ref().bie(icosphere_patches(2), 1, k, mode=2, use_tree=False)
    xyz, fw = sysr.samples()
    corr = sysr.corrections()
    rhs = sysr.rhs(direction)
    # ordered accumulation: "the same operator" below must be a function, not a run-to-run variable
    op = HfmmCuda(k=k, order=order, ncrit=16, flags=HFMM_FLAG_DETERMINISTIC)
    op.set_points(xyz)
    op.set_corrections(sysr.ni, far_weight=fw, **corr)
    assert np.abs(op.assemble_rhs(direction) - rhs).max() < 1e-13
    f = oracle.fmm(xyz, k, order, ncrit=16, leaf_cap=1.0 / k, theta=0.4, kd_max=1.0)

    def minv(u):
        return oracle.block_lu_solve(sysr.ni, corr["block_lu"], corr["block_piv"], u)

    def z_cpu(u):       # FP64 operator
        v = minv(u)
        return oracle.apply_corrections(sysr.ni, corr["patch_block"], corr["near_offset"],
                                        corr["near_source"], corr["near_delta"], v, f.matvec(v * fw))

    def z_gpu(u):       # the device operator (FP32 arithmetic) under the oracle's FP64 Krylov loop
        return op.matvec(minv(u))

    generic = direction[2] != 1.0
    # (1) without restarts
    x_gpu, rep = op.gmres(rhs, rtol=1e-4, restart=300, max_iterations=300)
    u, rep_o = oracle.gmres(z_cpu, rhs, rtol=1e-4, restart=300, max_iterations=300)
    assert rep["converged"] and rep_o["converged"]
    assert abs(rep["iterations"] - rep_o["iterations"]) <= 1, (rep["iterations"], rep_o["iterations"])
    assert rel_l2(x_gpu, minv(u)) < 2e-3
    # (2) restart 30
    x30, rep30 = op.gmres(rhs, rtol=1e-4, restart=30, max_iterations=300)
    _, rep30_same_op = oracle.gmres(z_gpu, rhs, rtol=1e-4, restart=30, max_iterations=300)
    _, rep30_cpu = oracle.gmres(z_cpu, rhs, rtol=1e-4, restart=30, max_iterations=300)
    assert rep30["converged"]
    assert abs(rep30["iterations"] - rep30_same_op["iterations"]) <= 1
    if generic:
        # the comparison the north star asks for ("in FP32 complex"): the REFERENCE in its own single-precision
        # near-field mode (kernel::Precision::f32, kernel.hpp:43-55; everything else FP64) under the same
        # FP64 Krylov loop.  Measured for five generic directions (scripts/diag_midsize.py and the reference
        # against itself): all-FP64 57 every time; reference f32 near field 58-59; FP64 operator applied to
        # the FP32-rounded operand 58-59; FP64 operator + 1e-7 noise 58-59; device 58-59.  The 57 is the
        # outlier of exact arithmetic — the residual of iteration 57 sits 6 % under the threshold — so the
        # device is pinned to +-1 of the reference's FP32 mode and to +2 of the all-FP64 run.
        fr = Ref().fmm(xyz, k, order, ncrit=16, leaf_cap=1.0 / k, theta=0.4, kd_max=1.0)

        def z_ref32(u):
            v = minv(u)
            return oracle.apply_corrections(sysr.ni, corr["patch_block"], corr["near_offset"],
                                            corr["near_source"], corr["near_delta"], v,
                                            fr.matvec(v * fw, f32_p2p=True))

        _, rep30_ref32 = oracle.gmres(z_ref32, rhs, rtol=1e-4, restart=30, max_iterations=300)
        assert abs(rep30["iterations"] - rep30_ref32["iterations"]) <= 1, \
            (rep30["iterations"], rep30_ref32["iterations"])
        assert rep30_ref32["iterations"] >= rep30_cpu["iterations"]
    assert abs(rep30["iterations"] - rep30_cpu["iterations"]) <= (2 if generic else 5), \
        (rep30["iterations"], rep30_cpu["iterations"])
    assert rel_l2(x30, x_gpu) < 2e-3


@pytest.mark.parametrize("ranks", [2, 3])
def test_sharded_gmres_matches_single_domain(ranks):
    """the library's sharded solver (hfmm_cuda_dist_solve: Morton-sharded Krylov vectors,
    device-side all-reduce of the inner products, locally-essential-tree exchanges inside the operator) takes
    the single-domain iteration and returns the same solution.  Ranks are host threads on one device joined
    by the host transport."""
    from paper_1803_09948_b200.distributed import emulate_gmres_on_one_device

    single = _bie_operator(G)
    order = single.body_order()
    ops = []
    for r in range(ranks):
        k, p = float(G["bie_k"]), int(G["bie_order"])
        op = HfmmCuda(k=k, order=p, ncrit=16, theta=0.4, kd_max=1.0, leaf_cap=-1.0)
        op.set_partition(r, ranks)
        op.set_points(G["bie_xyz"])
        op.set_corrections(int(G["bie_ni"]), far_weight=G["bie_far_weight"], patch_block=G["bie_patch_block"],
                           near_offset=G["bie_near_offset"], near_source=G["bie_near_source"],
                           near_delta=G["bie_near_delta"], block_lu=G["bie_block_lu"],
                           block_piv=G["bie_block_piv"])
        ops.append(op)
    assert sum(int(op.partition().body_count) for op in ops) == len(order)
    rhs_morton = np.asarray(G["bie_rhs"])[order]
    for precondition in (True, False):
        x1, rep1 = single.gmres(G["bie_rhs"], rtol=1e-4, restart=30, max_iterations=200,
                                precondition=precondition)
        res = emulate_gmres_on_one_device(ops, rhs_morton, rtol=1e-4, restart=30, max_iterations=200,
                                          precondition=precondition)
        x = np.concatenate([xr for xr, _ in res])
        reps = [rep for _, rep in res]
        assert all(rep["converged"] for rep in reps)
        assert len({rep["iterations"] for rep in reps}) == 1          # ranks stay in lock step
        assert abs(reps[0]["iterations"] - rep1["iterations"]) <= 1, (reps[0]["iterations"], rep1["iterations"])
        assert reps[0]["final_residual"] <= 1.05e-4
        assert rel_l2(x, x1[order]) < 2e-3
        np.testing.assert_allclose(reps[0]["residuals"][:5], rep1["residuals"][:5], rtol=1e-4)


def test_sharded_operator_over_nccl_world_of_one():
    """The NCCL transport of the library (dlopen of libnccl, ncclCommInitRank from a unique id, grouped
    send / receive, device-side all-reduce) with the one GPU this box has: world size 1 — every call on
    the multi-GPU code path is made, the peer loops are empty."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_1803_09948_b200.distributed import ShardedFmm

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dev = torch.device("cuda", 0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        single = _bie_operator(G)
        op = HfmmCuda(k=float(G["bie_k"]), order=int(G["bie_order"]), ncrit=16, theta=0.4, kd_max=1.0,
                      leaf_cap=-1.0)
        op.set_partition(0, 1)
        op.set_points(G["bie_xyz"])
        op.set_corrections(int(G["bie_ni"]), far_weight=G["bie_far_weight"], patch_block=G["bie_patch_block"],
                           near_offset=G["bie_near_offset"], near_source=G["bie_near_source"],
                           near_delta=G["bie_near_delta"], block_lu=G["bie_block_lu"],
                           block_piv=G["bie_block_piv"])
        sh = ShardedFmm(op, dist, 0, 1, dev, transport="nccl")
        order = op.body_order()
        assert sh.count == len(order) and sh.let_bytes == {"charges": 0, "multipoles": 0}
        x1, rep1 = single.gmres(G["bie_rhs"], rtol=1e-4, restart=30, max_iterations=200)
        x, rep = sh.gmres(np.asarray(G["bie_rhs"])[order], rtol=1e-4, restart=30, max_iterations=200)
        assert rep["converged"] and abs(rep["iterations"] - rep1["iterations"]) <= 1
        assert rel_l2(x, x1[order]) < 2e-3
        # the plain FMM product over the communicator against the single-handle FMM
        plain = HfmmCuda(k=float(G["bie_k"]), order=int(G["bie_order"]), ncrit=16, theta=0.4, kd_max=1.0,
                         leaf_cap=-1.0)
        plain.set_points(G["bie_xyz"])
        op2 = HfmmCuda(k=float(G["bie_k"]), order=int(G["bie_order"]), ncrit=16, theta=0.4, kd_max=1.0, leaf_cap=-1.0)
        op2.set_partition(0, 1)
        op2.set_points(G["bie_xyz"])
        sh2 = ShardedFmm(op2, dist, 0, 1, dev, transport="nccl")
        q = charges(len(order), 3)
        qm = q[order]
        q_local = torch.from_numpy(np.stack([qm.real, qm.imag], 1).astype(np.float32)).to(dev)
        y = sh2.matvec(q_local)
        op2.sync()
        y = y.cpu().numpy()
        assert rel_l2(y[:, 0] + 1j * y[:, 1], plain.matvec(q)[order]) < 2e-6
    finally:
        dist.destroy_process_group()


def _two_process_worker(rank, world, port, queue):
    """one rank of the two-process test: both ranks use cuda:0, they meet on the host only (gloo)"""
    import torch
    import torch.distributed as dist

    from paper_1803_09948_b200.distributed import ShardedFmm
    from paper_1803_09948_b200.workloads import plummer_points

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        out = {}
        # (a) plain FMM product on a clustered volume, locally-essential-tree exchange
        n, k, order = 30000, 6.0, 8
        xyz, q = plummer_points(n, 12, a=0.08), charges(n, 12)
        op = HfmmCuda(k=k, order=order, ncrit=48, theta=0.4)
        op.set_partition(rank, world)
        op.set_points(xyz)
        sh = ShardedFmm(op, dist, rank, world, dev, transport="host")
        morton = op.body_order()
        qm = q[morton][sh.first:sh.first + sh.count]
        q_local = torch.from_numpy(np.stack([qm.real, qm.imag], 1).astype(np.float32)).to(dev)
        for _ in range(2):              # twice: the exchange buffers are reused
            y = sh.matvec(q_local)
            op.sync()
        y = y.cpu().numpy()
        out["matvec"] = (sh.first, sh.count, y[:, 0] + 1j * y[:, 1], sh.let_bytes, sh.owned_m2l_pairs)
        # (b) the BIE system of the reference fixture: sharded GMRES with block-Jacobi and corrections
        bie = HfmmCuda(k=float(G["bie_k"]), order=int(G["bie_order"]), ncrit=16, theta=0.4, kd_max=1.0, leaf_cap=-1.0)
        bie.set_partition(rank, world)
        bie.set_points(G["bie_xyz"])
        bie.set_corrections(int(G["bie_ni"]), far_weight=G["bie_far_weight"], patch_block=G["bie_patch_block"],
                            near_offset=G["bie_near_offset"], near_source=G["bie_near_source"],
                            near_delta=G["bie_near_delta"], block_lu=G["bie_block_lu"], block_piv=G["bie_block_piv"])
        shb = ShardedFmm(bie, dist, rank, world, dev, transport="host")
        rhs = np.asarray(G["bie_rhs"])[bie.body_order()][shb.first:shb.first + shb.count]
        x, rep = shb.gmres(rhs, rtol=1e-4, restart=30, max_iterations=200, precondition=True)
        out["gmres"] = (shb.first, shb.count, x, rep["iterations"], rep["converged"], rep["final_residual"])
        # (c) the plain operator (no corrections): the solver's owned-slice path, pruned exchanges only
        xp, repp = sh.gmres(qm * 0 + 1.0, rtol=1e-2, restart=10, max_iterations=3, precondition=False)
        out["plain_solve"] = (repp["iterations"], float(np.abs(xp).sum()))
        queue.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_processes_share_one_gpu_through_the_host_transport():
    """Two RANK PROCESSES on cuda:0 (gloo, pinned host staging: they only ever meet on the host) run the
    real ShardedFmm.matvec and .gmres — the library's pack / exchange / unpack data plane and sharded
    solver — against the single-domain results (reference distributed_matvec, let.cpp:320-362)."""
    import socket

    import torch.multiprocessing as mp

    from paper_1803_09948_b200.workloads import plummer_points

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    procs = [ctx.Process(target=_two_process_worker, args=(r, 2, port, queue)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(queue.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert sorted(got) == [0, 1]
    # (a) against the single-domain matvec
    n, k, order = 30000, 6.0, 8
    xyz, q = plummer_points(n, 12, a=0.08), charges(n, 12)
    single = HfmmCuda(k=k, order=order, ncrit=48, theta=0.4)
    single.set_points(xyz)
    y1 = single.matvec(q)[single.body_order()]
    y = np.zeros(n, dtype=np.complex128)
    covered = 0
    for r in (0, 1):
        f, c, yr, let, pairs = got[r]["matvec"]
        y[f:f + c] = yr
        covered += c
        assert let["charges"] > 0 and let["multipoles"] > 0 and pairs > 0     # both ranks work, both receive a halo
        assert let["charges"] < 8 * n and let["multipoles"] < 0.8 * single.stats()["n_cells"] * 8 * (order + 1) ** 2
    assert covered == n and got[0]["matvec"][0] == 0 and got[1]["matvec"][0] == got[0]["matvec"][1]
    assert rel_l2(y, y1) < 3e-6
    # (b) against the single-domain solve
    op1 = _bie_operator(G)
    x1, rep1 = op1.gmres(G["bie_rhs"], rtol=1e-4, restart=30, max_iterations=200, precondition=True)
    x = np.concatenate([got[r]["gmres"][2] for r in (0, 1)])
    its = {got[r]["gmres"][3] for r in (0, 1)}
    assert len(its) == 1 and abs(its.pop() - rep1["iterations"]) <= 1       # the ranks stay in lock step
    assert all(got[r]["gmres"][4] and got[r]["gmres"][5] <= 1.05e-4 for r in (0, 1))
    assert rel_l2(x, x1[op1.body_order()]) < 2e-3
    assert got[0]["plain_solve"][0] == got[1]["plain_solve"][0] == 3


# ---- the correction builders on the device ---------------------------
def _tables(g, prefix):
    keys = ("sample_ref", "far_weight", "near_pts", "near_basis", "self_npts", "self_pts", "self_basis")
    return {k: g[prefix + k] for k in keys}


def _check_corrections(got, want, tol=2e-13):
    # lists, pivots: exact; values: FP64 with device exp / sin / cos (an ulp from glibc's)
    for key in ("near_offset", "near_source", "block_piv"):
        assert np.array_equal(got[key], want[key]), key
    for key in ("patch_block", "block_lu", "near_delta"):
        assert got[key].shape == want[key].shape, key
        if want[key].size:
            assert np.abs(got[key] - want[key]).max() <= tol * np.abs(want[key]).max(), key


@pytest.mark.parametrize("case", ["order1", "order2"])
def test_device_correction_builders_match_reference_fixture(case):
    """build_patch_blocks / build_near_corrections (solver.cpp:80-230) on the GPU against the arrays
    the reference produced (rule tables stored with the fixture)"""
    here = os.path.join(os.path.dirname(__file__), "golden")
    if case == "order1":
        g, pre, rp, order = G, "bie_", "bie_rule_", int(G["bie_order"])
    else:
        g, pre, rp, order = np.load(os.path.join(here, "corrections_order2.npz")), "", "rule_", 6
    k = float(g[pre + "k"])
    op = HfmmCuda(k=k, order=order, ncrit=16, theta=0.4, kd_max=1.0, leaf_cap=-1.0)
    op.set_points(g[pre + "xyz"])
    got = op.build_corrections(g[pre + "patches"], _tables(g, rp), mode=2)
    _check_corrections(got, {key: g[pre + key] for key in got})
    if case == "order1":
        # the installed (FP32) corrections reproduce the reference's operator and solve
        assert rel_l2(op.matvec(G["bie_x"]), G["bie_y"]) < 1e-5
        x, rep = op.gmres(G["bie_rhs"], rtol=1e-4, restart=30, max_iterations=200)
        assert rep["converged"] and abs(rep["iterations"] - int(G["bie_iterations"])) <= 1
    # modes: no near lists for self_only, no LU for none
    only = op.build_corrections(g[pre + "patches"], _tables(g, rp), mode=1)
    assert only["near_source"].size == 0 and np.array_equal(only["block_piv"], g[pre + "block_piv"])
    none = op.build_corrections(g[pre + "patches"], _tables(g, rp), mode=0)
    assert none["block_lu"].size == 0 and np.abs(none["patch_block"]).max() > 0
    with pytest.raises(HfmmError) as e:
        op.build_corrections(g[pre + "patches"][:-1], _tables(g, rp))
    assert e.value.kind == "config_error"


def test_device_correction_builders_against_oracle_midsize(oracle):
    """1,280 curved triangles, second-order basis (7,680 unknowns): device builder against the oracle's
    restatement (itself bit-identical to the reference, tests/test_oracle_golden.py)"""
    g2 = np.load(os.path.join(os.path.dirname(__file__), "golden", "corrections_order2.npz"))
    tables = _tables(g2, "rule_")
    patches = icosphere_patches(3)
    k = 3.0
    want = oracle.build_corrections(patches, tables, k)
    op = HfmmCuda(k=k, order=8, ncrit=32)
    op.set_points(want["xyz"])
    got = op.build_corrections(patches, tables)
    _check_corrections(got, want)
    assert got["near_source"].size > 1_000_000


def test_config3_pipeline_on_device_against_mie_series():
    """BASELINE config 3 at 20,480 triangles (61,440 unknowns), everything on the device: tree, lists,
    corrections, GMRES(30) to 1e-4; scattered field at r = 4 against the analytic Mie series
    (workloads.mie_soft_sphere, the series of oracle.cpp:11-59).  The mismatch is the discretisation error of the order-1 quadrature."""
    from paper_1803_09948_b200.workloads import patch_samples

    k = 4.0
    tables = _tables(G, "bie_rule_")
    patches = icosphere_patches(5)
    xyz = patch_samples(patches, tables["sample_ref"])
    op = HfmmCuda(k=k, order=12, ncrit=64, theta=0.4, kd_max=1.0, leaf_cap=-1.0)
    op.set_points(xyz)
    assert op.build_corrections(patches, tables, fetch=False) > 0
    x, rep = op.gmres(np.exp(1j * k * xyz[:, 2]), rtol=1e-4, restart=30, max_iterations=600, precondition=False)
    assert rep["converged"] and rep["final_residual"] <= 1.05e-4
    th = np.linspace(0, np.pi, 37)
    obs = np.stack([4 * np.sin(th), 0 * th, 4 * np.cos(th)], 1)
    scat = -op.evaluate_field(x, obs)       # physical field = minus the layer sum (solver.hpp:134-136)
    from paper_1803_09948_b200.workloads import mie_soft_sphere
    mie = mie_soft_sphere(1.0, k, 4.0, th)
    assert rel_l2(scat, mie) < 0.035
    if have_ref():   # the package's series is the reference's (oracle.cpp:11-59)
        from checkers import Ref
        assert rel_l2(mie, Ref().mie_soft_sphere(1.0, k, np.stack([4 + 0 * th, th, 0 * th], 1))) < 1e-12


def test_config3_full_size_iteration_count_against_the_reference_histories():
    """BASELINE config 3 as it stands (327,680 curved triangles, 983,040 unknowns, k = 4, P = 12, GMRES(30) to 1e-4),
    everything on the device, against the reference's OWN solves of the same system (tests/golden/
    config3_full_reference_gmres.json: 35 and 38 minutes on 16 host cores).  The north star's comparison is the
    reference "in FP32 complex": with its own single-precision near field the reference takes 25 iterations, the
    device must be within +-1 of that; the all-FP64 reference takes 22 and its first ten residuals are the device's
    to 1e-5 (identical operators), after which FP32 and FP64 part ways on the slowly converging tail."""
    import json

    from paper_1803_09948_b200.workloads import patch_samples

    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "config3_full_reference_gmres.json")))
    k = 4.0
    tables = _tables(G, "bie_rule_")
    patches = icosphere_patches(7)
    xyz = patch_samples(patches, tables["sample_ref"])
    assert len(xyz) == 983040
    op = HfmmCuda(k=k, order=12, ncrit=64, theta=0.4, kd_max=1.0, leaf_cap=-1.0)
    op.set_points(xyz)
    assert op.build_corrections(patches, tables, fetch=False) > 0
    x, rep = op.gmres(np.exp(1j * k * xyz[:, 2]), rtol=1e-4, restart=30, max_iterations=200, precondition=False)
    assert rep["converged"] and rep["final_residual"] <= 1.0e-4
    assert abs(rep["iterations"] - ref["fp32_near_field"]["iterations"]) <= 1, rep["iterations"]
    r, r64 = np.asarray(rep["residuals"][:10]), np.asarray(ref["fp64"]["residuals"][:10])
    assert np.max(np.abs(r - r64) / r64) < 1e-5
    assert rep["iterations"] >= ref["fp64"]["iterations"]


def test_device_correction_builders_edge_cases(oracle):
    """one patch, the near regime disabled (distance 0), every other patch near (huge distance)"""
    tables = _tables(G, "bie_rule_")
    patches = G["bie_patches"]
    k = 1.3
    for sel, dist in ((slice(0, 1), -1.0), (slice(0, 12), 0.0), (slice(0, 12), 50.0), (slice(0, 7), 0.4)):
        p = patches[sel]
        want = oracle.build_corrections(p, tables, k, mode=2, near_patch_distance=dist)
        op = HfmmCuda(k=k, order=4, ncrit=8)
        op.set_points(want["xyz"])
        got = op.build_corrections(p, tables, mode=2, near_patch_distance=dist)
        _check_corrections(got, want)
        if dist == 0.0 or len(p) == 1:
            assert got["near_source"].size == 0
        if dist == 50.0:   # every sample of every other patch, minus the coincident ones at shared vertices
            assert got["near_source"].size > 0.85 * len(p) * 3 * (len(p) - 1) * 3
        # the operator with these corrections still applies (empty CSR included)
        x = charges(len(want["xyz"]), 5)
        y = op.matvec(x)
        assert np.isfinite(y).all()


def test_deterministic_gmres_history_is_bitwise_reproducible():
    """with HFMM_FLAG_DETERMINISTIC two solves (fresh handles, corrections rebuilt on the device) give the
    same residual history and solution to the last bit; the Krylov reductions sum block partials in
    block order in every mode (gmres.cpp:13-23 accumulates in index order)"""
    from paper_1803_09948_b200.api import HFMM_FLAG_DETERMINISTIC
    from paper_1803_09948_b200.workloads import patch_samples

    k = 4.0
    tables = _tables(G, "bie_rule_")
    patches = icosphere_patches(3)
    xyz = patch_samples(patches, tables["sample_ref"])
    runs = []
    for _ in range(2):
        op = HfmmCuda(k=k, order=10, ncrit=32, theta=0.4, kd_max=1.0, leaf_cap=-1.0, flags=HFMM_FLAG_DETERMINISTIC)
        op.set_points(xyz)
        op.build_corrections(patches, tables, fetch=False)
        x, rep = op.gmres(np.exp(1j * k * xyz[:, 2]), rtol=1e-4, restart=30, max_iterations=300, precondition=True)
        assert rep["converged"]
        runs.append((x, rep["residuals"].copy(), rep["iterations"]))
    assert runs[0][2] == runs[1][2]
    assert np.array_equal(runs[0][1], runs[1][1])
    assert np.array_equal(runs[0][0], runs[1][0])


def test_repartitioning_loop_converges_on_a_clustered_set():
    """SURVEY.md section 8 row f3 end to end (partition.cpp:143-227): the loop measure -> update_alpha ->
    re-cut (distributed.Repartitioner) on a Plummer set with four emulated ranks.  The "runtime" fed to
    update_alpha is the slowest rank's modelled work (owned near body pairs + 1600 x owned M2L pairs, the
    measured kernel-time ratio), which makes the run deterministic.  The golden-section search must stay in
    [0, alpha_max] and settle, every partition it visits must reproduce the single-domain matvec, and the
    partition it settles on must not be worse than the one it started from."""
    import torch

    from paper_1803_09948_b200.distributed import Repartitioner, emulate_matvec_on_one_device
    from paper_1803_09948_b200.workloads import plummer_points

    n, k, order, ranks = 40000, 6.0, 6, 4
    xyz, q = plummer_points(n, 21), charges(n, 21)
    single = HfmmCuda(k=k, order=order, ncrit=32, theta=0.4)
    single.set_points(xyz)
    y1, order_m = single.matvec(q), single.body_order()
    qm = q[order_m]
    qd = torch.from_numpy(np.stack([qm.real, qm.imag], 1).astype(np.float32)).cuda()

    def make_ops(alpha):
        ops = []
        for rank in range(ranks):
            op = HfmmCuda(k=k, order=order, ncrit=32, theta=0.4)
            op.set_partition(rank, ranks)
            op.set_partition_alpha(alpha)
            op.set_points(xyz)
            ops.append(op)
        return ops

    def slowest(ops):
        return max(int(op.partition().owned_p2p_body_pairs) + 1600 * int(op.partition().owned_m2l_pairs) for op in ops)

    rp = Repartitioner(make_ops, alpha_max=2.0)
    visited, work = [], []
    for _ in range(12):
        ops = rp.operator
        y = emulate_matvec_on_one_device(ops, qd).cpu().numpy()
        assert rel_l2(y[:, 0] + 1j * y[:, 1], y1[order_m]) < 3e-6
        visited.append(rp.alpha)
        work.append(slowest(ops))
        if not rp.record(work[-1]):
            break
    assert all(0.0 <= a <= 2.0 for a in visited)
    assert len(visited) >= 4                                   # it searched
    assert abs(visited[-1] - visited[-2]) < abs(visited[1] - visited[0])   # and the bracket shrank
    assert work[-1] <= 1.02 * min(work)                       # it sits at (or next to) the best partition it saw


def test_gmres_with_repartitioning_between_restart_cycles():
    """f3 inside the solver: restart cycles driven by the caller (hfmm_cuda_dist_solve with max_iterations =
    restart on the residual equation, hfmm_cuda_get_solve_residual), the Morton partition re-cut by the
    repartitioning loop at every restart boundary.  Same iteration as the monolithic restarted solver: same
    count +-1, same solution."""
    from paper_1803_09948_b200.distributed import repartitioned_gmres_emulated

    single = _bie_operator(G)
    order = single.body_order()
    rhs = np.asarray(G["bie_rhs"])

    def make_ops(alpha):
        ops = []
        for r in range(2):
            op = HfmmCuda(k=float(G["bie_k"]), order=int(G["bie_order"]), ncrit=16, theta=0.4, kd_max=1.0, leaf_cap=-1.0)
            op.set_partition(r, 2)
            op.set_partition_alpha(alpha)
            op.set_points(G["bie_xyz"])
            op.set_corrections(int(G["bie_ni"]), far_weight=G["bie_far_weight"], patch_block=G["bie_patch_block"],
                               near_offset=G["bie_near_offset"], near_source=G["bie_near_source"],
                               near_delta=G["bie_near_delta"], block_lu=G["bie_block_lu"], block_piv=G["bie_block_piv"])
            ops.append(op)
        return ops

    for precondition in (True, False):
        x1, rep1 = single.gmres(rhs, rtol=1e-4, restart=6, max_iterations=300, precondition=precondition)
        assert rep1["converged"] and rep1["iterations"] > 12          # several restart cycles
        x, rep = repartitioned_gmres_emulated(make_ops, rhs[order], rtol=1e-4, restart=6, max_iterations=300,
                                              precondition=precondition)
        assert rep["converged"] and rep["final_residual"] <= 1.05e-4
        assert abs(rep["iterations"] - rep1["iterations"]) <= 1, (rep["iterations"], rep1["iterations"])
        assert rep["recuts"] >= 2 and len(set(rep["alphas"])) >= 3   # the loop moved alpha between cycles
        assert rel_l2(x, x1[order]) < 2e-3
        # the single-domain solver exposes the same vector: b - Z u of the last solve
        r1 = single.solve_residual()
        assert abs(np.linalg.norm(r1) / np.linalg.norm(rhs) - rep1["final_residual"]) < 1e-6


def test_cli_solve_verify_scaling(tmp_path, capsys):
    """SPEC cmd_solve (report JSON, residual CSV, field CSV; exit 0 on convergence), cmd_verify (Mie error per basis
    order, decreasing with the order) and cmd_scaling (one CSV row per N, duplicates averaged) through the package's
    command line"""
    import json

    from paper_1803_09948_b200.__main__ import main

    prefix = str(tmp_path / "run")
    assert main(["solve", "--subdivisions", "2", "--k", "2", "--order", "8", "--out-prefix", prefix]) == 0
    rep = json.load(open(prefix + ".report.json"))
    assert rep["converged"] and rep["final_residual"] <= 1e-4 and len(rep["residuals"]) == rep["iterations"]
    assert len(open(prefix + ".residuals.csv").read().splitlines()) == rep["iterations"] + 1
    assert len(open(prefix + ".field.csv").read().splitlines()) == 37 + 1
    capsys.readouterr()
    assert main(["verify", "--subdivisions", "2", "--k", "2", "--order", "8", "--orders", "1", "2"]) == 0
    out = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    errs = [r["mie_mismatch_rel_l2"] for r in out["rows"]]
    assert out["errors_decrease"] and errs[1] < errs[0] < 0.3
    assert main(["verify", "--k", "0"]) == 64                                  # zero frequency is rejected
    assert main(["scaling", "--n", "20000", "40000", "20000", "--order", "6"]) == 0
    rows = capsys.readouterr().out.strip().splitlines()
    assert rows[0] == "n,fmm_seconds,count" and len(rows) == 3 and rows[1].endswith(",2") and rows[2].endswith(",1")
