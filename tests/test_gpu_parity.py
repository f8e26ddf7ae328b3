"""GPU parity of the FMM matvec (through the C ABI) against the CPU oracle.

Tolerance: BASELINE.json's north star — relative L2 <= 1e-5 in complex FP32 against the
reference's own FMM matvec on the same inputs and expansion order."""
import numpy as np
import pytest

from checkers import rel_l2
from paper_1803_09948_b200 import HfmmCuda, HfmmError
from paper_1803_09948_b200.workloads import charges, plummer_points, sphere_points

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _run(xyz, q, k, order, **kw):
    op = HfmmCuda(k=k, order=order, **kw)
    op.set_points(xyz)
    return op, op.matvec(q)


@pytest.mark.parametrize("n,k,order,ncrit,cap", [
    (1000, 2.0, 10, 20, 0.5),      # reference tests/test_fmm.cpp:941-961 (pipeline vs direct sum)
    (4096, 1.0, 8, 32, -1.0),
    (6000, 4.0, 12, 64, -1.0),
])
def test_matvec_vs_oracle_fmm(oracle, n, k, order, ncrit, cap):
    xyz, q = sphere_points(n, 5), charges(n, 5)
    cap_res = cap if cap >= 0 else 1.0 / k
    op, y = _run(xyz, q, k, order, ncrit=ncrit, leaf_cap=cap)
    f = oracle.fmm(xyz, k, order, ncrit=ncrit, leaf_cap=cap_res, theta=0.4, kd_max=1.0)
    y_ref = f.matvec(q)
    c = f.counts()
    st = op.stats()
    assert st["n_cells"] == c["cells"] and st["n_leaves"] == c["leaves"]
    assert st["m2l_pairs"] == c["m2l_pairs"] and st["p2p_pairs"] == c["p2p_pairs"]
    assert st["p2p_body_pairs"] == c["p2p_body_pairs"]
    assert rel_l2(y, y_ref) < TOL


@pytest.mark.parametrize("n,k,ncrit,grain,cap", [(5000, 2.0, 20, 40, 0.5), (3000, 4.0, 32, 32, -1.0),
                                                 (40, 1.0, 64, 128, 0.0), (2000, 1.0, 16, 4000, 0.0)])
def test_task_and_starved_counters_match_the_reference(n, k, ncrit, grain, cap):
    """FmmStats::tasks (traversal.cpp:56-59) and ::starved_cells (expansion.cpp:253-262), device and host builder"""
    from checkers import Ref, have_ref
    if not have_ref():
        pytest.skip("compiled reference not on this box")
    from paper_1803_09948_b200.api import HFMM_FLAG_HOST_TREE
    xyz, q = plummer_points(n, 77), charges(n, 77)
    cap_res = cap if cap >= 0 else 1.0 / k
    f = Ref().fmm(xyz, k, 6, ncrit=ncrit, leaf_cap=cap_res, theta=0.4, kd_max=1.0, s=grain)
    f.matvec(q)
    for flags in (0, HFMM_FLAG_HOST_TREE):
        op = HfmmCuda(k=k, order=6, ncrit=ncrit, grain=grain, leaf_cap=cap, flags=flags)
        op.set_points(xyz)
        st = op.stats()
        assert st["host_tree_used"] == (1 if flags else 0)
        assert st["tasks"] == f.tasks(), (flags, st["tasks"], f.tasks())
        assert st["starved_cells"] == f.starved()
    # a wavenumber small enough for j_P(k r) to underflow in FP64: every cell is starved, on both sides
    f2 = Ref().fmm(xyz, 1e-30, 12, ncrit=ncrit, leaf_cap=0.0, theta=0.4, kd_max=0.0, s=grain)
    f2.matvec(q)
    op = HfmmCuda(k=1e-30, order=12, ncrit=ncrit, grain=grain, leaf_cap=0.0, kd_max=0.0)
    op.set_points(xyz)
    assert f2.starved() == f2.counts()["cells"] == op.stats()["starved_cells"]


def test_near_field_only(oracle):
    # theta tiny-ish and kd gate closed => everything is P2P: checks the near kernel alone
    n, k = 3000, 3.0
    xyz, q = sphere_points(n, 9), charges(n, 9)
    op, y = _run(xyz, q, k, 4, ncrit=50, kd_max=1e-9, leaf_cap=0.0)
    assert op.stats()["m2l_pairs"] == 0
    assert rel_l2(y, oracle.direct_sum(xyz, q, k)) < 2e-6


def test_expansions_match_oracle(oracle):
    n, k, order = 3000, 2.0, 8
    xyz, q = sphere_points(n, 21), charges(n, 21)
    op, _ = _run(xyz, q, k, order, ncrit=24, leaf_cap=0.5)
    f = oracle.fmm(xyz, k, order, ncrit=24, leaf_cap=0.5)
    f.matvec(q)
    # match cells by (level, ix, iy, iz)
    key = lambda c: [tuple(r) for r in c[:, :4].tolist()]
    mine = {kk: i for i, kk in enumerate(key(op.cells()))}
    theirs = key(f.cells())
    perm = np.array([mine[kk] for kk in theirs])
    lvl = f.cells()[:, 0]
    for which, name in ((0, "multipole"), (1, "local")):
        a = op.expansions(which)[perm]
        b = f.expansions(which, order)
        # only levels that take part in translations are computed on the device
        used = np.abs(a).sum(axis=1) > 0
        assert used.any()
        err = np.linalg.norm(a[used] - b[used], axis=1) / np.linalg.norm(b[used], axis=1)
        assert err.max() < 5e-5, (name, err.max(), lvl[used][err.argmax()])


def test_clustered_volume(oracle):
    n, k, order = 8000, 8.0, 10
    xyz, q = plummer_points(n, 3, a=0.05), charges(n, 3)
    op, y = _run(xyz, q, k, order, ncrit=64, theta=0.35)
    assert rel_l2(y, oracle.direct_sum(xyz, q, k)) < TOL


def test_linearity_and_repeatability():
    n, k = 5000, 2.0
    xyz = sphere_points(n, 2)
    q1, q2 = charges(n, 1), charges(n, 2)
    op = HfmmCuda(k=k, order=8)
    op.set_points(xyz)
    y1, y2, y12 = op.matvec(q1), op.matvec(q2), op.matvec(q1 + 2j * q2)
    assert rel_l2(y12, y1 + 2j * y2) < 5e-6
    assert np.abs(op.matvec(np.zeros(n))).max() == 0.0


@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_sharded_matvec_equals_single_domain(nranks):
    """Multi-GPU mode, ranks emulated sequentially on one device (distributed.py): partitioned work
    lists + charge / multipole exchange reproduce the single-domain matvec; the reference's own
    simulator agrees with its single-rank run to 1e-9, ours to FP32 summation order."""
    import torch

    from paper_1803_09948_b200.distributed import emulate_ranks_on_one_device

    n, k, order = 20000, 4.0, 10
    xyz, q = sphere_points(n, 12), charges(n, 12)
    single = HfmmCuda(k=k, order=order)
    single.set_points(xyz)
    y_ref = single.matvec(q)
    morton = single.body_order()
    ops = []
    for r in range(nranks):
        op = HfmmCuda(k=k, order=order)
        op.set_partition(r, nranks)
        op.set_points(xyz)
        ops.append(op)
    qm = q[morton]
    q_dev = torch.from_numpy(np.stack([qm.real, qm.imag], 1).astype(np.float32)).cuda()
    out, parts = emulate_ranks_on_one_device(ops, q_dev)
    y = out.cpu().numpy()
    y = y[:, 0] + 1j * y[:, 1]
    y_caller = np.empty_like(y)
    y_caller[morton] = y
    assert rel_l2(y_caller, y_ref) < 2e-6
    # every body owned exactly once, all work accounted for
    assert sum(int(p.body_count) for p in parts) == n
    st = single.stats()
    assert sum(int(p.owned_m2l_pairs) for p in parts) == st["m2l_pairs"]
    assert sum(int(p.owned_p2p_body_pairs) for p in parts) == st["p2p_body_pairs"]


@pytest.mark.parametrize("nranks,dist_kind", [(2, "sphere"), (4, "plummer"), (8, "sphere")])
def test_pair_lists_are_built_per_rank(nranks, dist_kind):
    """Multi-rank setup: a rank stores only the walk's pairs whose target it owns (its work) or whose source
    it owns (what it must send) — reference: one tree per rank + grafted LETs, let.cpp:98-123, 150-318.  The
    union over the ranks of the target-owned pairs is the single-domain list, every pair exactly once; the
    statistics stay those of the global lists; the cuts are the ones every rank derives on its own."""
    n, k, order = 30000, 4.0, 8
    xyz = sphere_points(n, 21) if dist_kind == "sphere" else plummer_points(n, 21, a=0.05)
    single = HfmmCuda(k=k, order=order)
    single.set_points(xyz)
    st = single.stats()
    glob = [set(map(tuple, single.pairs(w).tolist())) for w in (0, 1)]
    assert len(glob[0]) == st["m2l_pairs"] and len(glob[1]) == st["p2p_pairs"]
    seen = [set(), set()]
    stored = 0
    cuts = None
    for r in range(nranks):
        op = HfmmCuda(k=k, order=order)
        op.set_partition(r, nranks)
        op.set_points(xyz)
        sr = op.stats()
        for key in ("m2l_pairs", "p2p_pairs", "p2p_body_pairs", "tasks", "n_cells"):
            assert sr[key] == st[key], key
        _, _, owner = op.exchange_masks()
        cuts = owner if cuts is None else cuts
        assert np.array_equal(owner, cuts)  # same partition on every rank, no handshake
        for w in (0, 1):
            pr = op.pairs(w)
            stored += len(pr)
            t_mine, s_mine = owner[pr[:, 0]] == r, owner[pr[:, 1]] == r
            assert np.all(t_mine | s_mine)  # nothing the rank neither computes nor sends
            mine = set(map(tuple, pr[t_mine].tolist()))
            assert len(mine) == int(t_mine.sum()) and not (mine & seen[w])
            seen[w] |= mine
            # complete on the sending side too: every global pair out of one of its cells is there
            need = {p for p in glob[w] if owner[p[1]] == r}
            assert need <= set(map(tuple, pr.tolist()))
        del op
    assert seen[0] == glob[0] and seen[1] == glob[1]
    total = len(glob[0]) + len(glob[1])
    # each pair is stored by the owner of its target and the owner of its source: at most twice over all ranks,
    # against `nranks` copies of the global lists before
    assert stored <= 2 * total


@pytest.mark.parametrize("nranks,dist_kind", [(2, "sphere"), (5, "plummer"), (8, "sphere")])
def test_library_data_plane_reproduces_the_single_domain_matvec(nranks, dist_kind):
    """hfmm_cuda_dist_matvec (csrc/comm.cu): pack kernel -> exchange -> unpack kernel for the halo charges and the
    remote multipoles, index lists derived inside the library.  Ranks are host threads on this one GPU joined by the
    host transport; everything except the ncclSend / ncclRecv calls is the code a multi-GPU run executes."""
    import torch

    from paper_1803_09948_b200.distributed import emulate_matvec_on_one_device

    n, k, order = 24000, 5.0, 9
    xyz = sphere_points(n, 31) if dist_kind == "sphere" else plummer_points(n, 31, a=0.06)
    q = charges(n, 31)
    single = HfmmCuda(k=k, order=order, ncrit=40)
    single.set_points(xyz)
    morton = single.body_order()
    y_ref = single.matvec(q)[morton]
    ops = []
    for r in range(nranks):
        op = HfmmCuda(k=k, order=order, ncrit=40)
        op.set_partition(r, nranks)
        op.set_points(xyz)
        ops.append(op)
    qm = q[morton]
    q_dev = torch.from_numpy(np.stack([qm.real, qm.imag], 1).astype(np.float32)).cuda()
    for _ in range(2):                   # the second product reuses plan and buffers
        out = emulate_matvec_on_one_device(ops, q_dev)
    y = out.cpu().numpy()
    assert rel_l2(y[:, 0] + 1j * y[:, 1], y_ref) < 3e-6
    vol = [op.exchange_volume() for op in ops]
    full = 8 * n + single.stats()["n_cells"] * 8 * (order + 1) ** 2
    assert all(c + m < full for c, m in vol) and sum(c for c, _ in vol) > 0
    # a new point set rebuilds the exchange lists
    xyz2 = sphere_points(n, 32)
    single.set_points(xyz2)
    for op in ops:
        op.set_points(xyz2)
    m2 = single.body_order()
    q2 = q[m2]
    out = emulate_matvec_on_one_device(ops, torch.from_numpy(np.stack([q2.real, q2.imag], 1).astype(np.float32)).cuda())
    y = out.cpu().numpy()
    assert rel_l2(y[:, 0] + 1j * y[:, 1], single.matvec(q)[m2]) < 3e-6


@pytest.mark.parametrize("nranks,dist_kind", [(3, "sphere"), (8, "plummer")])
def test_pruned_let_exchange_is_sufficient(nranks, dist_kind):
    """a rank receives only the multipoles its own M2L lists translate
    from and the bodies of the leaves on its own near lists (all other charges are poisoned, all
    other multipole rows stay zero) and still reproduces the single-domain matvec; send and receive
    lists of every pair of ranks agree element for element"""
    import torch

    from paper_1803_09948_b200.distributed import emulate_ranks_on_one_device, let_index_lists

    n, k, order = 30000, 6.0, 8
    xyz = sphere_points(n, 14) if dist_kind == "sphere" else plummer_points(n, 14)
    q = charges(n, 14)
    single = HfmmCuda(k=k, order=order, ncrit=48)
    single.set_points(xyz)
    y_ref = single.matvec(q)
    morton = single.body_order()
    ops = []
    for r in range(nranks):
        op = HfmmCuda(k=k, order=order, ncrit=48)
        op.set_partition(r, nranks)
        op.set_points(xyz)
        ops.append(op)
    qm = q[morton]
    q_dev = torch.from_numpy(np.stack([qm.real, qm.imag], 1).astype(np.float32)).cuda()
    out, parts = emulate_ranks_on_one_device(ops, q_dev, pruned=True)
    y = out.cpu().numpy()
    assert rel_l2(y[:, 0] + 1j * y[:, 1], y_ref[morton]) < 3e-6
    # the halo is a fraction of a full gather
    n_cells = single.stats()["n_cells"]
    lists = [let_index_lists(op, r, nranks) for r, op in enumerate(ops)]
    recv_cells = max(sum(len(a) for a in l["recv_cells"]) for l in lists)
    recv_bodies = max(sum(len(a) for a in l["recv_bodies"]) for l in lists)
    assert recv_cells < 0.8 * n_cells and recv_bodies < 0.8 * n


def _geo_pairs(cells, pairs):
    key = lambda c: ((cells[c, 0].astype(np.int64) << 57) | (cells[c, 1].astype(np.int64) << 38)
                     | (cells[c, 2].astype(np.int64) << 19) | cells[c, 3].astype(np.int64))
    a = np.stack([key(pairs[:, 0]), key(pairs[:, 1])], 1)
    return a[np.lexsort((a[:, 1], a[:, 0]))]


@pytest.mark.parametrize("case", ["pipeline", "sphere", "plummer", "gate_off"])
def test_device_built_tree_and_lists_equal_the_reference(case):
    """Tree and interaction lists built ON THE GPU (tree_build.cu) against the fixtures the
    reference generated: same Morton order, same cell set, same M2L / P2P pair sets — including the
    `pipeline` case whose theta = 0.5 lattice produces exact admissibility ties — and the same
    results as the host builder (HFMM_FLAG_HOST_TREE)."""
    import os

    from paper_1803_09948_b200.api import HFMM_FLAG_HOST_TREE

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "fmm.npz"))
    k, order, ncrit, cap, theta, kd = g[f"{case}_params"]
    kw = dict(k=float(k), order=int(order), ncrit=int(ncrit), theta=float(theta), kd_max=float(kd),
              leaf_cap=float(cap))
    dev = HfmmCuda(**kw)
    dev.set_points(g[f"{case}_xyz"])
    host = HfmmCuda(flags=HFMM_FLAG_HOST_TREE, **kw)
    host.set_points(g[f"{case}_xyz"])
    ref_cells = g[f"{case}_cells"]
    canon = lambda c: (lambda a: a[np.lexsort(a.T[::-1])])(c[:, :6].astype(np.int64))
    assert (dev.body_order() == g[f"{case}_order"]).all()
    assert (canon(dev.cells()) == canon(ref_cells)).all()
    assert (dev.cells() == host.cells()).all()               # identical level-order numbering
    for which, name in ((0, "m2l"), (1, "p2p")):
        ref_pairs = _geo_pairs(ref_cells, g[f"{case}_{name}"])
        assert (_geo_pairs(dev.cells(), dev.pairs(which)) == ref_pairs).all()
        assert (_geo_pairs(host.cells(), host.pairs(which)) == ref_pairs).all()
    sd, sh = dev.stats(), host.stats()
    for key in ("n_cells", "n_leaves", "max_level", "m2l_pairs", "p2p_pairs", "p2p_body_pairs",
                "m2l_shift_classes", "rotation_tables", "coaxial_tables"):
        assert sd[key] == sh[key], key
    q = g[f"{case}_q"]
    yd, yh = dev.matvec(q), host.matvec(q)
    assert rel_l2(yd, g[f"{case}_y"]) < TOL and rel_l2(yh, g[f"{case}_y"]) < TOL
    assert rel_l2(yd, yh) < 2e-6


# ---- edge cases (reference tests/test_fmm.cpp:897-939 "base cases", octree.cpp degenerate leaves) ----
def _check_against_direct(oracle, xyz, q, k, order, tol=TOL, **kw):
    op = HfmmCuda(k=k, order=order, **kw)
    op.set_points(xyz)
    y = op.matvec(q)
    exact = oracle.direct_sum(xyz, q, k)
    assert np.isfinite(y).all()
    if np.linalg.norm(exact) > 0:
        assert rel_l2(y, exact) < tol
    else:
        assert np.abs(y).max() == 0
    return op


def test_tiny_inputs(oracle):
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 17, 65):
        xyz = rng.uniform(-1, 1, (n, 3))
        q = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        op = _check_against_direct(oracle, xyz, q, 1.5, 6, ncrit=4)
        assert op.stats()["n_bodies"] == n


def test_coincident_and_degenerate_geometry(oracle):
    rng = np.random.default_rng(4)
    q = rng.uniform(-1, 1, 300) + 1j * rng.uniform(-1, 1, 300)
    # all bodies on one point: the box degenerates (width := 1), every pair is skipped (R = 0)
    same = np.tile([[0.3, -0.2, 0.7]], (300, 1))
    _check_against_direct(oracle, same, q, 2.0, 6, ncrit=16)
    # 40 bodies on one point inside a cloud: an over-full leaf at level 21 (degenerate leaf)
    cloud = rng.uniform(-1, 1, (300, 3))
    cloud[:40] = cloud[0]
    _check_against_direct(oracle, cloud, q, 2.0, 8, ncrit=16)
    # collinear and coplanar sets
    line = np.zeros((300, 3)); line[:, 0] = np.linspace(-1, 1, 300)
    _check_against_direct(oracle, line, q, 3.0, 8, ncrit=8)
    plane = rng.uniform(-1, 1, (300, 3)); plane[:, 2] = 0.25
    _check_against_direct(oracle, plane, q, 3.0, 8, ncrit=8)


@pytest.mark.parametrize("order", [0, 1, 2, 5, 16])
def test_expansion_orders(oracle, order):
    # any order up to the supported maximum; accuracy is checked against the oracle FMM at the
    # SAME order (low orders truncate, they are not supposed to match the direct sum)
    n, k = 2500, 2.0
    xyz, q = sphere_points(n, 31), charges(n, 31)
    op = HfmmCuda(k=k, order=order, ncrit=32)
    op.set_points(xyz)
    y = op.matvec(q)
    y_ref = oracle.fmm(xyz, k, order, ncrit=32, leaf_cap=0.5, theta=0.4, kd_max=1.0).matvec(q)
    assert rel_l2(y, y_ref) < TOL


def test_leaf_capacity_extremes(oracle):
    n, k = 1500, 2.0
    xyz, q = sphere_points(n, 33), charges(n, 33)
    for ncrit in (1, 7, 200, 5000):      # 5000 > n: a single leaf, pure direct sum
        _check_against_direct(oracle, xyz, q, k, 10, ncrit=ncrit)


def test_argument_errors():
    from paper_1803_09948_b200 import HfmmError

    op = HfmmCuda(k=1.0, order=4)
    with pytest.raises(HfmmError) as e:      # matvec before set_points
        op.lib.hfmm_cuda_matvec  # noqa: B018
        op.n = 4
        op.matvec(np.zeros(4))
    assert e.value.kind == "config_error"
    bad = np.zeros((10, 3)); bad[3, 1] = np.nan
    with pytest.raises(HfmmError) as e:
        op.set_points(bad)
    assert e.value.kind == "domain_error"
    with pytest.raises(HfmmError) as e:
        op.set_points(np.zeros((0, 3)))
    assert e.value.kind == "config_error"    # "no bodies to enclose" (octree.cpp:54)
    op.set_points(np.random.default_rng(0).uniform(-1, 1, (50, 3)))
    with pytest.raises(ValueError):
        op.matvec(np.zeros(49))


def test_interaction_lists_cover_every_body_pair_exactly_once():
    """reference tests/test_fmm.cpp:865-895 (once-cover): the M2L cell pairs and the P2P leaf pairs of
    the device-built lists tile the (target body, source body) matrix — each entry exactly once"""
    n = 700
    xyz = np.concatenate([sphere_points(n - 200, 21), 0.3 * sphere_points(200, 22) + 0.1])
    op = HfmmCuda(k=3.0, order=4, ncrit=12, theta=0.5, kd_max=1.0, leaf_cap=-1.0)
    op.set_points(xyz)
    cells = op.cells()
    first, count = cells[:, 4].astype(np.int64), cells[:, 5].astype(np.int64)
    cover = np.zeros((n, n), dtype=np.int32)
    for which in (0, 1):
        for t, s in op.pairs(which):
            cover[first[t]:first[t] + count[t], first[s]:first[s] + count[s]] += 1
    assert cover.min() == 1 and cover.max() == 1
    # P2P pairs join leaves only; no M2L pair has a cell wider than the kd gate allows
    leaf = cells[:, 7] == 0
    p2p = op.pairs(1)
    assert leaf[p2p[:, 0]].all() and leaf[p2p[:, 1]].all()


def test_measured_weights_and_alpha_cuts(oracle):
    """per-body work estimates equal the reference's measure_weights
    (through the oracle restatement, pinned in tests/test_oracle_vs_reference.py); Morton cuts balanced
    by w = l + alpha r still reproduce the single-domain matvec and balance that estimate"""
    import torch

    from paper_1803_09948_b200.distributed import emulate_ranks_on_one_device

    n, k, order = 20000, 6.0, 6
    xyz, q = plummer_points(n, 12), charges(n, 12)
    single = HfmmCuda(k=k, order=order, ncrit=32, theta=0.4)
    single.set_points(xyz)
    fo = oracle.fmm(xyz, k, order, ncrit=32, leaf_cap=1.0 / k, theta=0.4, kd_max=1.0)
    lo, ro = fo.measure_weights()
    l, r = single.measure_weights()
    assert np.array_equal(l, lo) and np.array_equal(r, ro)
    y1 = single.matvec(q)
    order_m = single.body_order()
    for alpha in (0.0, 40.0):
        ops = []
        for rank in range(3):
            op = HfmmCuda(k=k, order=order, ncrit=32, theta=0.4)
            op.set_partition(rank, 3)
            op.set_partition_alpha(alpha)
            op.set_points(xyz)
            ops.append(op)
        qm = q[order_m]
        qd = torch.from_numpy(np.stack([qm.real, qm.imag], 1).astype(np.float32)).cuda()
        out, parts = emulate_ranks_on_one_device(ops, qd)
        y = out.cpu().numpy()
        assert rel_l2(y[:, 0] + 1j * y[:, 1], y1[order_m]) < 3e-6
        # the cuts balance the chosen estimate: no rank holds more than 45 % of sum(l + alpha r)
        w = (l + alpha * r)[order_m]
        tot = [w[int(p.body_first):int(p.body_first) + int(p.body_count)].sum() for p in parts]
        assert max(tot) / sum(tot) < 0.45



@pytest.mark.parametrize("k", [2.0 + 0.5j, 4.0 + 0.05j, 1.0 + 1.5j])
def test_complex_wavenumber(oracle, k):
    """k = k_r + i k_i (attenuation, common.hpp:36-40; e^{-k_i R} in kernel.hpp:20): near field,
    expansions with complex radial functions and complex translation tables against the FP64 direct
    sum, and against the compiled reference's FMM at the same order where it travelled to the box"""
    from checkers import have_ref

    n, order = 5000, 12
    xyz = np.concatenate([sphere_points(n - 1500, 31), 0.4 * sphere_points(1500, 32) + 0.05])
    q = charges(n, 31)
    op = HfmmCuda(k=k, order=order, ncrit=40, theta=0.4, kd_max=1.0, leaf_cap=-1.0)
    op.set_points(xyz)
    y = op.matvec(q)
    st = op.stats()
    assert st["m2l_pairs"] > 0 and st["p2p_pairs"] > 0
    exact = oracle.direct_sum(xyz, q, k)
    assert rel_l2(y, exact) < 1e-5
    # the oracle's FMM at the same order (bit-identical to the reference's for complex k as well,
    # tests/test_oracle_golden.py): identical lists, FP32 distance of the potentials
    fo = oracle.fmm(xyz, k, order, ncrit=40, leaf_cap=1.0 / abs(k), theta=0.4, kd_max=1.0)
    co = fo.counts()
    assert st["m2l_pairs"] == co["m2l_pairs"] and st["p2p_body_pairs"] == co["p2p_body_pairs"]
    assert rel_l2(y, fo.matvec(q)) < 1e-5
    # near field alone (gate closed: every pair is evaluated directly)
    near = HfmmCuda(k=k, order=4, ncrit=50, kd_max=1e-9, leaf_cap=0.0)
    near.set_points(xyz[:2500])
    assert near.stats()["m2l_pairs"] == 0
    assert rel_l2(near.matvec(q[:2500]), oracle.direct_sum(xyz[:2500], q[:2500], k)) < 2e-6
    # exterior field evaluation uses the same damped kernel
    obs = np.array([[3.0, 0.5, -1.0], [0.0, 0.0, 2.5], [-2.0, 2.0, 2.0]])
    d = np.linalg.norm(obs[:, None, :] - xyz[None, :, :], axis=2)
    want = (np.exp(1j * k * d) / (4 * np.pi * d)) @ q
    assert rel_l2(op.evaluate_field(q, obs), want) < 5e-6
    if have_ref():
        from checkers import Ref
        f = Ref().fmm(xyz, k, order, ncrit=40, leaf_cap=1.0 / abs(k), theta=0.4, kd_max=1.0)
        c = f.counts()
        assert st["m2l_pairs"] == c["m2l_pairs"] and st["p2p_body_pairs"] == c["p2p_body_pairs"]
        assert rel_l2(y, f.matvec(q)) < 1e-5


@pytest.mark.parametrize("order", [0, 1, 3, 7, 10, 12, 13, 14, 16])
def test_64_pair_translation_kernel_against_the_32_pair_kernel(oracle, monkeypatch, order):
    """orders <= 16 run the 64-pair in-place kernel (kernels_translate64.cu: two 8-warp CTAs per SM up to
    P = 12, one 16-warp CTA with pair-split tasks beyond; P = 10, 12, 14 are compile-time specialisations);
    HFMM_TRANSLATE=32 forces the 32-pair ping-pong kernel on the same lists: same operator, two work layouts"""
    n, k = 12000, 5.0
    xyz, q = plummer_points(n, 43), charges(n, 43)
    res = {}
    for kernel in ("64", "32"):
        monkeypatch.setenv("HFMM_TRANSLATE", kernel)
        op = HfmmCuda(k=k, order=order, ncrit=32)
        op.set_points(xyz)
        res[kernel] = op.matvec(q)
        if kernel == "64":
            pairs, batches = op.stats()["m2l_pairs"], op.stats()["m2l_batches"]
            assert pairs > 0 and batches * 32 < 2 * pairs + 64 * 2000   # 64-pair batches
    assert rel_l2(res["64"], res["32"]) < 2e-6
    if order >= 7:
        tg = np.arange(0, n, 23)
        assert rel_l2(res["64"][tg], oracle.direct_sum(xyz, q, k, tg)) < (1e-3 if order == 7 else 2e-6)


@pytest.mark.parametrize("order", [6, 13])
def test_both_batch_layouts_of_the_translation_kernel(oracle, monkeypatch, order):
    """batches cut per table group (per-pair azimuth phases) and per shift class (per-class phases) are two
    instantiations of the kernel; the library picks by batch count — force each and compare (order 13
    runs the 16-warp variant)"""
    n, k = 9000, 5.0
    xyz, q = plummer_points(n, 41), charges(n, 41)
    res, batches = {}, {}
    monkeypatch.setenv("HFMM_TRANSLATE", "32")     # the 64-pair kernel always batches per table group
    for layout in ("group", "class"):
        monkeypatch.setenv("HFMM_BATCHING", layout)
        op = HfmmCuda(k=k, order=order, ncrit=32)
        op.set_points(xyz)
        res[layout] = op.matvec(q)
        batches[layout] = op.stats()["m2l_batches"]
    assert batches["group"] < batches["class"]
    assert rel_l2(res["group"], res["class"]) < 1e-6
    tg = np.arange(0, n, 23)
    assert rel_l2(res["class"][tg], oracle.direct_sum(xyz, q, k, tg)) < (2e-5 if order == 6 else 2e-6)


def test_deterministic_flag_gives_bitwise_reproducible_results(monkeypatch):
    """TraversalConfig::deterministic (traversal.hpp:11-22) / test_fmm.cpp:1024-1050: with the flag the
    far field adds the contributions of every cell in list order (staged rows + ordered reduction, no
    floating-point atomics): repeated matvecs and fresh handles agree to the last bit, with either
    tree builder, and with the staging buffer cut into many ranges"""
    from paper_1803_09948_b200.api import HFMM_FLAG_DETERMINISTIC, HFMM_FLAG_HOST_TREE
    n, k = 20000, 5.0
    xyz, q = plummer_points(n, 77), charges(n, 77)
    ref_op = HfmmCuda(k=k, order=8, ncrit=32)
    ref_op.set_points(xyz)
    y_default = ref_op.matvec(q)
    for flags, budget in ((HFMM_FLAG_DETERMINISTIC, None), (HFMM_FLAG_DETERMINISTIC | HFMM_FLAG_HOST_TREE, None),
                          (HFMM_FLAG_DETERMINISTIC, "1")):
        if budget:
            monkeypatch.setenv("HFMM_ORDERED_STAGING_MB", budget)
        runs = []
        for _ in range(2):
            op = HfmmCuda(k=k, order=8, ncrit=32, flags=flags)
            op.set_points(xyz)
            runs.append(op.matvec(q))
            runs.append(op.matvec(q))
        for y in runs[1:]:
            assert np.array_equal(y, runs[0])
        assert rel_l2(runs[0], y_default) < 1e-6
        monkeypatch.delenv("HFMM_ORDERED_STAGING_MB", raising=False)


def test_sharded_matvec_with_ordered_accumulation_is_reproducible():
    """HFMM_FLAG_DETERMINISTIC on every rank of the (emulated) sharded matvec: two runs agree bit for
    bit — each rank reduces the pairs of its own targets in list order, the exchanges copy bits"""
    import torch

    from paper_1803_09948_b200.api import HFMM_FLAG_DETERMINISTIC
    from paper_1803_09948_b200.distributed import emulate_ranks_on_one_device

    n, k, order, nranks = 20000, 4.0, 8, 3
    xyz, q = sphere_points(n, 21), charges(n, 21)
    outs = []
    for _ in range(2):
        ops = []
        for r in range(nranks):
            op = HfmmCuda(k=k, order=order, flags=HFMM_FLAG_DETERMINISTIC)
            op.set_partition(r, nranks)
            op.set_points(xyz)
            ops.append(op)
        qm = q[ops[0].body_order()]
        q_dev = torch.from_numpy(np.stack([qm.real, qm.imag], 1).astype(np.float32)).cuda()
        out, _ = emulate_ranks_on_one_device(ops, q_dev, pruned=True)
        outs.append(out.cpu().numpy())
        out, _ = emulate_ranks_on_one_device(ops, q_dev, pruned=True)
        outs.append(out.cpu().numpy())
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_complex_wavenumber_with_wide_leaves(oracle):
    """gate off (kd_max = 0) and no leaf cap: the leaf expansions leave the low-frequency series and run
    the complex Miller recurrence (special.cpp:36-53 with a complex argument), whose normalisation
    once squared a 1e250-scaled iterate (found by scripts/fuzz_parity.py).  Far from the regime the
    truncated expansion is accurate in, so parity is against the oracle's FMM — the reference's
    pipeline in FP64 — not against the direct sum"""
    rng = np.random.default_rng(51)
    n = 6000
    xyz = rng.uniform(-1, 1, size=(n, 3))
    q = charges(n, 51)
    for k, order in ((12 + 0.6j, 4), (6 + 3j, 8)):
        op = HfmmCuda(k=k, order=order, ncrit=64, theta=0.4, kd_max=0.0, leaf_cap=0.0)
        op.set_points(xyz)
        y = op.matvec(q)
        assert np.isfinite(y).all()
        assert op.stats()["m2l_pairs"] > 0
        y64 = oracle.fmm(xyz, k, order, ncrit=64, leaf_cap=0.0, theta=0.4, kd_max=0.0).matvec(q)
        assert rel_l2(y, y64) < 1e-5


def test_deep_tree_of_coincident_points(oracle):
    """clusters of more than ncrit coincident points drive the octree to its last level (21): both builders
    produce the same tree and lists, and the matvec stays accurate"""
    rng = np.random.default_rng(104)
    base = rng.uniform(-1, 1, size=(160, 3))
    xyz = base[rng.integers(0, len(base), 500)]
    q = charges(500, 104)
    op = HfmmCuda(k=1 + 2j, order=10, ncrit=4, theta=0.3, kd_max=2.0, leaf_cap=0.0)
    op.set_points(xyz)
    st = op.stats()
    assert st["max_level"] >= 20 and st["m2l_pairs"] > 0
    y = op.matvec(q)
    assert rel_l2(y, oracle.direct_sum(xyz, q, 1 + 2j)) < 3e-6
    host = HfmmCuda(k=1 + 2j, order=10, ncrit=4, theta=0.3, kd_max=2.0, leaf_cap=0.0, flags=1)
    host.set_points(xyz)
    assert host.stats()["host_tree_used"] == 1
    assert (host.stats()["m2l_pairs"], host.stats()["p2p_pairs"]) == (st["m2l_pairs"], st["p2p_pairs"])
    assert rel_l2(host.matvec(q), y) < 2e-6


def test_device_builder_limit_is_reported_not_hidden(oracle):
    """The device builder's lists grow until they fit (60 % of the free device memory, 32-bit indexing).  A gate that
    forbids every translation turns the near lists into all pairs of leaves: the device builder takes them as long as
    they fit.  Beyond that (here: a 256 MB budget set for the test), HFMM_FLAG_NO_HOST_FALLBACK makes set_points fail
    with the builder's status instead of switching to the host builder; without the flag the switch shows in
    hfmm_cuda_stats::host_tree_used"""
    import os

    from paper_1803_09948_b200.api import HFMM_FLAG_NO_HOST_FALLBACK
    xyz = sphere_points(24000, 3)
    kw = dict(k=50.0, order=4, ncrit=1, kd_max=1e-9, leaf_cap=0.0)
    dev = HfmmCuda(flags=HFMM_FLAG_NO_HOST_FALLBACK, **kw)
    dev.set_points(xyz[:7000])                      # 49 M leaf pairs, 96 x the initial list capacity: still the device builder
    st = dev.stats()
    assert st["host_tree_used"] == 0 and st["p2p_pairs"] == 7000 * 7000 and st["m2l_pairs"] == 0
    q = charges(7000, 3)
    sample = np.arange(0, 7000, 7)
    assert rel_l2(dev.matvec(q)[sample], oracle.direct_sum(xyz[:7000], q, 50.0, targets=sample)) < 5e-6
    del dev
    os.environ["HFMM_DEBUG_LIST_BUDGET_MB"] = "256"
    try:
        strict = HfmmCuda(flags=HFMM_FLAG_NO_HOST_FALLBACK, **kw)
        with pytest.raises(HfmmError) as e:
            strict.set_points(xyz)
        assert e.value.kind == "structural_error" and "interaction lists exceed" in str(e.value)
        strict.set_points(sphere_points(2000, 3))      # the handle stays usable, and says which builder ran
        assert strict.stats()["host_tree_used"] == 0 and strict.stats()["p2p_pairs"] == 2000 * 2000
        loose = HfmmCuda(**kw)
        loose.set_points(xyz[:7000])                    # beyond the (test) budget of the device lists, within the host's reach
        assert loose.stats()["host_tree_used"] == 1 and loose.stats()["p2p_pairs"] == 7000 * 7000
    finally:
        del os.environ["HFMM_DEBUG_LIST_BUDGET_MB"]


def test_m2l_shifts_beyond_the_packed_key_range(oracle):
    """A lattice shift that does not fit the 18-bit fields of the device builder's sort key (a deep leaf translated
    straight from a coarse cell) keeps its pair index as key and is grouped into classes on the host.  The path is
    forced on an ordinary input by lowering the limit: same classes, same pairs, same potentials."""
    import os

    n, k = 12000, 3.0
    xyz, q = plummer_points(n, 31, a=0.05), charges(n, 31)
    ref = HfmmCuda(k=k, order=8, theta=0.4)
    ref.set_points(xyz)
    y_ref, st_ref = ref.matvec(q), ref.stats()
    os.environ["HFMM_DEBUG_SHIFT_LIMIT"] = "6"         # most shifts now take the unpacked path
    try:
        op = HfmmCuda(k=k, order=8, theta=0.4)
        op.set_points(xyz)
    finally:
        del os.environ["HFMM_DEBUG_SHIFT_LIMIT"]
    st = op.stats()
    assert st["host_tree_used"] == 0
    for key in ("m2l_pairs", "p2p_pairs", "m2l_shift_classes", "rotation_tables", "coaxial_tables"):
        assert st[key] == st_ref[key], key
    y = op.matvec(q)
    assert rel_l2(y, y_ref) < 2e-6
    sample = np.arange(0, n, 6)
    assert rel_l2(y[sample], oracle.direct_sum(xyz, q, k, targets=sample)) < 1e-5


def test_partition_of_a_clustered_set_without_leaf_cap():
    """non-uniform points, no leaf cap, no gate: shallow levels interleave owned leaves with interior cells
    nobody owns; the partition must still be describable (only exchanged levels need contiguous rows)"""
    n, k, R = 20000, 2.0, 3
    xyz = plummer_points(n, 5, a=0.02)
    cells_owned = np.zeros(0)
    total = 0
    for r in range(R):
        op = HfmmCuda(k=k, order=6, ncrit=32, theta=0.4, kd_max=0.0, leaf_cap=0.0)
        op.set_partition(r, R)
        op.set_points(xyz)
        p = op.partition()                          # used to raise "owned cells of a level are not contiguous"
        total += int(p.body_count)
        far, near, owner = op.exchange_masks()
        lvl = op.cells()[:, 0]
        for L in range(int(p.level_first), int(p.level_last) + 1):
            mine = np.nonzero((owner == r) & (lvl == L))[0]
            if len(mine):
                assert mine[0] == p.cell_first[L] and len(mine) == p.cell_count[L]
                assert np.array_equal(mine, np.arange(mine[0], mine[0] + len(mine)))
    assert total == n


def test_distinct_targets_and_sources(oracle):
    """execute_plan / fmm_evaluate with a target tree that is not the source tree (traversal.hpp:59-67):
    potentials of the sources at other points — outside the surface, inside it, one ON a source (that pair is
    skipped, kernel.hpp:22) — against the FP64 direct sum; the union tree is reused until the targets change"""
    n, m, k, order = 30000, 5000, 5.0, 10
    xyz, q = sphere_points(n, 31), charges(n, 31)
    rng = np.random.default_rng(32)
    tg = rng.uniform(-1.6, 1.6, size=(m, 3))
    tg[7] = xyz[123]
    op = HfmmCuda(k=k, order=order, ncrit=64)
    op.set_points(xyz)
    y_self = op.matvec(q)
    y = op.evaluate_targets(tg, q)
    exact = oracle.direct_sum(np.vstack([xyz, tg]), np.concatenate([q, np.zeros(m)]), k, targets=np.arange(n, n + m))
    assert rel_l2(y, exact) < 1e-5
    assert abs(y[7] - y_self[123]) < 1e-5 * abs(y_self[123])          # the coincident pair contributes nothing
    t_first = op.evaluate_targets(tg, 2 * q)                          # same targets: the tree is kept, linear in q
    assert rel_l2(t_first, 2 * y) < 1e-6
    assert rel_l2(op.evaluate_targets(tg[:100] + 0.01, q),
                  oracle.direct_sum(np.vstack([xyz, tg[:100] + 0.01]), np.concatenate([q, np.zeros(100)]), k,
                                    targets=np.arange(n, n + 100))) < 1e-5
    assert rel_l2(op.matvec(q), y_self) < 1e-6                         # the handle's own operator is untouched


def test_partition_of_a_clustered_set_without_leaf_cap():
    """Advisor finding (round 1): with leaf_cap = 0 a clustered set puts owned leaves beside unowned interior
    cells on the levels ABOVE the partition cut; those levels are never exchanged and must not trip the
    contiguity check of hfmm_cuda_get_partition.  Three emulated ranks still reproduce the single-domain matvec."""
    import torch

    from paper_1803_09948_b200.distributed import emulate_matvec_on_one_device

    n, k, order = 30000, 3.0, 6
    xyz, q = plummer_points(n, 77, a=0.02), charges(n, 77)
    kw = dict(k=k, order=order, ncrit=48, theta=0.4, kd_max=1.0, leaf_cap=0.0)
    single = HfmmCuda(**kw)
    single.set_points(xyz)
    y1, order_m = single.matvec(q), single.body_order()
    ops = []
    for rank in range(3):
        op = HfmmCuda(**kw)
        op.set_partition(rank, 3)
        op.set_points(xyz)
        p = op.partition()                      # raised HFMM_ERR_STRUCTURAL before the fix
        assert int(p.body_count) > 0
        ops.append(op)
    levels = single.cells()[:, 0]
    assert levels.max() - levels[single.cells()[:, 7] == 0].min() >= 3      # leaves spread over several levels
    qm = q[order_m]
    qd = torch.from_numpy(np.stack([qm.real, qm.imag], 1).astype(np.float32)).cuda()
    y = emulate_matvec_on_one_device(ops, qd).cpu().numpy()
    assert rel_l2(y[:, 0] + 1j * y[:, 1], y1[order_m]) < 3e-6
