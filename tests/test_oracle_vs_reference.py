"""Live comparison of the oracle restatement with the compiled reference (oracle/_ref).  Skipped
where /root/reference was not available to build it (the committed fixtures cover that case)."""
import numpy as np

from checkers import rel_l2
from paper_1803_09948_b200.workloads import charges, plummer_points, sphere_points


def test_special_and_translation(oracle, ref):
    rng = np.random.default_rng(0)
    for z in rng.uniform(0.01, 20, 12):
        assert np.allclose(oracle.sph_jn(24, z), ref.sph_jn(24, z), rtol=1e-12, atol=1e-300)
        assert np.allclose(oracle.sph_hn(24, z), ref.sph_hn(24, z), rtol=1e-12)
    for _ in range(4):
        t = rng.uniform(-1, 1, 3)
        for sing in (0, 1):
            a, b = oracle.translation_matrix(2.2, t, 7, sing), ref.translation_matrix(2.2, t, 7, sing)
            assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max()


def test_fmm_matvec_and_lists(oracle, ref):
    for xyz, k, order, ncrit, cap, theta in (
            (sphere_points(3000, 1), 2.0, 8, 32, 0.5, 0.4),
            (plummer_points(2500, 2, 0.05), 8.0, 6, 24, 0.125, 0.35)):
        q = charges(len(xyz), 5)
        fo = oracle.fmm(xyz, k, order, ncrit=ncrit, leaf_cap=cap, theta=theta)
        fr = ref.fmm(xyz, k, order, ncrit=ncrit, leaf_cap=cap, theta=theta, threads=2)
        assert fo.counts() == fr.counts()
        assert (fo.cells() == fr.cells()).all() and (fo.body_order() == fr.body_order()).all()
        assert rel_l2(fo.matvec(q), fr.matvec(q)) < 1e-13


def test_simulated_ranks_reproduce_single_domain(oracle, ref):
    # reference let.cpp:320-362 (untested upstream): 2/4 simulated ranks vs 1 domain
    xyz, q = sphere_points(2048, 9), charges(2048, 9)
    y1 = oracle.fmm(xyz, 2.0, 8, ncrit=32, leaf_cap=0.5).matvec(q)
    for nr in (2, 4):
        yd, let_bytes = ref.distributed_matvec(xyz, q, 2.0, 8, nr, ncrit=32, leaf_cap=0.5)
        assert rel_l2(yd, y1) < 1e-8
        assert (let_bytes > 0).all()


def test_repartitioning_loop_pieces(oracle, ref):
    """measure_weights and update_alpha (partition.cpp:143-227): oracle restatement vs the reference"""
    from checkers import update_alpha
    from paper_1803_09948_b200.workloads import plummer_points, sphere_points

    for xyz, k, cap in ((sphere_points(3000, 3), 3.0, 1.0 / 3.0), (plummer_points(2500, 4), 6.0, 0.0)):
        fo = oracle.fmm(xyz, k, 6, ncrit=24, leaf_cap=cap, theta=0.4, kd_max=1.0)
        fr = ref.fmm(xyz, k, 6, ncrit=24, leaf_cap=cap, theta=0.4, kd_max=1.0)
        lo, ro = fo.measure_weights()
        lr, rr = fr.measure_weights()
        assert np.array_equal(lo, lr) and np.array_equal(ro, rr)
        assert lo.sum() == fo.counts()["p2p_body_pairs"]
    rng = np.random.default_rng(5)
    curve = lambda a: (a - 0.7) ** 2 + 1.0
    hist_a, hist_t = [], []
    for step in range(16):       # replay the search the way the driver would: probe, measure, ask again
        a_ref = update_alpha(ref.lib, "ref", hist_a, hist_t) if hist_a else None
        if hist_a:
            a_or = update_alpha(oracle.lib, "ho", hist_a, hist_t)
            assert a_or == a_ref
            nxt = a_ref
        else:
            nxt = 2.0 - 0.6180339887498948 * 2.0
        hist_a.append(nxt)
        hist_t.append(curve(nxt) + 1e-3 * rng.standard_normal())
    assert abs(hist_a[-1] - 0.7) < 0.05
    for _ in range(50):          # arbitrary histories
        m = int(rng.integers(1, 9))
        a, t = rng.uniform(0, 2, m), rng.uniform(1, 2, m)
        assert update_alpha(oracle.lib, "ho", a, t) == update_alpha(ref.lib, "ref", a, t)


def test_mie_series_of_the_package_is_the_reference_s(ref):
    """workloads.mie_soft_sphere (scipy) against oracle::mie_soft_sphere (oracle.cpp:11-59)"""
    from paper_1803_09948_b200.workloads import mie_soft_sphere

    th = np.linspace(0, np.pi, 19)
    for k, r in ((1.0, 1.0), (4.0, 4.0), (12.0, 2.5)):
        want = ref.mie_soft_sphere(1.0, k, np.stack([r + 0 * th, th, 0 * th], 1))
        assert rel_l2(mie_soft_sphere(1.0, k, r, th), want) < 1e-12
    # boundary condition on the sphere: incident + scattered = 0 (test_oracle.cpp:47-57)
    tot = np.exp(1j * 4.0 * np.cos(th)) + mie_soft_sphere(1.0, 4.0, 1.0, th)
    assert np.abs(tot).max() < 1e-10



def test_random_configurations_bitwise(oracle, ref):
    """the oracle's FMM pipeline against the compiled reference on random point sets (coincident points,
    near-collinear sets, single bodies), real and complex wavenumbers, gates on and off, leaf caps:
    identical to the last bit (deterministic accumulation on both sides)"""
    for case in range(14):
        rng = np.random.default_rng([3, case])
        n = int(rng.choice([1, 5, 60, 400, 1500]))
        kind = rng.choice(["cube", "sphere", "dup", "line"])
        if kind == "cube":
            xyz = rng.uniform(-1, 1, (n, 3))
        elif kind == "sphere":
            v = rng.normal(size=(n, 3))
            xyz = v / np.linalg.norm(v, axis=1, keepdims=True)
        elif kind == "dup":
            base = rng.uniform(-1, 1, (max(1, n // 3), 3))
            xyz = base[rng.integers(0, len(base), n)]
        else:
            xyz = np.stack([rng.uniform(0, 3, n), 1e-3 * rng.normal(size=n), np.zeros(n)], 1)
        q = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        k = float(rng.choice([0.3, 1.0, 4.0, 9.0]))
        if rng.uniform() < 0.3:
            k = complex(k, 0.3 * k)
        kw = dict(ncrit=int(rng.choice([4, 16, 64])), theta=float(rng.choice([0.3, 0.5, 0.7])),
                  kd_max=float(rng.choice([0.0, 1.0, 2.0])), leaf_cap=float(rng.choice([0.0, 0.3])))
        order = int(rng.choice([2, 5, 8, 11]))
        yo = oracle.fmm(xyz, k, order, **kw).matvec(q)
        yr = ref.fmm(xyz, k, order, threads=4, **kw).matvec(q)
        assert np.array_equal(yo, yr), (case, n, kind, k, order, kw)


def test_correction_builders_with_complex_wavenumber_bitwise(oracle, ref):
    """build_patch_blocks / build_near_corrections of the oracle against the compiled reference for
    complex wavenumbers, both basis orders, all singularity modes (the device builders are checked
    against the oracle by the GPU tests and scripts/fuzz_bie.py)"""
    from paper_1803_09948_b200.workloads import icosphere_patches

    patches = icosphere_patches(1) * np.array([1.0, 0.8, 1.3])
    for basis_order in (1, 2):
        tables = ref.correction_tables(basis_order)
        for k in (2.0 + 0.6j, 0.5 + 1.0j):
            for mode in (0, 1, 2):
                want = ref.bie(patches, basis_order, k, mode=mode, use_tree=False).corrections()
                got = oracle.build_corrections(patches, tables, k, mode=mode)
                for key in ("patch_block", "block_lu", "block_piv", "near_offset", "near_source", "near_delta"):
                    if want.get(key) is not None:
                        assert np.array_equal(got[key], np.asarray(want[key])), (basis_order, k, mode, key)


def test_symmetric_problem_iteration_count_is_not_robust_in_fp32(oracle, ref):
    """Evidence for the one exemption from "GMRES iteration count +-1" (tests/test_gpu_solver.py,
    tests/test_gpu_dropin.py): on the reference's lat-long sphere with the incident wave along the polar
    axis the all-FP64 GMRES stays inside the invariant subspace of the mesh's rotational symmetry and stops
    early.  The reference's OWN single-precision near field (kernel::Precision::f32, kernel.hpp:43-55 —
    everything else still FP64) breaks that symmetry at the 1e-7 level and takes about twice as many
    iterations; with a generic wave direction the same switch leaves the count where it was.  No device
    code is involved: this is the reference against itself."""
    def counts_for(segments, rings, k, order, direction):
        patches = ref.sphere_mesh(1.0, segments, rings)
        sysr = ref.bie(patches, 1, k, mode=2, use_tree=True, order=order, ncrit=32, theta=0.4, kd_max=1.0)
        xyz, fw = sysr.samples()
        corr = sysr.corrections()
        fr = ref.fmm(xyz, k, order, ncrit=32, leaf_cap=1.0 / k, theta=0.4, kd_max=1.0, threads=8)
        rhs = sysr.rhs(direction)
        out = []
        for f32 in (False, True):
            op = lambda v: oracle.apply_corrections(sysr.ni, corr["patch_block"], corr["near_offset"], corr["near_source"],
                                                    corr["near_delta"], v, fr.matvec(v * fw, f32_p2p=f32))
            _, rep = oracle.gmres(op, rhs, rtol=1e-4, restart=30, max_iterations=400)
            assert rep["converged"]
            out.append(rep["iterations"])
        return out

    axis64, axis32 = counts_for(16, 10, 4.0, 10, (0.0, 0.0, 1.0))        # 864 unknowns; measured 23 -> 43
    gen64, gen32 = counts_for(12, 8, 2.5, 8, (0.36, 0.48, 0.8))          # 504 unknowns; measured 70 -> 70
    assert axis32 >= axis64 + 8, (axis64, axis32)
    assert abs(gen32 - gen64) <= 1, (gen64, gen32)
    assert gen64 > 2 * axis64          # the symmetric solve is the short one although its system is larger
