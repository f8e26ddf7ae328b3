"""The CPU oracle (oracle/hfmm_oracle.c) against the committed fixtures the UNMODIFIED reference
generated (tests/golden/make_golden.py) and against the closed forms the reference's own tests use.
This is what pins the oracle."""
import os

import numpy as np
import pytest

from checkers import rel_l2

G = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(G, name))


def test_special_functions_match_reference_fixtures(oracle):
    g = load("special.npz")
    for z, jn, hn in zip(g["zs"], g["jn"], g["hn"]):
        a = oracle.sph_jn(28, float(z))
        assert np.allclose(a, jn, rtol=1e-13, atol=1e-300)
        assert np.allclose(oracle.sph_hn(28, float(z)), hn, rtol=1e-13)
    for d, y in zip(g["dirs"], g["ynm"]):
        assert np.abs(oracle.ynm(12, d) - y).max() < 1e-14
    for args, v in zip(g["w3_args"], g["w3_vals"]):
        assert abs(oracle.wigner3j(*args) - v) < 1e-13


def test_closed_forms(oracle):
    # reference tests/test_special.cpp:48-123 — j0 = sin z/z, j1, h0 = -i e^{iz}/z
    for z in (0.2, 0.7, 3.3):
        j = oracle.sph_jn(2, z).real
        assert abs(j[0] - np.sin(z) / z) < 1e-14
        assert abs(j[1] - (np.sin(z) / z ** 2 - np.cos(z) / z)) < 1e-13
        assert abs(oracle.sph_hn(0, z)[0] - (-1j * np.exp(1j * z) / z)) < 1e-14
    # Y_0^0, Y_1^0, Y_1^1 with Condon-Shortley phase (tests/test_special.cpp:149-198)
    d = np.array([0.3, -0.4, 0.5])
    r = np.linalg.norm(d)
    y = oracle.ynm(1, d)
    assert abs(y[0] - np.sqrt(1 / (4 * np.pi))) < 1e-15
    assert abs(y[2] - np.sqrt(3 / (4 * np.pi)) * d[2] / r) < 1e-15
    assert abs(y[3] - (-np.sqrt(3 / (8 * np.pi)) * (d[0] + 1j * d[1]) / r)) < 1e-15
    # 3j spot values (tests/test_special.cpp:215-240)
    assert abs(oracle.wigner3j(1, 1, 0, 0, 0, 0) - (-1 / np.sqrt(3))) < 1e-14
    assert abs(oracle.wigner3j(2, 2, 2, 0, 0, 0) - (-np.sqrt(2 / 35))) < 1e-14
    assert oracle.wigner3j(1, 1, 1, 0, 0, 0) == 0


def test_gegenbauer_series_reproduces_kernel(oracle):
    # reference tests/test_special.cpp:281-306: e^{ikR}/(4 pi R) = ik sum_n j_n(kr<) h_n(kr>) sum_m ...
    k, P = 1.3, 30
    x, y = np.array([0.2, -0.1, 0.15]), np.array([1.1, 0.7, -0.9])
    rx, ry = np.linalg.norm(x), np.linalg.norm(y)
    j, h = oracle.sph_jn(P, k * rx), oracle.sph_hn(P, k * ry)
    yx, yy = oracle.ynm(P, x), oracle.ynm(P, y)
    s = 0
    for n in range(P + 1):
        sl = slice(n * n, (n + 1) ** 2)
        s += j[n] * h[n] * np.sum(yy[sl] * np.conj(yx[sl]))
    R = np.linalg.norm(x - y)
    assert abs(1j * k * s - np.exp(1j * k * R) / (4 * np.pi * R)) < 1e-13


def test_translation_matrices_match_reference_fixtures(oracle):
    g = load("translations.npz")
    k, P = float(g["k"]), int(g["order"])
    for t, s, r in zip(g["shifts"], g["singular"], g["regular"]):
        assert np.abs(oracle.translation_matrix(k, t, P, 1) - s).max() <= 1e-12 * np.abs(s).max()
        assert np.abs(oracle.translation_matrix(k, t, P, 0) - r).max() <= 1e-12 * np.abs(r).max()
    M = oracle.p2m(g["p2m_pts"], g["p2m_q"], g["p2m_center"], k, int(g["p2m_order"]))
    assert rel_l2(M, g["p2m_coeff"]) < 1e-13
    for p, v in zip(g["eval_points"], g["eval_multipole"]):
        assert abs(oracle.eval_expansion(0, int(g["p2m_order"]), M, g["p2m_center"], p, k) - v) < 1e-13 * abs(v)


def test_m2l_monopole_column_closed_form(oracle):
    # reference tests/test_fmm.cpp:544-572: L_n^m = i k (-1)^n h_n(k|t|) conj Y_n^m(t^)
    k, P = 2.0, 7
    t = np.array([0.6, -0.3, 0.5])
    T = oracle.translation_matrix(k, t, P, 1)
    h, y = oracle.sph_hn(P, k * np.linalg.norm(t)), oracle.ynm(P, t)
    # monopole moment of a unit charge at the centre: M_0^0 = i k j_0(0) conj Y_0^0 = i k / sqrt(4 pi)
    col = T[:, 0] * (1j * k / np.sqrt(4 * np.pi))
    for n in range(P + 1):
        for m in range(-n, n + 1):
            i = n * (n + 1) + m
            assert abs(col[i] - 1j * k * (-1) ** n * h[n] * np.conj(y[i])) < 1e-12 * abs(h[n])


def test_zero_shift_is_identity(oracle):
    # reference tests/test_fmm.cpp:529-542
    T = oracle.translation_matrix(1.5, [0, 0, 0], 5, 0)
    assert np.abs(T - np.eye(36)).max() < 1e-13


@pytest.mark.parametrize("case", ["pipeline", "sphere", "plummer", "gate_off"])
def test_fmm_pipeline_matches_reference_fixtures(oracle, case):
    g = load("fmm.npz")
    k, order, ncrit, cap, theta, kd = g[f"{case}_params"]
    f = oracle.fmm(g[f"{case}_xyz"], float(k), int(order), ncrit=int(ncrit), leaf_cap=float(cap),
                   theta=float(theta), kd_max=float(kd))
    assert (f.cells() == g[f"{case}_cells"]).all()          # same tree, same numbering
    assert (f.body_order() == g[f"{case}_order"]).all()
    for which, name in ((0, "m2l"), (1, "p2p")):
        a, b = f.pair_set(which), g[f"{case}_{name}"]
        canon = lambda p: p[np.lexsort((p[:, 1], p[:, 0]))]
        assert a.shape == b.shape and (canon(a) == canon(b)).all()
    y = f.matvec(g[f"{case}_q"])
    assert rel_l2(y, g[f"{case}_y"]) < 1e-13
    assert rel_l2(f.matvec(g[f"{case}_q"], f32_p2p=True), g[f"{case}_y_f32p2p"]) < 1e-6
    assert rel_l2(oracle.direct_sum(g[f"{case}_xyz"], g[f"{case}_q"], float(k)), g[f"{case}_direct"]) < 1e-13
    # the reference's own accuracy expectation for its pipeline test (tests/test_fmm.cpp:941-961)
    if case == "pipeline":
        assert rel_l2(y, g[f"{case}_direct"]) < 1e-6


def test_gmres_matches_reference_fixture(oracle):
    g = load("solver.npz")
    A, b = g["A"], g["b"]
    x, rep = oracle.gmres(lambda v: A @ v, b, rtol=1e-6, restart=10, max_iterations=200)
    assert rep["iterations"] == int(g["iterations"])
    assert np.allclose(rep["residuals"], g["residuals"], rtol=1e-9)
    assert rel_l2(x, g["x"]) < 1e-12
    assert abs(rep["final_residual"] - float(g["final_residual"])) < 1e-12


def test_operator_tail_and_preconditioner_match_reference_fixture(oracle):
    # apply_operator = FMM(x * far_weight) + blockdiag x + CSR x  (solver.cpp:314-359)
    g = load("solver.npz")
    xyz, fw, x, ni = g["bie_xyz"], g["bie_far_weight"], g["bie_x"], int(g["bie_ni"])
    k, order = float(g["bie_k"]), int(g["bie_order"])
    f = oracle.fmm(xyz, k, order, ncrit=16, leaf_cap=1.0 / k, theta=0.4, kd_max=1.0)
    y = f.matvec(x * fw)
    y = oracle.apply_corrections(ni, g["bie_patch_block"], g["bie_near_offset"], g["bie_near_source"],
                                 g["bie_near_delta"], x, y)
    assert rel_l2(y, g["bie_y"]) < 1e-12
    # block-Jacobi right preconditioned GMRES reproduces the reference's iteration count exactly
    def op(u):
        v = oracle.block_lu_solve(ni, g["bie_block_lu"], g["bie_block_piv"], u)
        w = f.matvec(v * fw)
        return oracle.apply_corrections(ni, g["bie_patch_block"], g["bie_near_offset"],
                                        g["bie_near_source"], g["bie_near_delta"], v, w)
    u, rep = oracle.gmres(op, g["bie_rhs"], rtol=1e-4, restart=30, max_iterations=200)
    sol = oracle.block_lu_solve(ni, g["bie_block_lu"], g["bie_block_piv"], u)
    assert rep["iterations"] == int(g["bie_iterations"])
    assert rel_l2(sol, g["bie_sol"]) < 1e-9


def _tables(g, prefix):
    keys = ("sample_ref", "far_weight", "near_pts", "near_basis", "self_npts", "self_pts", "self_basis")
    return {k: g[prefix + k] for k in keys}


@pytest.mark.parametrize("case", ["order1", "order2"])
def test_correction_builders_match_reference_fixture(oracle, case):
    """build_patch_blocks / build_near_corrections (solver.cpp:80-230) restated in the oracle against
    arrays the reference produced; the quadrature tables are the reference's (stored with the fixture)"""
    here = os.path.join(os.path.dirname(__file__), "golden")
    if case == "order1":
        g = np.load(os.path.join(here, "solver.npz"))
        patches, k, tables, pre = g["bie_patches"], float(g["bie_k"]), _tables(g, "bie_rule_"), "bie_"
    else:
        g = np.load(os.path.join(here, "corrections_order2.npz"))
        patches, k, tables, pre = g["patches"], float(g["k"]), _tables(g, "rule_"), ""
    got = oracle.build_corrections(patches, tables, k)
    assert np.array_equal(got["xyz"], g[pre + "xyz"])
    for key in ("near_offset", "near_source", "block_piv"):
        assert np.array_equal(got[key], g[pre + key]), key
    for key in ("patch_block", "block_lu", "near_delta"):
        assert np.abs(got[key] - g[pre + key]).max() <= 1e-15 * np.abs(g[pre + key]).max(), key


def test_complex_wavenumber_pipeline_matches_reference_fixture(oracle):
    """k = k_r + i k_i: the oracle's special functions, translation matrices, expansions and near field
    in complex arithmetic against potentials the reference produced (tests/golden/fmm_complex_k.npz)
    and against its dense translation matrices (translations.npz, complex_*)"""
    g = load("fmm_complex_k.npz")
    k = complex(g["k"])
    f = oracle.fmm(g["xyz"], k, int(g["order"]), ncrit=int(g["ncrit"]), leaf_cap=float(g["leaf_cap"]),
                   theta=float(g["theta"]), kd_max=float(g["kd_max"]))
    c = f.counts()
    assert c["m2l_pairs"] == int(g["m2l_pairs"]) and c["p2p_body_pairs"] == int(g["p2p_body_pairs"])
    assert rel_l2(f.matvec(g["q"]), g["y"]) < 1e-13
    assert rel_l2(oracle.direct_sum(g["xyz"], g["q"], k), g["direct"]) < 1e-13
    assert rel_l2(g["y"], g["direct"]) < 1e-6          # the pipeline itself is accurate at this order
    t = load("translations.npz")
    kc, order = complex(t["complex_k"]), int(t["complex_order"])
    for shift, kind, ref_T in zip(t["complex_shifts"], t["complex_kinds"], t["complex_T"]):
        T = oracle.translation_matrix(kc, shift, order, 1 if kind == 0 else 0)
        assert np.abs(T - ref_T).max() <= 1e-13 * np.abs(ref_T).max()
