"""CPU-side checks of the product library (no device): the C ABI surface, configuration errors,
the host tree / dual-tree-traversal builder, and the FP32 translation tables."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from checkers import rel_l2
from paper_1803_09948_b200 import HfmmCuda, HfmmError, api, library_path
from paper_1803_09948_b200.workloads import CONFIGS, icosphere_patches, make_points, plummer_points, sphere_points

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "hfmm_cuda.h")).read()
    names = sorted(set(re.findall(r"\b(hfmm_cuda_[a-z0-9_]+)\s*\(", hdr)))
    assert len(names) >= 20
    lib = C.CDLL(library_path())
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert b"sm_100a" in api.load_library().hfmm_cuda_version()


def test_config_errors_mirror_the_reference(gpu_available):
    # traversal.cpp:16-21 (s >= c >= 1, 0 < theta <= 1), :212-213 (order >= 0): config_error
    for kw in (dict(ncrit=0), dict(ncrit=64, grain=32), dict(theta=0.0), dict(theta=1.5),
               dict(order=-1), dict(order=99), dict(k=-1.0), dict(wave_i=float("nan")), dict(wave_i=9.0)):
        args = dict(k=1.0, order=4)
        args.update(kw)
        with pytest.raises(HfmmError) as e:
            HfmmCuda(**args)
        assert e.value.kind == "config_error"
    if not gpu_available:
        # no device: the product refuses loudly instead of falling back to a CPU path
        with pytest.raises(HfmmError) as e:
            HfmmCuda(k=1.0, order=4)
        assert e.value.kind == "device_error"


def _canon_cells(c):
    a = c[:, :6].astype(np.int64)
    return a[np.lexsort(a.T[::-1])]


def _geo_pairs(cells, pairs):
    key = lambda c: ((cells[c, 0].astype(np.int64) << 57) | (cells[c, 1].astype(np.int64) << 38)
                     | (cells[c, 2].astype(np.int64) << 19) | cells[c, 3].astype(np.int64))
    a = np.stack([key(pairs[:, 0]), key(pairs[:, 1])], 1)
    return a[np.lexsort((a[:, 1], a[:, 0]))]


@pytest.mark.parametrize("name,xyz,k,ncrit,cap,theta,kd", [
    ("sphere", sphere_points(6000, 3), 4.0, 32, 0.25, 0.4, 1.0),
    ("plummer", plummer_points(5000, 4, 0.05), 8.0, 16, 0.125, 0.35, 1.0),
    ("nocap_gate", sphere_points(3000, 5), 4.0, 64, 0.0, 0.4, 1.0),
    ("gate_off", sphere_points(3000, 6), 1.0, 24, 0.0, 0.5, 0.0),
])
def test_host_tree_and_lists_equal_the_oracle(oracle, name, xyz, k, ncrit, cap, theta, kd):
    d = api.debug_host_tree(xyz, ncrit, cap, k, theta, kd)
    f = oracle.fmm(xyz, k, 2, ncrit=ncrit, leaf_cap=cap, theta=theta, kd_max=kd)
    assert (_canon_cells(d["cells"]) == _canon_cells(f.cells())).all()   # same cell set
    assert (d["order"] == f.body_order()).all()                          # same Morton order
    for which, nm in ((0, "m2l"), (1, "p2p")):                           # same pair sets
        assert (_geo_pairs(d["cells"], d[nm]) == _geo_pairs(f.cells(), f.pair_set(which))).all()
    # level-order invariants of the device layout: parents precede children, siblings contiguous
    cells = d["cells"]
    lv = cells[:, 0].astype(int)
    assert (np.diff(lv) >= 0).all()
    for c in np.nonzero(cells[:, 7])[0][:200]:
        ch = cells[cells[c, 6]:cells[c, 6] + cells[c, 7]]
        assert (ch[:, 0] == cells[c, 0] + 1).all()
        assert ch[:, 5].sum() == cells[c, 5] and ch[0, 4] == cells[c, 4]


@pytest.mark.parametrize("order", [4, 10, 14])
def test_factored_tables_compose_to_the_dense_operator(oracle, order):
    """R^H C R built from the FP32 device tables == the reference's dense translation matrix
    (expansion.cpp:95-124), for M2L (singular) and M2M/L2L (regular) shifts, any level scales."""
    rng = np.random.default_rng(order)
    k = 3.0
    shifts = [rng.uniform(-0.4, 0.4, 3), np.array([0, 0, 0.31]), np.array([0, 0, -0.31]),
              np.array([0.2, 0, 0]), np.array([0.0625, -0.0625, 0.0625])]
    for t in shifts:
        for kind, sing, (ss, sd) in ((0, 1, (0.3, 0.15)), (1, 0, (0.2, 0.4))):
            ref_T = oracle.translation_matrix(k, t, order, sing)
            T = api.debug_compose_translation(order, k, t, kind, ss, sd)
            assert np.abs(T - ref_T).max() <= 5e-7 * np.abs(ref_T).max(), (order, t, kind)


def test_factored_tables_for_a_complex_wavenumber():
    """the same composition for k = k_r + i k_i against dense matrices the reference produced
    (tests/golden/translations.npz, complex_* entries; translation_matrix takes a complex k throughout)"""
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "translations.npz"))
    k = complex(g["complex_k"])
    order = int(g["complex_order"])
    for t, kind, ref_T in zip(g["complex_shifts"], g["complex_kinds"], g["complex_T"]):
        ss, sd = (0.3, 0.15) if kind == 0 else (0.2, 0.4)
        T = api.debug_compose_translation(order, k, t, int(kind), ss, sd)
        assert np.abs(T - ref_T).max() <= 5e-7 * np.abs(ref_T).max(), (t, kind)


def test_workload_generators():
    c = CONFIGS["cfg2"]
    assert c.n == 1_048_576 and c.k == 4.0 and c.order == 12 and c.resolved_leaf_cap() == 0.25
    p = make_points(CONFIGS["cfg1"], 1000)
    assert np.allclose(np.linalg.norm(p, axis=1), 1.0)
    assert (make_points(CONFIGS["cfg1"], 1000) == p).all()                # seeded
    pl = plummer_points(2000, 1, 0.05)
    assert pl.min() >= 0 and pl.max() <= 1
    ico = icosphere_patches(2)
    assert ico.shape == (320, 6, 3) and np.allclose(np.linalg.norm(ico, axis=2), 1.0)
    # config 3: 7 subdivisions -> 327,680 triangles -> 983,040 order-1 unknowns
    assert 20 * 4 ** 7 == 327_680


def test_update_alpha_matches_the_oracle_and_converges(oracle):
    """hfmm_partition_update_alpha (host logic, no GPU): the reference's golden-section replay
    (partition.cpp:175-227) — same answers as the oracle restatement on arbitrary histories, and the
    driver loop homes in on the minimum of a noisy runtime curve"""
    from checkers import update_alpha as checker_update_alpha
    from paper_1803_09948_b200.api import HfmmError, update_alpha

    rng = np.random.default_rng(17)
    for _ in range(200):
        m = int(rng.integers(1, 10))
        amax = float(rng.choice([0.5, 2.0, 64.0]))
        a, t = rng.uniform(0, amax, m), rng.uniform(1, 2, m)
        if rng.random() < 0.5:   # histories that follow the search path exercise the deeper branches
            a[0] = amax - 0.6180339887498948 * amax
            if m > 1:
                a[1] = 0.6180339887498948 * amax
        assert update_alpha(a, t, amax) == checker_update_alpha(oracle.lib, "ho", a, t, amax)
    hist_a, hist_t = [], []
    alpha = 2.0 - 0.6180339887498948 * 2.0
    for _ in range(14):
        hist_a.append(alpha)
        hist_t.append((alpha - 1.3) ** 2 + 0.5)
        alpha = update_alpha(hist_a, hist_t, 2.0)
    assert abs(alpha - 1.3) < 0.02
    for bad in (([], [], 2.0), ([0.5], [1.0], 0.0)):
        with pytest.raises(HfmmError) as e:
            update_alpha(*bad)
        assert e.value.kind == "config_error"


def test_mesh_ingestion_reads_the_reference_s_files(tmp_path):
    """meshio.py against files the reference wrote (tests/golden/sphere_8x5.msh / .hfmm, mesh_io.cpp):
    both encodings carry the same elements, the writers reproduce the files byte for byte, rank blocks
    tile the mesh, and the parser's refusals carry the reference's error kinds"""
    from paper_1803_09948_b200 import meshio

    here = os.path.join(os.path.dirname(__file__), "golden")
    g, b = os.path.join(here, "sphere_8x5.msh"), os.path.join(here, "sphere_8x5.hfmm")
    a, skipped = meshio.read_gmsh(g)
    assert a.shape == (64, 6, 3) and skipped == 0
    assert np.array_equal(a, meshio.read_binary(b)) and np.array_equal(a, meshio.read_mesh(b))
    assert np.allclose(np.linalg.norm(a.reshape(-1, 3), axis=1), 1.0, atol=1e-12)
    meshio.write_gmsh(a, tmp_path / "w.msh")
    assert meshio.write_binary(a, tmp_path / "w.hfmm") == 32 + 144 * 64
    assert open(tmp_path / "w.msh").read() == open(g).read()
    assert open(tmp_path / "w.hfmm", "rb").read() == open(b, "rb").read()
    parts = [meshio.read_binary(b, r, 5) for r in range(5)]
    assert [len(p) for p in parts] == [(r + 1) * 64 // 5 - r * 64 // 5 for r in range(5)]
    assert np.array_equal(np.concatenate(parts), a)
    # other element types are skipped and counted; unknown sections are skipped
    text = open(g).read().replace("$Elements\n64\n", "$Elements\n65\n900 15 2 0 0 1\n")
    text = text.replace("$Nodes", "$Comments\nanything\n$EndComments\n$Nodes", 1)
    (tmp_path / "mixed.msh").write_text(text)
    a2, skipped2 = meshio.read_gmsh(tmp_path / "mixed.msh")
    assert skipped2 == 1 and np.array_equal(a2, a)
    for bad, kind in ((text.replace("2.2 0 8", "4.1 0 8"), "format_error"),
                      (text.replace("$EndNodes", "$EndNods"), "parse_error"),
                      (open(g).read().replace(" 9 2 0 0 1 ", " 9 2 0 0 99999 ", 1), "structural_error")):
        (tmp_path / "bad.msh").write_text(bad)
        with pytest.raises(meshio.MeshError) as e:
            meshio.read_gmsh(tmp_path / "bad.msh")
        assert e.value.kind == kind, (kind, str(e.value))
    (tmp_path / "bad.hfmm").write_bytes(b"NOTAMESH" + bytes(24))
    with pytest.raises(meshio.MeshError) as e:
        meshio.read_binary(tmp_path / "bad.hfmm")
    assert e.value.kind == "format_error"
    with pytest.raises(meshio.MeshError) as e:
        meshio.read_binary(b, 3, 3)
    assert e.value.kind == "config_error"



def test_cli_host_verbs(tmp_path):
    """SPEC cmd_convert (idempotent, missing file -> nonzero exit), usage error -> 64, partition statistics: the
    verbs of python -m paper_1803_09948_b200 that need no GPU"""
    from paper_1803_09948_b200.__main__ import main
    from paper_1803_09948_b200.meshio import read_mesh, write_gmsh
    from paper_1803_09948_b200.workloads import icosphere_patches

    patches = icosphere_patches(1)
    msh, b1, b2 = (str(tmp_path / f) for f in ("s.msh", "a.bin", "b.bin"))
    write_gmsh(patches, msh)
    assert main(["convert", msh, b1]) == 0 and main(["convert", b1, b2]) == 0
    assert open(b1, "rb").read() == open(b2, "rb").read()                      # convert twice -> identical bytes
    assert len(open(b1, "rb").read()) == 32 + 144 * len(patches)               # SPEC: 32 + 144 E bytes
    assert np.allclose(read_mesh(b1), patches, rtol=0, atol=1e-15)
    assert main(["convert", str(tmp_path / "missing.msh"), b2]) != 0
    assert main(["solve", "--no-such-flag"]) == 64
    assert main(["partition", "--config", "cfg4", "--n", "20000", "--ranks", "4"]) == 0
