"""Command-line surface (the reference's SPEC names cmd_solve / cmd_verify
/ cmd_scaling): thin drivers over the C ABI, everything heavy runs in libhfmm_b200.so on the GPU.

  python -m paper_1803_09948_b200 solve   --subdivisions 5 --k 4      sphere scattering, Mie check
  python -m paper_1803_09948_b200 solve   --mesh sphere.msh --k 2      the same on a mesh file (meshio.py)
  python -m paper_1803_09948_b200 matvec  --config cfg2 [--n N]        one BASELINE FMM configuration
  python -m paper_1803_09948_b200 info                                 library version, device probes

The quadrature tables of the correction builders are the reference's (geometry.cpp); the package ships
them for basis orders 1 and 2 (data/quadrature_rules.npz, --basis-order), --rules reads other ones from a
.npz with the keys sample_ref, far_weight, near_pts, near_basis, self_npts, self_pts, self_basis."""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

RULE_KEYS = ("sample_ref", "far_weight", "near_pts", "near_basis", "self_npts", "self_pts", "self_basis")


def _load_rules(path: str):
    g = np.load(path)
    prefix = "bie_rule_" if "bie_rule_sample_ref" in g.files else ("rule_" if "rule_sample_ref" in g.files else "")
    return {k: g[prefix + k] for k in RULE_KEYS}


def cmd_solve(a):
    from . import HfmmCuda
    from .api import HFMM_FLAG_DETERMINISTIC
    from .workloads import icosphere_patches, mie_soft_sphere, patch_samples

    from .workloads import quadrature_tables
    tables = _load_rules(a.rules) if a.rules else quadrature_tables(a.basis_order)
    if a.mesh:       # GMSH MSH 2.2 ASCII or the reference's binary block format (meshio.py)
        from .meshio import read_mesh
        patches = read_mesh(a.mesh)
        a.radius = float(np.linalg.norm(patches.reshape(-1, 3), axis=1).max())   # Mie check: a sphere about the origin
    else:
        patches = icosphere_patches(a.subdivisions, a.radius)
    xyz = patch_samples(patches, tables["sample_ref"])
    op = HfmmCuda(k=a.k, order=a.order, ncrit=a.ncrit, theta=a.theta, kd_max=a.kd_max, leaf_cap=-1.0,
                  flags=HFMM_FLAG_DETERMINISTIC if a.deterministic else 0)
    t0 = time.perf_counter(); op.set_points(xyz); t_tree = time.perf_counter() - t0
    t0 = time.perf_counter(); nnz = op.build_corrections(patches, tables, mode=2, fetch=False); t_corr = time.perf_counter() - t0
    rhs = op.assemble_rhs((0.0, 0.0, 1.0))          # plane wave e^{ikz} (reference assemble_rhs)
    t0 = time.perf_counter()
    x, rep = op.gmres(rhs, rtol=a.rtol, restart=a.restart, max_iterations=a.max_iterations,
                      precondition=a.block_jacobi)
    t_solve = time.perf_counter() - t0
    th = np.linspace(0, np.pi, a.observations)
    r_obs = a.obs_radius * a.radius
    obs = np.stack([r_obs * np.sin(th), 0 * th, r_obs * np.cos(th)], 1)
    scat = -op.evaluate_field(x, obs)
    mie = mie_soft_sphere(a.radius, a.k, r_obs, th)
    out = {"triangles": int(len(patches)), "unknowns": int(len(xyz)), "k": a.k, "order": a.order,
           "near_correction_nnz": int(nnz), "tree_and_lists_seconds": t_tree, "corrections_seconds": t_corr,
           "iterations": int(rep["iterations"]), "converged": bool(rep["converged"]),
           "final_residual": float(rep["final_residual"]), "solve_seconds": t_solve,
           "mie_mismatch_rel_l2": float(np.linalg.norm(scat - mie) / np.linalg.norm(mie))}
    print(json.dumps(out))
    return 0 if rep["converged"] else 2


def cmd_matvec(a):
    from . import HfmmCuda
    from .api import HFMM_FLAG_DETERMINISTIC
    from .workloads import CONFIGS, charges, make_points

    cfg = CONFIGS[a.config]
    n = a.n or cfg.n
    xyz, q = make_points(cfg, n), charges(n, cfg.seed)
    op = HfmmCuda(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max, leaf_cap=cfg.leaf_cap,
                  flags=HFMM_FLAG_DETERMINISTIC if a.deterministic else 0)
    op.set_points(xyz)
    y = op.matvec(q)
    t0 = time.perf_counter()
    for _ in range(a.repeat):
        y = op.matvec(q)
    ms = (time.perf_counter() - t0) / a.repeat * 1e3
    # FP64 direct sum on a few targets (numpy, host)
    rng = np.random.default_rng(0)
    tg = rng.choice(n, size=min(a.check, n), replace=False)
    exact = np.zeros(len(tg), dtype=np.complex128)
    for i, t in enumerate(tg):
        d = np.linalg.norm(xyz - xyz[t], axis=1)
        keep = d > 0          # coincident points (the target itself) are skipped, as in the reference
        exact[i] = np.sum(np.exp(1j * cfg.k * d[keep]) / (4 * np.pi * d[keep]) * q[keep])
    st = op.stats()
    print(json.dumps({"config": a.config, "points": n, "ms_per_matvec_host_to_host": ms,
                      "rel_l2_vs_direct_sum": float(np.linalg.norm(y[tg] - exact) / np.linalg.norm(exact)),
                      "m2l_pairs": st["m2l_pairs"], "p2p_body_pairs": st["p2p_body_pairs"],
                      "setup_seconds": st["setup_seconds"]}))
    return 0


def cmd_info(a):
    from . import HfmmCuda
    from .api import load_library

    lib = load_library()
    out = {"library": lib.hfmm_cuda_version().decode()}
    try:
        op = HfmmCuda(k=1.0, order=4)
        out["fp32_peak_tflops"] = op.fp32_peak_tflops()
    except Exception as e:  # no device: the library refuses, there is no CPU path
        out["device"] = str(e)
    print(json.dumps(out))
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_1803_09948_b200", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve", help="plane-wave scattering off a sound-soft sphere, checked against the Mie series")
    s.add_argument("--subdivisions", type=int, default=5)
    s.add_argument("--mesh", default=None, help="mesh file (MSH 2.2 ASCII with 6-node triangles, or HFMMMESH binary) instead of the icosphere")
    s.add_argument("--radius", type=float, default=1.0)
    s.add_argument("--k", type=float, default=4.0)
    s.add_argument("--order", type=int, default=12)
    s.add_argument("--ncrit", type=int, default=64)
    s.add_argument("--theta", type=float, default=0.4)
    s.add_argument("--kd-max", type=float, default=1.0)
    s.add_argument("--rtol", type=float, default=1e-4)
    s.add_argument("--restart", type=int, default=30)
    s.add_argument("--max-iterations", type=int, default=1000)
    s.add_argument("--block-jacobi", action="store_true")
    s.add_argument("--deterministic", action="store_true", help="ordered accumulation: bitwise reproducible runs")
    s.add_argument("--observations", type=int, default=37)
    s.add_argument("--obs-radius", type=float, default=4.0, help="in sphere radii")
    s.add_argument("--basis-order", type=int, default=1, choices=[1, 2], help="Lagrange basis of the shipped tables")
    s.add_argument("--rules", default=None, help=".npz with other quadrature tables (default: the shipped ones)")
    s.set_defaults(fn=cmd_solve)
    m = sub.add_parser("matvec", help="one BASELINE FMM configuration, checked against an FP64 direct sum")
    m.add_argument("--config", default="cfg2")
    m.add_argument("--n", type=int, default=None)
    m.add_argument("--repeat", type=int, default=5)
    m.add_argument("--deterministic", action="store_true", help="ordered accumulation: bitwise reproducible runs")
    m.add_argument("--check", type=int, default=64)
    m.set_defaults(fn=cmd_matvec)
    i = sub.add_parser("info", help="library version and device probes")
    i.set_defaults(fn=cmd_info)
    a = ap.parse_args(argv)
    return a.fn(a)


if __name__ == "__main__":
    sys.exit(main())
