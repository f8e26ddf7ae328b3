"""Command-line surface (the reference's SPEC names cmd_solve / cmd_verify
/ cmd_scaling): thin drivers over the C ABI, everything heavy runs in libhfmm_b200.so on the GPU.

  python -m paper_1803_09948_b200 solve   --subdivisions 5 --k 4      sphere scattering, Mie check
  python -m paper_1803_09948_b200 solve   --mesh sphere.msh --k 2      the same on a mesh file (meshio.py)
  python -m paper_1803_09948_b200 solve   ... --out-prefix run1        + run1.report.json, run1.residuals.csv, run1.field.csv
  python -m paper_1803_09948_b200 verify  --orders 1 2 --k 2           Mie error per basis order (SPEC cmd_verify)
  python -m paper_1803_09948_b200 scaling --n 20000 40000 80000        CSV of (N, FMM seconds) + fitted slope (cmd_scaling)
  python -m paper_1803_09948_b200 convert in.msh out.bin               ASCII mesh -> binary blocks (cmd_convert; no GPU)
  python -m paper_1803_09948_b200 partition --ranks 8 --config cfg4    Morton partition statistics (host; no GPU)
  python -m paper_1803_09948_b200 matvec  --config cfg2 [--n N]        one BASELINE FMM configuration
  python -m paper_1803_09948_b200 info                                 library version, device probes
Exit codes follow the SPEC: 0 converged / done, 2 not converged, 64 usage error.

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
    if a.out_prefix:   # SPEC cmd_solve: report JSON, residual CSV, field CSV
        out["residuals"] = [float(v) for v in rep["residuals"]]
        with open(a.out_prefix + ".report.json", "w") as f:
            json.dump(out, f, indent=1)
        with open(a.out_prefix + ".residuals.csv", "w") as f:
            f.write("iteration,relative_residual,seconds,matvec_seconds\n")
            for i, (r, t, m) in enumerate(zip(rep["residuals"], rep["seconds_history"], rep["matvec_seconds_history"])):
                f.write(f"{i + 1},{r:.9e},{t:.6e},{m:.6e}\n")
        with open(a.out_prefix + ".field.csv", "w") as f:
            f.write("theta,re_scattered,im_scattered,re_mie,im_mie\n")
            for t, u, v in zip(th, scat, mie):
                f.write(f"{t:.9f},{u.real:.9e},{u.imag:.9e},{v.real:.9e},{v.imag:.9e}\n")
    return 0 if rep["converged"] else 2


def cmd_verify(a):
    """SPEC cmd_verify: sound-soft sphere against the Mie series, one row per basis order (p-refinement)"""
    import argparse as _ap
    if not a.k > 0:
        print("verify: k must be positive", file=sys.stderr)
        return 64
    rows = []
    for bo in a.orders:
        sub = _ap.Namespace(**{**vars(a), "basis_order": bo, "rules": None, "mesh": None, "out_prefix": None})
        import io, contextlib
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = cmd_solve(sub)
        row = json.loads(buf.getvalue().strip().splitlines()[-1])
        row["basis_order"], row["exit_code"] = bo, rc
        rows.append(row)
    print(json.dumps({"k": a.k, "subdivisions": a.subdivisions, "rows": rows,
                      "errors_decrease": all(x["mie_mismatch_rel_l2"] > y["mie_mismatch_rel_l2"]
                                             for x, y in zip(rows, rows[1:]))}))
    return 0 if all(r["converged"] for r in rows) else 2


def cmd_scaling(a):
    """SPEC cmd_scaling: FMM matvec seconds over a list of N (uniform sphere surface), CSV on stdout; duplicate N
    are averaged (count column); the log-log slope of the fit goes to stderr as JSON"""
    from . import HfmmCuda
    from .workloads import charges, sphere_points

    acc = {}
    for n in a.n:
        xyz, q = sphere_points(n, a.seed), charges(n, a.seed)
        op = HfmmCuda(k=a.k, order=a.order, ncrit=a.ncrit, theta=a.theta, kd_max=1.0, leaf_cap=0.0 if a.no_leaf_cap else -1.0)
        op.set_points(xyz)
        op.matvec(q)
        ts = []
        for _ in range(a.repeat):
            op.matvec(q)
            ts.append(op.stats()["matvec_seconds"])
        acc.setdefault(n, []).append(float(np.median(ts)))
        op.close()
    print("n,fmm_seconds,count")
    for n in sorted(acc):
        print(f"{n},{np.mean(acc[n]):.6e},{len(acc[n])}")
    if len(acc) > 1:
        ns = np.array(sorted(acc), dtype=float)
        t = np.array([np.mean(acc[int(v)]) for v in ns])
        print(json.dumps({"loglog_slope": float(np.polyfit(np.log(ns), np.log(t), 1)[0])}), file=sys.stderr)
    return 0


def cmd_convert(a):
    """SPEC cmd_convert: ASCII mesh -> the reference's binary block format (mesh-io); no GPU"""
    from .meshio import MeshError, read_mesh, write_binary
    try:
        write_binary(read_mesh(a.mesh), a.out)
    except (OSError, ValueError, MeshError) as e:
        print(f"convert: {e}", file=sys.stderr)
        return 1
    return 0


def cmd_partition(a):
    """Morton partition of a BASELINE point set over R ranks (host tree, no GPU): bodies, modelled work and
    the work-balanced cuts (near body pairs + 1600 x M2L pairs) and the bodies each rank then owns — the partition
    the reference's cmd_partition_sim starts its network simulation from (the simulator itself is out of scope)"""
    from .api import debug_partition
    from .workloads import CONFIGS, make_points

    cfg = CONFIGS[a.config]
    n = a.n or min(cfg.n, 262144)
    if a.ranks < 1:
        print("partition: --ranks must be >= 1", file=sys.stderr)
        return 64
    first, count, _, lcut = debug_partition(make_points(cfg, n), cfg.ncrit, cfg.resolved_leaf_cap(), cfg.k, cfg.theta,
                                            cfg.kd_max, a.ranks)
    print(json.dumps({"config": a.config, "points": n, "ranks": a.ranks, "cut_level": int(lcut),
                      "body_first": [int(v) for v in first], "bodies": [int(v) for v in count],
                      "bodies_max_over_mean": float(count.max() / count.mean())}))
    return 0


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
    s.add_argument("--out-prefix", default=None, help="also write <prefix>.report.json, .residuals.csv, .field.csv")
    v = sub.add_parser("verify", help="Mie error of the sphere solve per basis order")
    for flag, typ, dflt in (("--subdivisions", int, 3), ("--radius", float, 1.0), ("--k", float, 2.0), ("--order", int, 10),
                            ("--ncrit", int, 64), ("--theta", float, 0.4), ("--kd-max", float, 1.0), ("--rtol", float, 1e-4),
                            ("--restart", int, 30), ("--max-iterations", int, 1000), ("--observations", int, 37),
                            ("--obs-radius", float, 4.0)):
        v.add_argument(flag, type=typ, default=dflt)
    v.add_argument("--orders", type=int, nargs="+", default=[1, 2], choices=[1, 2])
    v.add_argument("--block-jacobi", action="store_true")
    v.add_argument("--deterministic", action="store_true")
    v.set_defaults(fn=cmd_verify)
    c = sub.add_parser("scaling", help="FMM seconds over a list of N")
    c.add_argument("--n", type=int, nargs="+", required=True)
    c.add_argument("--seed", type=int, default=1)
    c.add_argument("--k", type=float, default=4.0)
    c.add_argument("--order", type=int, default=10)
    c.add_argument("--ncrit", type=int, default=64)
    c.add_argument("--theta", type=float, default=0.4)
    c.add_argument("--repeat", type=int, default=5)
    c.add_argument("--no-leaf-cap", action="store_true", help="leaves bounded by ncrit only (fixed k: the leaf cap fixes the leaf SIZE)")
    c.set_defaults(fn=cmd_scaling)
    cv = sub.add_parser("convert", help="ASCII mesh -> binary mesh")
    cv.add_argument("mesh")
    cv.add_argument("out")
    cv.set_defaults(fn=cmd_convert)
    pt = sub.add_parser("partition", help="Morton partition statistics of a BASELINE point set (host)")
    pt.add_argument("--config", default="cfg2")
    pt.add_argument("--n", type=int, default=None)
    pt.add_argument("--ranks", type=int, default=8)
    pt.set_defaults(fn=cmd_partition)
    i = sub.add_parser("info", help="library version and device probes")
    i.set_defaults(fn=cmd_info)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:      # argparse exits with 2 on a usage error: the SPEC says 64
        return 64 if e.code not in (0, None) else 0
    return a.fn(a)


if __name__ == "__main__":
    sys.exit(main())
