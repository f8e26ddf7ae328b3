#!/usr/bin/env python
"""bench.py — the FMM Helmholtz matvec (BASELINE.json's hot path) on N B200s of one node.

    python bench.py --gpus 1 --steps K --warmup W              # this repo's CUDA path
    python bench.py --impl reference --gpus 1 --steps K ...     # the reference's CPU path, same metric
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...   # N > 1

A "step" is one FMM matvec (P2M, M2M, M2L, L2L, L2P, P2P) over one synthetic charge vector.
N = 1 runs BASELINE.json configs[1] (1,048,576 points on the unit sphere, k = 4, P = 12,
ncrit = 64, theta = 0.4; kd_max = 1 and leaf cap kd_max/k as the reference's solver path).
Prints ONE JSON line (rank 0).  `value` is device-resident throughput (operands in HBM, CUDA
events on the library's stream); `e2e` is the same matvec through the C ABI with pinned HOST
buffers, host<->device copies inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1803_09948_b200.workloads import CONFIGS, charges, make_points  # noqa: E402

METRIC = "fmm_matvec_throughput"
UNIT = "Mpoints/s"


def m2l_flops_per_pair(order: int) -> tuple[int, int]:
    """(executed, dense-equivalent) FP32 flops of one M2L cell pair:
    executed = 2 flop x [2 rotations x 2 sum_n ((n+1)^2 + n^2) real-x-complex MACs (folded +-m blocks)
                         + 4 sum_m (P+1-|m|)^2 complex MACs (coaxial step)];  dense = 8 (P+1)^4."""
    rot = sum((n + 1) ** 2 + n ** 2 for n in range(order + 1))
    coax = sum((order + 1 - abs(m)) ** 2 for m in range(-order, order + 1))
    return 2 * (2 * 2 * rot + 4 * coax), 8 * (order + 1) ** 4


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms while the timed regions run"""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.samples, self.reasons, self.proc = [], set(), None
        self.index = index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.proc.stdout:
            f = [x.strip() for x in line.split(",")]
            try:
                self.samples.append((float(f[0]), float(f[1])))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    self.reasons.add(nm)

    def stop(self) -> dict:
        if self.proc:
            self.proc.terminate()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        loaded = [s for s, _ in self.samples]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": self.samples[0][1],
                "reasons": sorted(self.reasons), "samples": len(loaded)}


def cpu_reference_arm(cfg, n_sample: int, steps: int, warmup: int, budget_s: float = 0.0) -> dict:
    """The reference's own CPU implementation (oracle/_ref when it compiled, else our C port) on a
    bounded sample of the workload, all host threads.  With a budget the number of timed matvecs is
    cut so that the whole arm ends inside it (the first matvec is always run)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from checkers import Oracle, Ref, have_ref

    kind = "reference" if have_ref() else "port"
    eng = Ref() if have_ref() else Oracle()
    n_sample = min(n_sample, cfg.n)
    xyz, q = make_points(cfg, n_sample), charges(n_sample, cfg.seed)
    cores = os.cpu_count() or 1
    f = eng.fmm(xyz, cfg.k, cfg.order, ncrit=cfg.ncrit, leaf_cap=cfg.resolved_leaf_cap(),
                theta=cfg.theta, kd_max=cfg.kd_max, threads=cores)
    t_start = time.perf_counter()
    for _ in range(warmup):
        f.matvec(q)
    t0 = time.perf_counter()
    done = 0
    while done < max(steps, 1):
        f.matvec(q)
        done += 1
        per = (time.perf_counter() - t_start) / (warmup + done)
        if budget_s and time.perf_counter() - t_start + per > budget_s:
            break
    dt = (time.perf_counter() - t0) / done
    return {"value": n_sample / dt * 1e-6, "unit": UNIT, "cores": cores, "kind": kind,
            "seconds_per_matvec": dt, "steps": done,
            "sample": f"{n_sample} of {cfg.n} points, same distribution/k/P/ncrit/theta/kd_max/cap; "
                      f"{done} matvec(s) after {warmup} warm-up; FP64, std::thread x{cores}"
                      if kind == "reference" else
                      f"{n_sample} of {cfg.n} points; C port with OpenMP x{cores}"}


def run_reference(args, cfg, rank: int):
    if rank != 0:
        return
    # The sample is a quarter of the points (262,144 of cfg 2's 1,048,576): the reference rebuilds one
    # dense translation matrix per distinct shift on every call (traversal.cpp:252-256), a cost that
    # does not shrink with the sample (6 s per matvec on 16 cores), so a small sample would understate
    # its throughput: measured 0.0026 / 0.0052 / 0.0059 Mpoints/s at 16 k / 131 k / 262 k points.
    # One matvec takes ~45 s on 16 cores; the arm is budgeted to ~170 s: at most one warm-up and as
    # many of the requested timed matvecs as fit.
    warmup = min(args.warmup, 1)
    base = cpu_reference_arm(cfg, args.ref_arm_points, max(1, min(args.steps, 7)), warmup, budget_s=170.0)
    steps = base["steps"]
    line = {
        "impl": "reference", "metric": METRIC, "value": base["value"], "unit": UNIT,
        "n_gpus": args.gpus, "steps": steps, "warmup": warmup,
        "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": base["seconds_per_matvec"] * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg, cfg.n, args.gpus), "cpu_baseline": base,
        "e2e": {"value": base["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def workload_config(cfg, n_total: int, gpus: int) -> dict:
    return {"workload": f"BASELINE.json configs[{ {'cfg2': 1, 'cfg1': 0, 'cfg4': 3, 'cfg5': 4, 'cfg5_per_gpu': 4}.get(cfg.name, '?') }]: "
                        f"FMM Helmholtz matvec, {n_total} points {cfg.distribution}",
            "n_points": n_total, "k": cfg.k, "order": cfg.order, "ncrit": cfg.ncrit,
            "theta": cfg.theta, "kd_max": cfg.kd_max, "leaf_cap": cfg.resolved_leaf_cap(),
            "parallelism": f"morton{gpus}" if gpus > 1 else "single",
            "l2": "working set (expansions + lists + bodies) > 126 MB L2; no explicit flush"}


def run_single(args, cfg):
    import torch

    from paper_1803_09948_b200 import HfmmCuda

    torch.cuda.set_device(0)
    n = args.n or cfg.n
    xyz, q = make_points(cfg, n), charges(n, cfg.seed)
    op = HfmmCuda(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max,
                  leaf_cap=cfg.leaf_cap, device=0)
    op.set_points(xyz)
    setup_cold = op.stats()["setup_seconds"]   # includes the first launches' module loads
    setup_warm = []
    for _ in range(3):  # median of three: cudaMalloc / cudaFree of ~50 buffers makes a single call noisy
        op.set_points(xyz)
        setup_warm.append(op.stats()["setup_seconds"])
    st0 = op.stats()

    # ---- device-resident steps: operands already in HBM (complex FP32, caller order)
    q_dev = torch.from_numpy(np.stack([q.real, q.imag], 1).astype(np.float32)).cuda()
    out_dev = torch.empty_like(q_dev)
    torch.cuda.synchronize()
    sampler = ClockSampler(0)
    sampler.start()
    for _ in range(args.warmup):
        op.matvec_device(q_dev.data_ptr(), out_dev.data_ptr())
    op.sync()
    torch.cuda.synchronize()
    op.timer_record(0)
    for _ in range(args.steps):
        op.matvec_device(q_dev.data_ptr(), out_dev.data_ptr())
    op.timer_record(1)
    ms_total = op.timer_elapsed_ms(0, 1)
    op.sync()
    torch.cuda.synchronize()
    ms_step = ms_total / args.steps

    # ---- per-kernel durations, CUDA events on the launching streams, averaged over K more steps
    acc = {k: 0.0 for k in ("p2p", "p2m", "m2m", "m2l", "l2l", "l2p", "matvec")}
    for _ in range(args.steps):
        op.matvec_device(q_dev.data_ptr(), out_dev.data_ptr())
        st = op.stats()
        for k in acc:
            acc[k] += st[f"{k}_seconds"]
    kern = {k: v / args.steps for k, v in acc.items()}
    # the near field runs beside M2L on the same SMs (co-resident CTAs), so its event interval above
    # is stretched over the whole M2L launch: kernel-alone durations come from a second handle that
    # serialises the near field behind the far field (HFMM_FLAG_PHASE_TIMERS)
    from paper_1803_09948_b200.api import HFMM_FLAG_PHASE_TIMERS
    ops = HfmmCuda(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max,
                   leaf_cap=cfg.leaf_cap, device=0, flags=HFMM_FLAG_PHASE_TIMERS)
    ops.set_points(xyz)
    alone = {k: 0.0 for k in acc}
    for it in range(args.steps + 1):
        ops.matvec_device(q_dev.data_ptr(), out_dev.data_ptr())
        sts = ops.stats()
        if it:  # the first one warms up
            for k in alone:
                alone[k] += sts[f"{k}_seconds"]
    alone = {k: v / args.steps for k, v in alone.items()}
    del ops

    # ---- end to end through the C ABI with pinned host buffers
    qh = torch.from_numpy(q.copy()).pin_memory()
    oh = torch.empty(n, dtype=torch.complex128).pin_memory()
    for _ in range(min(args.warmup, 2)):
        op.matvec_into(qh.data_ptr(), oh.data_ptr())
    t0 = time.perf_counter()
    for _ in range(args.steps):
        op.matvec_into(qh.data_ptr(), oh.data_ptr())
    e2e_s = (time.perf_counter() - t0) / args.steps
    checksum = float(torch.view_as_real(oh).abs().sum())
    clocks = sampler.stop()

    fp32_peak = op.fp32_peak_tflops()
    nominal = 148 * 128 * 2 * 1.965e9 * 1e-12
    ex, dense = m2l_flops_per_pair(cfg.order)
    m2l_tf = st0["m2l_pairs"] * ex / kern["m2l"] * 1e-12 if kern["m2l"] > 0 else 0.0
    m2l_tf_alone = st0["m2l_pairs"] * ex / alone["m2l"] * 1e-12 if alone["m2l"] > 0 else 0.0
    p2p_tf = st0["p2p_body_pairs"] * 24 / alone["p2p"] * 1e-12 if alone["p2p"] > 0 else 0.0
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm = peaks.get("hbm_gbs", 6650.0)
    stride = (cfg.order + 1) ** 2
    tree_bytes = {  # algorithmic bytes of the HBM-bound passes
        "p2m": n * 20 + st0["n_leaves"] * 8 * stride,
        "l2p": n * 20 + st0["n_leaves"] * 8 * stride,
        "m2m": st0["n_cells"] * 2 * 8 * stride, "l2l": st0["n_cells"] * 2 * 8 * stride}

    cpu = cpu_reference_arm(cfg, args.ref_points, 1, 0) if not args.no_cpu_baseline else None
    line = {
        "metric": METRIC, "value": n / ms_step * 1e-3, "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": workload_config(cfg, n, 1),
        "e2e": {"value": n / e2e_s * 1e-6, "unit": UNIT, "ms_per_step": e2e_s * 1e3,
                "h2d_bytes_per_step": n * 16, "d2h_bytes_per_step": n * 16, "checksum": checksum},
        "gpu_launches": int(st0["kernel_launches"] or op.stats()["kernel_launches"]) * args.steps,
        "roofline": {
            "kernel": "translate_kernel (M2L launch)", "bound": "fp32",
            "achieved": m2l_tf, "peak": fp32_peak, "unit": "TFLOP/s",
            "frac": m2l_tf / fp32_peak if fp32_peak else None,
            "peak_source": "higher of the FFMA and FFMA2 (fma.rn.f32x2) probes in this run (MEASURED_PEAKS.json has no FP32 entry); "
                           f"nominal 148x128x2x1.965 GHz = {nominal:.1f}",
            "flops_per_unit": ex, "units_per_launch": st0["m2l_pairs"],
            "dense_equivalent_tflops": st0["m2l_pairs"] * dense / kern["m2l"] * 1e-12 if kern["m2l"] else None,
            # the same launch counted with UNFOLDED rotation blocks, (2n+1)^2 instead of (n+1)^2 + n^2
            "unfolded_rotation_equivalent_tflops": st0["m2l_pairs"] * 2 * (
                4 * sum((2 * j + 1) ** 2 for j in range(cfg.order + 1))
                + 4 * sum((cfg.order + 1 - abs(m)) ** 2 for m in range(-cfg.order, cfg.order + 1))
            ) / kern["m2l"] * 1e-12 if kern["m2l"] else None,
            "ms_per_launch": kern["m2l"] * 1e3,
            # the same launch timed alone (near field serialised behind it): in the timed region one
            # near-field CTA shares every SM with the two M2L CTAs
            "ms_per_launch_alone": alone["m2l"] * 1e3, "achieved_alone": m2l_tf_alone,
            "frac_alone": m2l_tf_alone / fp32_peak if fp32_peak else None,
            # dram__bytes_read + dram__bytes_write of this launch from the committed ncu --set full
            # capture of the same configuration (profiles/r01_ncu_final_cfg2_full.txt:
            # 11.12 GB read + 5.57 GB written); algorithmic bytes
            # are pairs x 2 x 8 (P+1)^2 (one source row read, one destination row reduced)
            "traffic": 16.69e9 if (cfg.name == "cfg2" and n == cfg.n) else None,
            "algorithmic_bytes": st0["m2l_pairs"] * 2 * 8 * (cfg.order + 1) ** 2},
        # kernel-alone durations (near field serialised behind the far field); "ms_in_step" is the event
        # interval inside the timed region, where P2P is co-resident with M2L
        "kernels": {
            "p2p": {"ms": alone["p2p"] * 1e3, "ms_in_step": kern["p2p"] * 1e3, "tflops_24flop_per_pair": p2p_tf,
                    "frac_of_fp32_peak": p2p_tf / fp32_peak if fp32_peak else None,
                    "body_pairs": st0["p2p_body_pairs"]},
            "m2l": {"ms": alone["m2l"] * 1e3, "ms_in_step": kern["m2l"] * 1e3, "tflops_executed": m2l_tf_alone,
                    "pairs": st0["m2l_pairs"]},
            **{k: {"ms": alone[k] * 1e3, "gbs": tree_bytes[k] / alone[k] * 1e-9 if alone[k] else None,
                   "frac_of_hbm": tree_bytes[k] / alone[k] * 1e-9 / hbm if alone[k] else None}
               for k in ("p2m", "m2m", "l2l", "l2p")},
            "matvec_device_ms": kern["matvec"] * 1e3, "matvec_device_ms_serialised": alone["matvec"] * 1e3},
        "tree": {k: st0[k] for k in ("n_cells", "n_leaves", "max_level", "m2l_pairs", "p2p_pairs",
                                     "p2p_body_pairs", "m2l_shift_classes")},
        "setup_seconds": statistics.median(setup_warm), "setup_seconds_first_call": setup_cold,
        "setup_seconds_calls": setup_warm, "clocks": clocks,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    if not args.no_bie and cfg.name == "cfg2" and n == cfg.n:
        del op
        line["bie_solve"] = run_bie_solve()
    print(json.dumps(line), flush=True)


def run_bie_solve(subdivisions: int = 7, k: float = 4.0, order: int = 12):
    """BASELINE.json configs[2] end to end on the device (reported next to the headline metric, not
    part of it): icosphere with 327,680 curved triangles, order-1 basis (983,040 unknowns), tree +
    interaction lists + singular / near corrections built by the library, GMRES(30) to 1e-4 on the
    plane wave e^{ikz}.  The quadrature tables are the reference's geometry.cpp rules stored with the
    fixtures (tests/golden/solver.npz); block-Jacobi is off (it slows GMRES(30) down on this
    first-kind system, in the reference as well: BASELINE.md section 2, 104 vs 67 iterations)."""
    import numpy as np

    from paper_1803_09948_b200 import HfmmCuda
    from paper_1803_09948_b200.workloads import icosphere_patches, patch_samples

    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "tests", "golden", "solver.npz"))
    tables = {key: g["bie_rule_" + key] for key in ("sample_ref", "far_weight", "near_pts", "near_basis",
                                                    "self_npts", "self_pts", "self_basis")}
    patches = icosphere_patches(subdivisions)
    xyz = patch_samples(patches, tables["sample_ref"])
    op = HfmmCuda(k=k, order=order, ncrit=64, theta=0.4, kd_max=1.0, leaf_cap=-1.0, device=0)
    t0 = time.perf_counter()
    op.set_points(xyz)
    t_tree = time.perf_counter() - t0
    t0 = time.perf_counter()
    nnz = op.build_corrections(patches, tables, mode=2, fetch=False)
    t_corr = time.perf_counter() - t0
    rhs = np.exp(1j * k * xyz[:, 2])
    t0 = time.perf_counter()
    x, rep = op.gmres(rhs, rtol=1e-4, restart=30, max_iterations=1000, precondition=False)
    t_solve = time.perf_counter() - t0
    from paper_1803_09948_b200.workloads import mie_soft_sphere
    th = np.linspace(0, np.pi, 37)
    obs = np.stack([4 * np.sin(th), 0 * th, 4 * np.cos(th)], 1)
    scat = -op.evaluate_field(x, obs)            # physical field = minus the layer sum (solver.hpp:134-136)
    mie = mie_soft_sphere(1.0, k, 4.0, th)
    mismatch = float(np.linalg.norm(scat - mie) / np.linalg.norm(mie))
    return {"workload": "BASELINE.json configs[2]: BIE GMRES solve, sound-soft unit sphere, plane wave e^{ikz}",
            "triangles": int(len(patches)), "unknowns": int(len(xyz)), "k": k, "order": order,
            "near_correction_nnz": int(nnz), "tree_and_lists_seconds": t_tree, "corrections_seconds": t_corr,
            "gmres": {"rtol": 1e-4, "restart": 30, "block_jacobi": False, "iterations": int(rep["iterations"]),
                      "converged": bool(rep["converged"]), "final_residual": float(rep["final_residual"])},
            "solve_seconds": t_solve, "checksum": float(np.abs(x).sum()),
            "mie_mismatch_rel_l2_at_r4": mismatch}


def run_multi(args, cfg, rank: int, world: int):
    from paper_1803_09948_b200.distributed import bench_distributed

    if "RANK" not in os.environ:   # single process: stand up a 1-rank group
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT="29517")

    line = bench_distributed(args, cfg, rank, world, METRIC, UNIT, workload_config, ClockSampler)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=None, help="cfg1|cfg2|cfg4|cfg5 (default: cfg2 at N=1, cfg5 weak at N>1)")
    ap.add_argument("--n", type=int, default=None, help="override the point count (debug)")
    ap.add_argument("--ref-points", type=int, default=131072,
                    help="sample size of the cpu_baseline leg of the default arm (one matvec, ~25 s on 16 cores)")
    ap.add_argument("--ref-arm-points", type=int, default=262144, help="sample size of --impl reference")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-bie", action="store_true", help="skip the configs[2] BIE solve reported next to the headline")
    ap.add_argument("--force-distributed", action="store_true",
                    help="run the N > 1 code path even with one rank (exercises the exchange plumbing)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    name = args.config or ("cfg2" if args.gpus == 1 else "cfg5_per_gpu")
    cfg = CONFIGS[name]
    if args.impl == "reference":
        run_reference(args, CONFIGS[args.config or "cfg2"], rank)
        return
    if args.gpus == 1 and world == 1 and not args.force_distributed:
        run_single(args, cfg)
    else:
        run_multi(args, cfg, rank, world)


if __name__ == "__main__":
    main()
