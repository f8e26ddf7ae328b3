#!/usr/bin/env python
"""bench.py — the FMM Helmholtz matvec (BASELINE.json's hot path) on N B200s of one node.

    python bench.py --gpus 1 --steps K --warmup W              # this repo's CUDA path
    python bench.py --impl reference --gpus 1 --steps K ...     # the reference's CPU path, same metric
    python bench.py --gpus N ...                                # N > 1: spawns its own N ranks (one per GPU)
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...   # N > 1 under torchrun

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
    # The arm runs the configuration it prints: by default ALL of cfg 2 (1,048,576 points), one matvec and no
    # warm-up — about three to four minutes on this box's host cores (the reference rebuilds ~10^4 dense
    # translation matrices on every call and streams a 457 KB matrix per cell pair).  --ref-arm-points N
    # shrinks it; the config printed is then that of the N-point run, so the line never claims a size it did
    # not run.
    n_run = min(args.ref_arm_points or cfg.n, cfg.n)
    full = n_run == cfg.n
    warmup = 0 if full else min(args.warmup, 1)
    steps = 1 if full else max(1, min(args.steps, 7))
    base = cpu_reference_arm(cfg, n_run, steps, warmup, budget_s=0.0 if full else 170.0)
    line = {
        "impl": "reference", "metric": METRIC, "value": base["value"], "unit": UNIT,
        "n_gpus": args.gpus, "steps": base["steps"], "warmup": warmup,
        "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": base["seconds_per_matvec"] * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg, n_run, 1), "cpu_baseline": base,
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


def committed_traffic(cfg, n: int):
    """dram__bytes_read.sum + dram__bytes_write.sum of the dominant launch from the committed `ncu --set full`
    capture of this configuration (profiles/m2l_dram_traffic.json names the report it was read from and the
    commit it was taken at); None when no capture of this configuration is on record"""
    try:
        rec = json.load(open(os.path.join(ROOT, "profiles", "m2l_dram_traffic.json")))
    except (OSError, ValueError):
        return None, None
    for e in rec.get("entries", []):
        if e.get("config") == cfg.name and e.get("n_points") == n and e.get("order") == cfg.order:
            return float(e["dram_bytes_read"]) + float(e["dram_bytes_write"]), e.get("source")
    return None, None


def kernel_roofline(cfg, n: int, steps: int, fp32_peak: float):
    """P2P and M2L of one configuration timed alone (near field serialised behind the far field)"""
    import torch

    from paper_1803_09948_b200 import HfmmCuda
    from paper_1803_09948_b200.api import HFMM_FLAG_PHASE_TIMERS

    xyz, q = make_points(cfg, n), charges(n, cfg.seed)
    op = HfmmCuda(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max,
                  leaf_cap=cfg.leaf_cap, device=0, flags=HFMM_FLAG_PHASE_TIMERS)
    t0 = time.perf_counter()
    op.set_points(xyz)
    setup = time.perf_counter() - t0
    q_dev = torch.from_numpy(np.stack([q.real, q.imag], 1).astype(np.float32)).cuda()
    out_dev = torch.empty_like(q_dev)
    acc = {k: 0.0 for k in ("p2p", "m2l", "matvec")}
    for it in range(steps + 1):
        op.matvec_device(q_dev.data_ptr(), out_dev.data_ptr())
        st = op.stats()
        if it:
            for k in acc:
                acc[k] += st[f"{k}_seconds"] / steps
    ex, dense = m2l_flops_per_pair(cfg.order)
    m2l_tf = st["m2l_pairs"] * ex / acc["m2l"] * 1e-12 if acc["m2l"] else 0.0
    p2p_tf = st["p2p_body_pairs"] * 24 / acc["p2p"] * 1e-12 if acc["p2p"] else 0.0
    op.close()
    return {"workload": workload_config(cfg, n, 1)["workload"], "n_points": n, "order": cfg.order,
            "setup_seconds": setup, "matvec_ms_serialised": acc["matvec"] * 1e3,
            "m2l": {"ms": acc["m2l"] * 1e3, "pairs": st["m2l_pairs"], "flops_per_pair": ex,
                    "tflops_executed": m2l_tf, "frac_of_fp32_peak": m2l_tf / fp32_peak if fp32_peak else None,
                    "dense_equivalent_tflops": st["m2l_pairs"] * dense / acc["m2l"] * 1e-12 if acc["m2l"] else None},
            "p2p": {"ms": acc["p2p"] * 1e3, "body_pairs": st["p2p_body_pairs"], "tflops_24flop_per_pair": p2p_tf,
                    "frac_of_fp32_peak": p2p_tf / fp32_peak if fp32_peak else None, "kernel_variant": st["p2p_mode"],
                    "kernel_variant_in_step": st["p2p_mode_in_step"]}}


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

    # the reference interface's default, TraversalConfig::deterministic = true (ordered accumulation), beside it
    from paper_1803_09948_b200.api import HFMM_FLAG_DETERMINISTIC
    det_ms = None
    if not args.no_deterministic:
        opd = HfmmCuda(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max,
                       leaf_cap=cfg.leaf_cap, device=0, flags=HFMM_FLAG_DETERMINISTIC)
        opd.set_points(xyz)
        for _ in range(2):
            opd.matvec_device(q_dev.data_ptr(), out_dev.data_ptr())
        opd.sync()
        ks = max(1, min(args.steps, 5))
        opd.timer_record(0)
        for _ in range(ks):
            opd.matvec_device(q_dev.data_ptr(), out_dev.data_ptr())
        opd.timer_record(1)
        det_ms = opd.timer_elapsed_ms(0, 1) / ks
        opd.close()
    traffic, traffic_source = committed_traffic(cfg, n)

    cpu = cpu_reference_arm(cfg, args.ref_points, 1, 0) if not args.no_cpu_baseline else None
    line = {
        "metric": METRIC, "value": n / ms_step * 1e-3, "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
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
            # dram__bytes_read + dram__bytes_write of this launch, read from the committed ncu --set full
            # capture of the same configuration (profiles/m2l_dram_traffic.json; null when none is on
            # record); algorithmic bytes are pairs x 2 x 8 (P+1)^2 (one source row read, one destination
            # row reduced)
            "traffic": traffic, "traffic_source": traffic_source,
            "algorithmic_bytes": st0["m2l_pairs"] * 2 * 8 * (cfg.order + 1) ** 2},
        # kernel-alone durations (near field serialised behind the far field); "ms_in_step" is the event
        # interval inside the timed region, where P2P is co-resident with M2L
        "kernels": {
            "p2p": {"ms": alone["p2p"] * 1e3, "ms_in_step": kern["p2p"] * 1e3, "tflops_24flop_per_pair": p2p_tf,
                    "frac_of_fp32_peak": p2p_tf / fp32_peak if fp32_peak else None,
                    "body_pairs": st0["p2p_body_pairs"], "kernel_variant": st0["p2p_mode"],
                    "kernel_variant_in_step": st0["p2p_mode_in_step"],
                    "near_r2_max": st0["near_r2_max"]},
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
        "host_tree_used": st0["host_tree_used"],
        # the same step with the reference interface's default TraversalConfig::deterministic = true
        "deterministic_ms_per_step": det_ms,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    if not args.no_cfg4 and cfg.name == "cfg2" and n == cfg.n:
        # BASELINE configs[3] (Plummer, P = 14, theta = 0.35): the order-14 kernels, otherwise unbenchmarked
        del op
        torch.cuda.empty_cache()
        line["cfg4_kernels"] = kernel_roofline(CONFIGS["cfg4"], CONFIGS["cfg4"].n, 2, fp32_peak)
        op = None
    if not args.no_bie and cfg.name == "cfg2" and n == cfg.n:
        op = None
        torch.cuda.empty_cache()
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

    from paper_1803_09948_b200.workloads import quadrature_tables
    tables = quadrature_tables(basis_order=1)
    patches = icosphere_patches(subdivisions)
    xyz = patch_samples(patches, tables["sample_ref"])
    op = HfmmCuda(k=k, order=order, ncrit=64, theta=0.4, kd_max=1.0, leaf_cap=-1.0, device=0)
    t0 = time.perf_counter()
    op.set_points(xyz)
    t_tree = time.perf_counter() - t0
    t0 = time.perf_counter()
    nnz = op.build_corrections(patches, tables, mode=2, fetch=False)
    t_corr = time.perf_counter() - t0
    rhs = op.assemble_rhs((0.0, 0.0, 1.0))      # reference assemble_rhs: e^{ikz} at the samples
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

    line = bench_distributed(args, cfg, rank, world, METRIC, UNIT, workload_config, ClockSampler)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` without torchrun: start N ranks of this script (one per GPU), pass rank 0's
    JSON line through.  Fails loudly when the node has fewer than N GPUs — never a silent world of one."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if args.share_gpu and args.transport != "host":
        sys.stderr.write("bench.py: --share-gpu needs --transport host (NCCL refuses two ranks on one device)\n")
        return 2
    if have < args.gpus and not (args.share_gpu and have >= 1):
        print(json.dumps({"error": f"--gpus {args.gpus} requested, this node has {have} GPU(s)", "n_gpus": args.gpus}),
              flush=True)
        sys.stderr.write(f"bench.py: --gpus {args.gpus} requested, this node has {have} GPU(s)\n")
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK="0" if args.share_gpu else str(r), WORLD_SIZE=str(args.gpus),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env))
    rc = 0
    for p in procs:
        rc = rc or p.wait()
    return rc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=None,
                    help="cfg1|cfg2|cfg4|cfg5 (default: cfg2 at N=1; at N>1 cfg5 strong, cfg5_per_gpu weak)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N>1: strong = the configuration's points shared out over the ranks (BASELINE configs[4]: "
                         "33,554,432), weak = that many per GPU")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "host"],
                    help="N>1: the library's NCCL data plane, or its host-staged transport over gloo")
    ap.add_argument("--n", type=int, default=None, help="override the point count (debug)")
    ap.add_argument("--ref-points", type=int, default=131072,
                    help="sample size of the cpu_baseline leg of the default arm (one matvec, ~25 s on 16 cores)")
    ap.add_argument("--ref-arm-points", type=int, default=None,
                    help="--impl reference: run this many points instead of the whole configuration")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-bie", action="store_true", help="skip the configs[2] BIE solve reported next to the headline")
    ap.add_argument("--no-cfg4", action="store_true", help="skip the configs[3] kernel rooflines (P = 14)")
    ap.add_argument("--no-deterministic", action="store_true", help="skip the ordered-accumulation step time")
    ap.add_argument("--no-single-domain", action="store_true", help="N>1: skip the one-domain baseline on rank 0")
    ap.add_argument("--share-gpu", action="store_true",
                    help="debug: all ranks on cuda:0 (with --transport host) — exercises the N>1 path on a one-GPU "
                         "box; its numbers are NOT scaling measurements")
    ap.add_argument("--force-distributed", action="store_true",
                    help="run the N > 1 code path even with one rank (exercises the exchange plumbing)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)
    if args.impl == "reference":
        run_reference(args, CONFIGS[args.config or "cfg2"], int(os.environ.get("RANK", "0")))
        return
    if args.gpus > 1 and "RANK" not in os.environ:
        sys.exit(spawn_ranks(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.gpus == 1 and world == 1 and not args.force_distributed:
        run_single(args, CONFIGS[args.config or "cfg2"])
        return
    if args.force_distributed and "RANK" not in os.environ:
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT="29517")
    name = args.config or ("cfg5" if args.scaling == "strong" else "cfg5_per_gpu")
    run_multi(args, CONFIGS[name], rank, world)


if __name__ == "__main__":
    main()
