"""Host cores only (no device code): BASELINE config 3 at full size with the reference's OWN single-precision
near field (kernel::Precision::f32, everything else FP64) inside an FP64 restarted GMRES (the oracle's restatement of
gmres.cpp) — the iteration count "in FP32 complex" the device is to be compared with, next to the all-FP64 count of
scripts/ref_bie_cpu.py.  ~35 minutes on 16 cores.

    python scripts/ref_f32_cfg3.py out.json [subdivisions]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from checkers import Oracle, Ref
from paper_1803_09948_b200.workloads import icosphere_patches

out = sys.argv[1]
sub = int(sys.argv[2]) if len(sys.argv) > 2 else 7
k, order = 4.0, 12
oracle, ref = Oracle(), Ref()
t0 = time.time()
sysr = ref.bie(icosphere_patches(sub), 1, k, mode=2, use_tree=False)
xyz, fw = sysr.samples()
corr = sysr.corrections()
fr = ref.fmm(xyz, k, order, ncrit=64, leaf_cap=1.0 / k, theta=0.4, kd_max=1.0, threads=os.cpu_count())
rhs = sysr.rhs((0, 0, 1))
t_build = time.time() - t0
calls = []


def A(u):
    t = time.time()
    y = oracle.apply_corrections(sysr.ni, corr["patch_block"], corr["near_offset"], corr["near_source"], corr["near_delta"],
                                 u, fr.matvec(u * fw, f32_p2p=True))
    calls.append(time.time() - t)
    print(f"matvec {len(calls)}: {calls[-1]:.1f} s", flush=True)
    return y


t0 = time.time()
_, rep = oracle.gmres(A, rhs, rtol=1e-4, restart=30, max_iterations=60)
json.dump({"triangles": 20 * 4 ** sub, "unknowns": int(sysr.n), "k": k, "order": order, "block_jacobi": False,
           "near_field": "reference kernel::Precision::f32", "krylov": "FP64 (oracle gmres)",
           "iterations": int(rep["iterations"]), "converged": bool(rep["converged"]),
           "final_residual": float(rep["final_residual"]), "build_s": t_build, "solve_s": time.time() - t0,
           "threads": os.cpu_count(), "residuals": [float(v) for v in rep["residuals"]]}, open(out, "w"))
print("iterations", rep["iterations"])
