"""GPU: BASELINE config 3 at a reduced mesh — plane-wave scattering from a sound-soft unit sphere.
The reference (oracle/_ref, host) builds the discrete system (samples, singular/near corrections,
block-Jacobi factors); the device runs restarted GMRES over the FMM operator; the scattered field
is compared with the reference's analytic Mie series (oracle.cpp:11-59)."""
import sys, os, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from checkers import Ref, rel_l2
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.workloads import icosphere_patches

sub = int(sys.argv[1]) if len(sys.argv) > 1 else 3
k, order = 4.0, 12
R = Ref()
t0 = time.time()
sysr = R.bie(icosphere_patches(sub), 1, k, mode=2, use_tree=False)
xyz, fw = sysr.samples(); corr = sysr.corrections(); rhs = sysr.rhs((0, 0, 1))
t_build = time.time() - t0
op = HfmmCuda(k=k, order=order, ncrit=64, theta=0.4, kd_max=1.0, leaf_cap=-1.0)
t0 = time.time(); op.set_points(xyz); op.set_corrections(sysr.ni, far_weight=fw, **corr); t_setup = time.time() - t0
t0 = time.time()
x, rep = op.gmres(rhs, rtol=1e-4, restart=30, max_iterations=500, precondition=True)
t_solve = time.time() - t0
x0, rep0 = op.gmres(rhs, rtol=1e-4, restart=30, max_iterations=500, precondition=False)
# scattered field on a ring of radius 4 in the x-z plane vs the Mie series
th = np.linspace(0, np.pi, 37)
obs = np.stack([4 * np.sin(th), 0 * th, 4 * np.cos(th)], 1)
scat = -op.evaluate_field(x, obs)                    # physical field = minus the layer sum (solver.hpp:134-136)
mie = R.mie_soft_sphere(1.0, k, np.stack([4 + 0 * th, th, 0 * th], 1))
print(json.dumps({"triangles": 20 * 4 ** sub, "unknowns": int(sysr.n), "near_nnz": int(sysr.nnz),
                  "reference_build_s": round(t_build, 2), "device_setup_s": round(t_setup, 2),
                  "iterations_block_jacobi": rep["iterations"], "iterations_plain": rep0["iterations"],
                  "final_residual": rep["final_residual"], "solve_s": round(t_solve, 3),
                  "matvec_s_total": round(rep["matvec_seconds"], 3),
                  "mie_mismatch_rel_l2": rel_l2(scat, mie)}))
