"""GPU: BASELINE config 3 end to end on the device — plane-wave scattering from a sound-soft unit
sphere.  Tree, interaction lists, singular / near corrections and block-Jacobi factors are built by
the library on the GPU (hfmm_cuda_set_points + hfmm_cuda_build_corrections, quadrature tables from
tests/golden); restarted GMRES runs over the FMM operator; the scattered field is compared with the
reference's analytic Mie series when the compiled reference travelled to the box."""
import sys, os, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.workloads import icosphere_patches, patch_samples

sub = int(sys.argv[1]) if len(sys.argv) > 1 else 7          # 7: 327,680 triangles, 983,040 unknowns
k = float(sys.argv[2]) if len(sys.argv) > 2 else 4.0
order = int(sys.argv[3]) if len(sys.argv) > 3 else 12
g = np.load(os.path.join(ROOT, "tests", "golden", "solver.npz"))
tables = {key: g["bie_rule_" + key] for key in ("sample_ref", "far_weight", "near_pts", "near_basis", "self_npts", "self_pts", "self_basis")}
t0 = time.time(); patches = icosphere_patches(sub); xyz = patch_samples(patches, tables["sample_ref"]); t_mesh = time.time() - t0
op = HfmmCuda(k=k, order=order, ncrit=64, theta=0.4, kd_max=1.0, leaf_cap=-1.0)
t0 = time.time(); op.set_points(xyz); t_tree = time.time() - t0
t0 = time.time(); nnz = op.build_corrections(patches, tables, mode=2, fetch=False); t_corr = time.time() - t0
rhs = np.exp(1j * k * xyz[:, 2])                               # assemble_rhs, solver.cpp:302-312, direction +z
precondition = (sys.argv[4] != "0") if len(sys.argv) > 4 else False   # block-Jacobi slows GMRES(30) down on this system
t0 = time.time()
x, rep = op.gmres(rhs, rtol=1e-4, restart=30, max_iterations=1000, precondition=precondition)
t_solve = time.time() - t0
out = {"triangles": len(patches), "unknowns": len(xyz), "k": k, "order": order, "near_nnz": nnz,
       "mesh_s": round(t_mesh, 2), "tree_and_lists_s": round(t_tree, 3), "corrections_s": round(t_corr, 3),
       "block_jacobi": precondition, "iterations": rep["iterations"], "converged": rep["converged"], "final_residual": rep["final_residual"],
       "solve_s": round(t_solve, 3), "matvec_s_total": round(rep["matvec_seconds"], 3), **{k_: v for k_, v in op.stats().items() if k_ in ("m2l_pairs", "p2p_body_pairs", "n_cells")}}
th = np.linspace(0, np.pi, 37)
obs = np.stack([4 * np.sin(th), 0 * th, 4 * np.cos(th)], 1)
scat = -op.evaluate_field(x, obs)                              # physical field = minus the layer sum (solver.hpp:134-136)
try:
    from checkers import Ref, rel_l2, have_ref
    if have_ref():
        mie = Ref().mie_soft_sphere(1.0, k, np.stack([4 + 0 * th, th, 0 * th], 1))
        out["mie_mismatch_rel_l2"] = rel_l2(scat, mie)
except Exception as e:  # the analytic check is optional
    out["mie"] = repr(e)
print(json.dumps(out))
