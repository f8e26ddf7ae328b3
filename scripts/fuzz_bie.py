"""GPU: randomised sweep of the BIE surfaces — correction builders against the oracle's (random shapes,
wavenumbers, both basis orders, all singularity modes, random near thresholds), GMRES convergence and
its true residual, the sharded matvec at random rank counts against the single-domain one."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
from checkers import Oracle, rel_l2
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.distributed import emulate_ranks_on_one_device
from paper_1803_09948_b200.workloads import icosphere_patches, patch_samples

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cases = int(sys.argv[2]) if len(sys.argv) > 2 else 30
oracle = Oracle()
g1 = np.load(os.path.join(ROOT, "tests", "golden", "solver.npz"))
g2 = np.load(os.path.join(ROOT, "tests", "golden", "corrections_order2.npz"))
KEYS = ("sample_ref", "far_weight", "near_pts", "near_basis", "self_npts", "self_pts", "self_basis")
T1 = {k: g1["bie_rule_" + k] for k in KEYS}
T2 = {k: g2["rule_" + k] for k in KEYS}
t0 = time.time()
for case in range(cases):
    rng = np.random.default_rng([seed, case])
    sub = int(rng.choice([0, 1, 2, 3]))
    tables = T1 if rng.uniform() < 0.6 else T2
    scale = rng.uniform(0.4, 1.6, 3)          # ellipsoids
    shift = rng.uniform(-0.5, 0.5, 3)
    patches = icosphere_patches(sub) * scale + shift
    if rng.uniform() < 0.3:                   # two bodies
        patches = np.concatenate([patches, icosphere_patches(max(sub - 1, 0)) * 0.5 + shift + np.array([2.5, 0, 0])])
    k = float(rng.choice([0.5, 2.0, 4.0]))
    if rng.uniform() < 0.25:
        k = complex(k, 0.3 * k)
    mode = int(rng.choice([0, 1, 2]))
    near = float(rng.choice([-1.0, 0.0, 0.3, 1.0]))
    order = int(rng.choice([6, 8, 10]))
    desc = f"case {case}: {len(patches)} patches ni={len(tables['far_weight'])} k={k} mode={mode} near={near} P={order}"
    want = oracle.build_corrections(patches, tables, k, mode=mode, near_patch_distance=near)
    op = HfmmCuda(k=k, order=order, ncrit=int(rng.choice([8, 32, 64])))
    op.set_points(want["xyz"])
    got = op.build_corrections(patches, tables, mode=mode, near_patch_distance=near)
    for key in ("near_offset", "near_source", "block_piv"):
        assert np.array_equal(got[key], want[key]), (desc, key)
    for key in ("patch_block", "block_lu", "near_delta"):
        a, b = got[key], want[key]
        assert a.shape == b.shape, (desc, key)
        if b.size:
            assert np.abs(a - b).max() <= 3e-13 * max(1.0, np.abs(b).max()), (desc, key, np.abs(a - b).max())
    # GMRES on a plane wave: converges or reports honestly; the reported residual is the true one
    xyz = want["xyz"]
    rhs = np.exp(1j * np.real(k) * xyz[:, 2])
    x, rep = op.gmres(rhs, rtol=1e-4, restart=30, max_iterations=400, precondition=bool(mode and rng.uniform() < 0.5))
    r = rhs - op.matvec(x)
    true_res = np.linalg.norm(r) / np.linalg.norm(rhs)
    assert abs(true_res - rep["final_residual"]) < 5e-6 + 0.02 * rep["final_residual"], (desc, true_res, rep["final_residual"])
    # sharded matvec (plain operator) at a random rank count
    nranks = int(rng.integers(2, 9))
    single = HfmmCuda(k=k, order=order, ncrit=32)
    single.set_points(xyz)
    q = rng.uniform(-1, 1, len(xyz)) + 1j * rng.uniform(-1, 1, len(xyz))
    y_ref = single.matvec(q)
    ops = []
    for rk in range(nranks):
        o = HfmmCuda(k=k, order=order, ncrit=32)
        o.set_partition(rk, nranks)
        o.set_points(xyz)
        ops.append(o)
    morton = single.body_order()
    qm = q[morton]
    q_dev = torch.from_numpy(np.stack([qm.real, qm.imag], 1).astype(np.float32)).cuda()
    out, parts = emulate_ranks_on_one_device(ops, q_dev, pruned=bool(rng.uniform() < 0.5))
    y = out.cpu().numpy()
    d = rel_l2(y[:, 0] + 1j * y[:, 1], y_ref[morton])
    assert d < 3e-6, (desc, nranks, d)
    print(desc, f"nnz={got['near_source'].size} gmres it={rep['iterations']} conv={rep['converged']} res={rep['final_residual']:.1e} "
          f"ranks={nranks} sharded diff={d:.1e}", flush=True)
print(f"{cases} cases ok in {time.time()-t0:.0f} s")
