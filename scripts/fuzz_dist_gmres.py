"""GPU: randomised sweep of the sharded GMRES (ranks = host threads on one device, emulate_gmres_on_one_device)
against the single-domain solver: random meshes, wavenumbers, rank counts, preconditioner on/off, both
accumulation modes."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from checkers import rel_l2
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.api import HFMM_FLAG_DETERMINISTIC
from paper_1803_09948_b200.distributed import emulate_gmres_on_one_device
from paper_1803_09948_b200.workloads import icosphere_patches, patch_samples

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cases = int(sys.argv[2]) if len(sys.argv) > 2 else 12
g1 = np.load(os.path.join(ROOT, "tests", "golden", "solver.npz"))
KEYS = ("sample_ref", "far_weight", "near_pts", "near_basis", "self_npts", "self_pts", "self_basis")
T1 = {k: g1["bie_rule_" + k] for k in KEYS}
t0 = time.time()
for case in range(cases):
    rng = np.random.default_rng([seed, case])
    sub = int(rng.choice([1, 2, 3]))
    patches = icosphere_patches(sub) * rng.uniform(0.6, 1.4, 3)
    k = float(rng.choice([1.0, 2.0, 4.0]))
    order = int(rng.choice([6, 8, 10]))
    ranks = int(rng.integers(2, 7))
    flags = HFMM_FLAG_DETERMINISTIC if rng.uniform() < 0.5 else 0
    pre = bool(rng.uniform() < 0.5)
    restart = int(rng.choice([10, 30, 80]))
    xyz = patch_samples(patches, T1["sample_ref"])
    single = HfmmCuda(k=k, order=order, ncrit=32, flags=flags)
    single.set_points(xyz)
    single.build_corrections(patches, T1, mode=2, fetch=False)
    rhs = np.exp(1j * k * xyz[:, 2])
    x1, rep1 = single.gmres(rhs, rtol=1e-4, restart=restart, max_iterations=300, precondition=pre)
    morton = single.body_order()
    ops = []
    for r in range(ranks):
        op = HfmmCuda(k=k, order=order, ncrit=32, flags=flags)
        op.set_partition(r, ranks)
        op.set_points(xyz)
        op.build_corrections(patches, T1, mode=2, fetch=False)
        ops.append(op)
    res = emulate_gmres_on_one_device(ops, rhs[morton], rtol=1e-4, restart=restart, max_iterations=300, precondition=pre)
    x = np.concatenate([xr for xr, _ in res])
    reps = [rep for _, rep in res]
    desc = f"case {case}: {len(patches)} patches k={k} P={order} ranks={ranks} flags={flags} pre={pre} restart={restart}"
    assert len({rep["iterations"] for rep in reps}) == 1, desc
    if max(reps[0]["iterations"], rep1["iterations"]) >= 270:
        # a restart length that stagnates: whether the cap of 300 is reached is a coin toss; only the
        # lock step of the ranks (above) is checked
        print(desc, f"near the iteration cap: single={rep1['iterations']} sharded={reps[0]['iterations']}", flush=True)
        continue
    assert all(rep["converged"] == rep1["converged"] for rep in reps), desc
    dit = abs(reps[0]["iterations"] - rep1["iterations"])
    d = rel_l2(x, x1[morton])
    print(desc, f"it single={rep1['iterations']} sharded={reps[0]['iterations']} sol diff={d:.1e}", flush=True)
    assert dit <= max(2, rep1["iterations"] // 20), desc
    if rep1["converged"]:   # two stagnated iterates at the iteration cap need not be close
        assert d < 5e-3, desc
    else:
        assert 0.5 < reps[0]["final_residual"] / rep1["final_residual"] < 2.0, desc
print(f"{cases} cases ok in {time.time()-t0:.0f} s")
