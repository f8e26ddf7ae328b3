"""GPU: randomised call sequences on ONE handle (point sets replaced, corrections set and dropped, errors
in between, the host-builder fallback, both accumulation modes) — after every step the handle must
behave like a fresh one given the same inputs."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from checkers import rel_l2
from paper_1803_09948_b200 import HfmmCuda, HfmmError
from paper_1803_09948_b200.api import HFMM_FLAG_DETERMINISTIC, HFMM_FLAG_HOST_TREE

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
trials = int(sys.argv[2]) if len(sys.argv) > 2 else 20


def point_set(rng):
    kind = rng.choice(["cube", "sphere", "deep", "tiny", "bad"])
    n = int(rng.choice([40, 700, 5000, 30000]))
    if kind == "cube":
        return kind, rng.uniform(-1, 1, (n, 3))
    if kind == "sphere":
        v = rng.normal(size=(n, 3)); return kind, v / np.linalg.norm(v, axis=1, keepdims=True)
    if kind == "deep":      # > ncrit coincident points: last-level tree -> host-builder fallback
        base = rng.uniform(-1, 1, (max(8, n // 40), 3)); return kind, base[rng.integers(0, len(base), n)]
    if kind == "tiny":
        return kind, rng.uniform(-1, 1, (int(rng.integers(1, 4)), 3))
    bad = rng.uniform(-1, 1, (n, 3)); bad[int(rng.integers(0, n)), 1] = np.nan
    return kind, bad


t0 = time.time()
for trial in range(trials):
    rng = np.random.default_rng([seed, trial])
    k = float(rng.choice([1.0, 3.0, 6.0]))
    if rng.uniform() < 0.2: k = complex(k, 0.2 * k)
    cfg = dict(k=k, order=int(rng.choice([4, 8, 12, 13])), ncrit=int(rng.choice([8, 32, 64])),
               flags=int(rng.choice([0, HFMM_FLAG_DETERMINISTIC, HFMM_FLAG_HOST_TREE])))
    op = HfmmCuda(**cfg)
    xyz, corr = None, None
    log = []
    for step in range(8):
        action = rng.choice(["points", "matvec", "corr", "uncorr", "gmres"])
        if action == "points" or xyz is None:
            kind, cand = point_set(rng)
            try:
                op.set_points(cand)
                xyz, corr = cand, None       # corrections belong to a point set
                log.append(f"points:{kind}:{len(cand)}")
            except HfmmError as e:
                assert kind == "bad" and e.kind == "domain_error", (trial, step, kind, str(e))
                log.append("points:refused")
                if xyz is not None:          # the handle keeps no half-built state: set the old set again
                    op.set_points(xyz); corr = None
            continue
        n = len(xyz)
        q = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        fresh = HfmmCuda(**cfg)
        fresh.set_points(xyz)
        if action == "corr":
            corr = (rng.uniform(5, 9, n) + 1j * rng.uniform(-1, 1, n)) * (n / 10.0)
            op.set_corrections(1, patch_block=corr)
            log.append("corr")
        elif action == "uncorr" and corr is not None:
            op.set_points(xyz); corr = None   # the way to drop corrections
            log.append("uncorr")
        if corr is not None:
            fresh.set_corrections(1, patch_block=corr)
        if action == "gmres" and corr is not None:
            x, rep = op.gmres(q, rtol=1e-5, restart=20, max_iterations=100, precondition=False)
            xf, repf = fresh.gmres(q, rtol=1e-5, restart=20, max_iterations=100, precondition=False)
            assert rep["converged"] == repf["converged"] and abs(rep["iterations"] - repf["iterations"]) <= 1, (trial, log)
            assert rel_l2(x, xf) < 1e-4, (trial, log)
            log.append(f"gmres:{rep['iterations']}")
        y, yf = op.matvec(q), fresh.matvec(q)
        d = rel_l2(y, yf) if np.linalg.norm(yf) > 0 else float(np.abs(y).max())
        if cfg["flags"] & HFMM_FLAG_DETERMINISTIC:
            assert np.array_equal(y, yf), (trial, log, d)
        assert d < 3e-6, (trial, log, d)
        log.append(f"matvec:{d:.0e}")
    print(f"trial {trial}: {cfg} :: {' '.join(log)}", flush=True)
print(f"{trials} trials ok in {time.time()-t0:.0f} s")
