"""GPU: run one BASELINE config, print stats/phase times and the error against an FP64 direct sum
on sampled targets."""
import sys, os, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from checkers import Oracle, rel_l2
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.api import HFMM_FLAG_PHASE_TIMERS
from paper_1803_09948_b200.workloads import CONFIGS, charges, make_points

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n_override = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = CONFIGS[name]
n = n_override or cfg.n
t0 = time.time(); xyz = make_points(cfg, n); q = charges(n, cfg.seed); print(f"inputs {time.time()-t0:.2f}s")
op = HfmmCuda(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max,
              leaf_cap=cfg.leaf_cap, flags=HFMM_FLAG_PHASE_TIMERS)
t0 = time.time(); op.set_points(xyz); print(f"set_points {time.time()-t0:.2f}s")
for it in range(3):
    t0 = time.time(); y = op.matvec(q); wall = time.time() - t0
    st = op.stats()
    print(f"matvec wall {wall*1e3:.1f} ms; device {st['matvec_seconds']*1e3:.2f} ms: "
          + " ".join(f"{k[:-8]}={st[k]*1e3:.2f}" for k in ("p2p_seconds","p2m_seconds","m2m_seconds","m2l_seconds","l2l_seconds","l2p_seconds")))
print(json.dumps({k: v for k, v in st.items() if not k.endswith("seconds")}))
rng = np.random.default_rng(0); tg = rng.choice(n, size=min(2048, n), replace=False)
t0 = time.time(); exact = Oracle().direct_sum(xyz, q, cfg.k, tg); print(f"direct sum {time.time()-t0:.1f}s")
print(f"rel_l2 vs FP64 direct sum on {len(tg)} targets: {rel_l2(y[tg], exact):.3e}")
