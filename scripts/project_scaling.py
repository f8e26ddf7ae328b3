"""GPU (one device): per-rank COMPUTE time of the sharded matvec, ranks run one after the other on the same GPU
(never concurrently: nothing waits on anything), against the single-domain matvec of the same point set.
A PROJECTION of strong scaling, not a measurement: the exchange is replaced by device copies and is reported
as bytes only (NVLink 5: 900 GB/s per direction).

    python scripts/project_scaling.py [cfg5] [n] [ranks ...]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.distributed import DevicePointerTensor, let_index_lists
from paper_1803_09948_b200.workloads import CONFIGS, charges, make_points

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
cfg = CONFIGS[name]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n
rank_counts = [int(v) for v in sys.argv[3:]] or [2, 4, 8]
xyz, q = make_points(cfg, n), charges(n, cfg.seed)
kw = dict(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max, leaf_cap=cfg.leaf_cap)

single = HfmmCuda(**kw)
t0 = time.perf_counter()
single.set_points(xyz)
setup1 = time.perf_counter() - t0
tt = []
for _ in range(4):
    y_ref = single.matvec(q)
    tt.append(single.stats()["matvec_seconds"] * 1e3)
t1 = float(np.median(tt[1:]))
morton = single.body_order()
st1 = single.stats()
del single
print(f"{name} n={n}: single domain {t1:.2f} ms per matvec, set_points {setup1:.2f} s, "
      f"{st1['m2l_pairs']} M2L pairs, {st1['p2p_body_pairs']} near body pairs", flush=True)

qm = q[morton]
q_dev = torch.from_numpy(np.stack([qm.real, qm.imag], 1).astype(np.float32)).cuda()


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for R in rank_counts:
    ops, setup = [], []
    for r in range(R):
        op = HfmmCuda(**kw)
        op.set_partition(r, R)
        t0 = time.perf_counter()
        op.set_points(xyz)
        setup.append(time.perf_counter() - t0)
        ops.append(op)
    parts = [op.partition() for op in ops]
    n_cells, stride = int(ops[0].stats()["n_cells"]), int(parts[0].coeff_stride)
    out = torch.zeros(n, 2, dtype=torch.float32, device="cuda")
    best = None
    for rep in range(3):
        up = []
        for op in ops:  # charges gathered: every rank reads the slots it needs
            up.append(timed(lambda: (op.dist_upward(q_dev.data_ptr()), op.sync())))
        mp = [torch.as_tensor(DevicePointerTensor(p.multipole_dev, n_cells * stride * 2), device="cuda").reshape(n_cells, stride * 2)
              for p in parts]
        for r in range(R):  # multipole exchange as device copies (owned level ranges)
            for s, ps in enumerate(parts):
                if s == r:
                    continue
                for L in range(int(ps.level_first), int(ps.level_last) + 1):
                    f, c = int(ps.cell_first[L]), int(ps.cell_count[L])
                    if c:
                        mp[r][f:f + c].copy_(mp[s][f:f + c])
        down = []
        for op in ops:
            down.append(timed(lambda: (op.dist_downward(out.data_ptr()), op.sync())))
        tot = [u + d for u, d in zip(up, down)]
        if best is None or max(tot) < max(best):
            best = tot
    y = out.cpu().numpy()
    y = y[:, 0] + 1j * y[:, 1]
    yc = np.empty_like(y)
    yc[morton] = y
    err = float(np.linalg.norm(yc - y_ref) / np.linalg.norm(y_ref))
    dim = (cfg.order + 1) ** 2
    vol = []
    for r, op in enumerate(ops):  # what the rank receives per matvec (sender-initiated LET lists)
        lists = let_index_lists(op, r, R)
        vol.append((8 * sum(len(v) for v in lists["recv_bodies"]), 8 * dim * sum(len(v) for v in lists["recv_cells"])))
    work = [float(p.owned_p2p_body_pairs) + 1600.0 * float(p.owned_m2l_pairs) for p in parts]
    line = (f"R={R}: per-rank compute ms max {max(best):.2f} mean {np.mean(best):.2f} min {min(best):.2f} | "
            f"projected efficiency t1 / (R max) = {t1 / (R * max(best)):.3f} | work balance max/mean "
            f"{max(work) / np.mean(work):.3f} | set_points per rank {np.mean(setup):.2f} s | sharded vs single rel L2 {err:.2e}")
    if vol:
        line += f" | exchange per rank (charges, multipoles) max {max(v[0] for v in vol) / 2**20:.1f} MiB, {max(v[1] for v in vol) / 2**20:.1f} MiB"
    print(line, flush=True)
    del ops, mp
    torch.cuda.empty_cache()
