"""Multi-GPU FMM matvec: one process per GPU, Morton-partitioned targets, torch.distributed for the
plumbing (NCCL over NVLink on GPUs; gloo in the CPU tests of the host-side logic).

Data flow of one matvec on rank r (stands in for the reference's simulated
part::distributed_matvec, let.cpp:320-362):

  1. charge exchange                       the bodies of the leaves on this rank's near lists
  2. device phase 1 (dist_upward)          P2M + M2M of the owned cells
  3. multipole exchange                    the multipoles this rank's M2L lists translate from
  4. device phase 2 (dist_downward)        M2L / L2L / L2P into the owned cells, near field of the
                                           owned leaves beside M2L, owned outputs
Exchanges 1 and 3 are the locally-essential-tree exchange (sender-initiated like the reference's
extract_let): every rank holds the global lists, derives matching send / receive index lists from
them (let_index_lists) and ships the rows with ONE all_to_all_single each.  pruned=False falls back
to all-gathering everything (per level a contiguous row range per rank; on NVSwitch even that is a
few ms — 2.5 M cells x 1.4 KB at BASELINE config 5 — against ~100 ms of compute).

The exchange helpers work on any tensors (CPU tensors under gloo in tests/test_distributed_gloo.py).
"""
from __future__ import annotations

import os
import time

import numpy as np


class DevicePointerTensor:
    """exposes a raw device allocation of the library to torch through __cuda_array_interface__"""

    def __init__(self, ptr: int, n_float32: int):
        self.__cuda_array_interface__ = {"shape": (n_float32,), "typestr": "<f4",
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def allgather_ranges(dist, buf, ranges, rank, world, scratch=None):
    """In-place all-gather of rank-owned row ranges of `buf` (first dim).

    ranges[r] = list of (row_first, row_count) owned by rank r, same list length on every rank.
    Owned rows are packed, exchanged with ONE padded all_gather_into_tensor, and the other ranks'
    rows unpacked into place.  Returns the scratch buffers for reuse."""
    import torch

    rows = [sum(c for _, c in rr) for rr in ranges]
    width = int(np.prod(buf.shape[1:])) if buf.dim() > 1 else 1
    maxrows = max(max(rows), 1)
    if scratch is None or scratch[0].shape[0] != maxrows * width:
        scratch = (torch.empty(maxrows * width, dtype=buf.dtype, device=buf.device),
                   torch.empty(world * maxrows * width, dtype=buf.dtype, device=buf.device))
    send, recv = scratch
    flat = buf.reshape(buf.shape[0], -1)
    off = 0
    for f, c in ranges[rank]:
        if c:
            send[off * width:(off + c) * width].copy_(flat[f:f + c].reshape(-1))
            off += c
    dist.all_gather_into_tensor(recv, send)
    for r in range(world):
        if r == rank:
            continue
        off = r * maxrows
        for f, c in ranges[r]:
            if c:
                flat[f:f + c].copy_(recv[off * width:(off + c) * width].reshape(c, width))
                off += c
    return scratch


def let_index_lists(op, rank: int, world: int):
    """Send / receive index lists of the locally-essential-tree exchange of `rank` (reference
    extract_let, let.cpp:150-253, sender-initiated): for every peer p
      send_cells[p]  own cells whose multipole p translates from     recv_cells[p]  p's cells this rank needs
      send_bodies[p] Morton slots of own leaves p sums directly      recv_bodies[p] slots of p's leaves needed here
    Every rank derives them from the same global masks, so send_*[p] here equals recv_*[rank] on p,
    element for element (ascending cell order)."""
    far, near, owner = op.exchange_masks()
    cells = op.cells()
    first, count = cells[:, 4].astype(np.int64), cells[:, 5].astype(np.int64)
    me = np.uint64(1) << np.uint64(rank)

    def slots(leaves):
        if len(leaves) == 0:
            return np.zeros(0, dtype=np.int64)
        return np.concatenate([np.arange(first[c], first[c] + count[c]) for c in leaves])

    out = dict(send_cells=[], recv_cells=[], send_bodies=[], recv_bodies=[])
    mine = owner == rank
    for p in range(world):
        bit = np.uint64(1) << np.uint64(p)
        theirs = owner == p
        if p == rank:
            for k in out:
                out[k].append(np.zeros(0, dtype=np.int64))
            continue
        out["send_cells"].append(np.nonzero(mine & ((far & bit) != 0))[0].astype(np.int64))
        out["recv_cells"].append(np.nonzero(theirs & ((far & me) != 0))[0].astype(np.int64))
        out["send_bodies"].append(slots(np.nonzero(mine & ((near & bit) != 0))[0]))
        out["recv_bodies"].append(slots(np.nonzero(theirs & ((near & me) != 0))[0]))
    return out


def exchange_rows(dist, buf, send_idx, recv_idx, device):
    """One all_to_all_single with uneven splits: rows buf[send_idx[p]] go to rank p, the rows received
    from p land in buf[recv_idx[p]] (in place; the index lists are device int64 tensors)."""
    import torch

    width = buf.shape[1]
    send = torch.cat([buf[i] for i in send_idx]) if sum(len(i) for i in send_idx) else buf.new_zeros((0, width))
    n_recv = sum(len(i) for i in recv_idx)
    recv = buf.new_empty((n_recv, width))
    dist.all_to_all_single(recv, send, output_split_sizes=[len(i) for i in recv_idx],
                           input_split_sizes=[len(i) for i in send_idx])
    if n_recv:
        buf[torch.cat(recv_idx)] = recv


class ShardedFmm:
    """The FMM operator of one rank.  Vectors are sharded by Morton range: rank r holds
    q[first_r : first_r + count_r] of the Morton-ordered charge vector and produces the same slice
    of the potential."""

    def __init__(self, op, dist, rank: int, world: int, device, pruned: bool = False):
        """pruned: exchange only the locally essential rows (all_to_all with index lists) instead of
        all-gathering every charge and every multipole"""
        import torch

        self.op, self.dist, self.rank, self.world, self.device = op, dist, rank, world, device
        p = op.partition()
        self.n = int(p.n_bodies)
        mine = torch.tensor([p.body_first, p.body_count, p.level_first, p.level_last]
                            + list(p.cell_first) + list(p.cell_count), dtype=torch.int64, device=device)
        allp = torch.empty(world * mine.numel(), dtype=torch.int64, device=device)
        dist.all_gather_into_tensor(allp, mine)
        allp = allp.reshape(world, -1).cpu().numpy()
        self.body_ranges = [[(int(a[0]), int(a[1]))] for a in allp]
        self.first, self.count = self.body_ranges[rank][0]
        lf, ll = int(p.level_first), int(p.level_last)
        self.cell_ranges = [[(int(a[4 + L]), int(a[4 + 22 + L])) for L in range(lf, ll + 1)] for a in allp]
        self.stride = int(p.coeff_stride)
        n_cells = int(op.stats()["n_cells"])
        self.q_full = torch.zeros(self.n, 2, dtype=torch.float32, device=device)
        self.out_full = torch.zeros(self.n, 2, dtype=torch.float32, device=device)
        self.multipole = None
        if p.multipole_dev:
            view = DevicePointerTensor(p.multipole_dev, n_cells * self.stride * 2)
            self.multipole = torch.as_tensor(view, device=device).reshape(n_cells, self.stride * 2)
        self._s1 = self._s2 = None
        self.pruned = pruned and world > 1
        if self.pruned:
            lists = let_index_lists(op, rank, world)
            to_dev = lambda v: [torch.from_numpy(a).to(device) for a in v]
            self.let = {k: to_dev(v) for k, v in lists.items()}
            self.let_bytes = {"charges": int(sum(len(a) for a in lists["recv_bodies"])) * 8,
                              "multipoles": int(sum(len(a) for a in lists["recv_cells"])) * self.stride * 8}
        self.owned_m2l_pairs = int(p.owned_m2l_pairs)
        self.owned_p2p_body_pairs = int(p.owned_p2p_body_pairs)

    def matvec(self, q_local):
        """q_local: (count, 2) float32 device tensor, the owned Morton slice -> same slice of A q"""
        import torch

        self.q_full[self.first:self.first + self.count].copy_(q_local)
        if self.pruned:
            exchange_rows(self.dist, self.q_full, self.let["send_bodies"], self.let["recv_bodies"], self.device)
        else:
            self._s1 = allgather_ranges(self.dist, self.q_full, self.body_ranges, self.rank, self.world, self._s1)
        torch.cuda.current_stream().synchronize()
        self.op.dist_upward(self.q_full.data_ptr())
        self.op.sync()
        if self.multipole is not None:
            if self.pruned:
                exchange_rows(self.dist, self.multipole, self.let["send_cells"], self.let["recv_cells"], self.device)
            else:
                self._s2 = allgather_ranges(self.dist, self.multipole, self.cell_ranges, self.rank,
                                            self.world, self._s2)
            torch.cuda.current_stream().synchronize()
        self.op.dist_downward(self.out_full.data_ptr())
        self.op.sync()
        return self.out_full[self.first:self.first + self.count]


    def gmres(self, rhs_local, rtol=1e-4, restart=30, max_iterations=500, precondition=True):
        """Distributed GMRES: rhs_local / the returned solution are the owned
        Morton slices (complex128 numpy).  Krylov vectors stay sharded on the GPUs; inner products
        are all-reduced, operands and multipoles all-gathered, by this rank's communicator."""
        import torch

        def allreduce_sum(values):
            t = torch.from_numpy(values).to(self.device)
            self.dist.all_reduce(t)
            values[:] = t.cpu().numpy()

        def gather_vector(ptr):
            full = torch.as_tensor(DevicePointerTensor(ptr, self.n * 2), device=self.device).reshape(self.n, 2)
            self._s1 = allgather_ranges(self.dist, full, self.body_ranges, self.rank, self.world, self._s1)
            torch.cuda.current_stream().synchronize()

        def gather_multipoles():
            if self.multipole is not None:
                if self.pruned:
                    exchange_rows(self.dist, self.multipole, self.let["send_cells"], self.let["recv_cells"],
                                  self.device)
                else:
                    self._s2 = allgather_ranges(self.dist, self.multipole, self.cell_ranges, self.rank,
                                                self.world, self._s2)
                torch.cuda.current_stream().synchronize()

        return self.op.dist_gmres(rhs_local, allreduce_sum, gather_vector, gather_multipoles, rtol=rtol,
                                  restart=restart, max_iterations=max_iterations, precondition=precondition)


class Repartitioner:
    """The reference's repartitioning loop (partition.cpp:137-227) around
    a sharded operator: time a window of matvecs (max over ranks), record (alpha, runtime), ask
    update_alpha for the next alpha, re-cut the Morton partition with w = l + alpha r.  Re-cutting
    rebuilds the rank's lists (set_points, ~0.2 s per million points), so it is done between
    GMRES restarts, when only the iterate and the right-hand side have to be re-sharded."""

    def __init__(self, make_operator, alpha_max: float = 2.0):
        # make_operator(alpha) -> a ShardedFmm (or anything whose matvec is timed by the caller)
        self.make_operator, self.alpha_max = make_operator, alpha_max
        self.alphas, self.runtimes = [], []
        inv_phi = 0.6180339887498948
        self.alpha = alpha_max - inv_phi * alpha_max      # the search's first probe
        self.operator = make_operator(self.alpha)

    def record(self, runtime_max_over_ranks: float) -> bool:
        """Feeds one measurement; returns True when the partition was re-cut (alpha changed)."""
        from .api import update_alpha

        self.alphas.append(self.alpha)
        self.runtimes.append(float(runtime_max_over_ranks))
        nxt = update_alpha(self.alphas, self.runtimes, self.alpha_max)
        if abs(nxt - self.alpha) <= 1e-12 * max(1.0, self.alpha_max):
            return False
        self.alpha = nxt
        self.operator = self.make_operator(nxt)
        return True


def emulate_gmres_on_one_device(ops, rhs_morton, timeout=120.0, **kw):
    """Distributed GMRES of `len(ops)` ranks on ONE GPU: one host thread per rank, the three
    exchanges replaced by barrier-separated device copies between the handles.  No kernel ever waits
    on another rank's kernel (every exchange happens on the host side of a stream synchronise), so
    this is safe on a single device.  Returns the per-rank (x_owned, report) list."""
    import threading

    import torch

    R = len(ops)
    parts = [op.partition() for op in ops]
    n = int(parts[0].n_bodies)
    dev = torch.device("cuda", torch.cuda.current_device())
    n_cells = int(ops[0].stats()["n_cells"])
    stride = int(parts[0].coeff_stride)
    barrier = threading.Barrier(R, timeout=timeout)
    scal = [None] * R
    vec = [None] * R
    mp = [torch.as_tensor(DevicePointerTensor(p.multipole_dev, n_cells * stride * 2),
                          device=dev).reshape(n_cells, stride * 2) if p.multipole_dev else None for p in parts]
    results, errors = [None] * R, []

    def run(r):
        torch.cuda.set_device(dev)
        p = parts[r]

        def allreduce_sum(values):
            scal[r] = values.copy()
            barrier.wait()
            total = sum(scal[s] for s in range(R))     # same order on every rank: identical bits
            barrier.wait()
            values[:] = total

        def gather_vector(ptr):
            vec[r] = torch.as_tensor(DevicePointerTensor(ptr, n * 2), device=dev).reshape(n, 2)
            barrier.wait()
            for s, ps in enumerate(parts):
                if s != r and ps.body_count:
                    f, c = int(ps.body_first), int(ps.body_count)
                    vec[r][f:f + c].copy_(vec[s][f:f + c])
            torch.cuda.synchronize()
            barrier.wait()

        def gather_multipoles():
            barrier.wait()
            if mp[r] is not None:
                for s, ps in enumerate(parts):
                    if s == r:
                        continue
                    for L in range(int(ps.level_first), int(ps.level_last) + 1):
                        f, c = int(ps.cell_first[L]), int(ps.cell_count[L])
                        if c:
                            mp[r][f:f + c].copy_(mp[s][f:f + c])
            torch.cuda.synchronize()
            barrier.wait()

        try:
            f, c = int(p.body_first), int(p.body_count)
            results[r] = ops[r].dist_gmres(rhs_morton[f:f + c], allreduce_sum, gather_vector,
                                           gather_multipoles, **kw)
        except BaseException as e:
            errors.append(e)
            barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(R)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return results


def emulate_ranks_on_one_device(ops, q_morton, pruned: bool = False):
    """Runs the sharded matvec of `len(ops)` ranks sequentially on ONE GPU (each op was created with
    set_partition(r, R) on the same global point set), replacing the two all-gathers by device
    copies.  Used by the GPU tests: one B200 is all this environment has, and ranks that wait on one
    another must not be run as concurrent kernels on a single device (B200_PROFILING.md)."""
    import torch

    parts = [op.partition() for op in ops]
    n = int(parts[0].n_bodies)
    dev = q_morton.device
    out = torch.zeros(n, 2, dtype=torch.float32, device=dev)
    n_cells = int(ops[0].stats()["n_cells"])
    stride = int(parts[0].coeff_stride)
    mp = []
    lets = [let_index_lists(op, r, len(ops)) for r, op in enumerate(ops)] if pruned else None
    for r, (op, p) in enumerate(zip(ops, parts)):
        if pruned:
            # a rank sees its own charges and the bodies of the leaves on its near lists, nothing else
            qr = torch.full_like(q_morton, float("nan"))
            f, c = int(p.body_first), int(p.body_count)
            qr[f:f + c] = q_morton[f:f + c]
            for s in range(len(ops)):
                idx = torch.from_numpy(lets[r]["recv_bodies"][s]).to(dev)
                assert np.array_equal(lets[r]["recv_bodies"][s], lets[s]["send_bodies"][r])
                qr[idx] = q_morton[idx]
            qr = torch.nan_to_num(qr, nan=1e30)   # a body that is read without having been received poisons the result
            op.dist_upward(qr.data_ptr())
        else:
            op.dist_upward(q_morton.data_ptr())     # every rank sees the gathered charges
        op.sync()
        mp.append(torch.as_tensor(DevicePointerTensor(p.multipole_dev, n_cells * stride * 2),
                                  device=dev).reshape(n_cells, stride * 2) if p.multipole_dev else None)
    for r, (op, p) in enumerate(zip(ops, parts)):     # multipole all-gather
        if mp[r] is None:
            continue
        for s, ps in enumerate(parts):
            if s == r:
                continue
            if pruned:
                idx = torch.from_numpy(lets[r]["recv_cells"][s]).to(dev)
                assert np.array_equal(lets[r]["recv_cells"][s], lets[s]["send_cells"][r])
                if len(idx):
                    mp[r][idx] = mp[s][idx]
                continue
            for L in range(int(ps.level_first), int(ps.level_last) + 1):
                f, c = int(ps.cell_first[L]), int(ps.cell_count[L])
                if c:
                    mp[r][f:f + c].copy_(mp[s][f:f + c])
    torch.cuda.synchronize()
    for op, p in zip(ops, parts):
        op.dist_downward(out.data_ptr())
        op.sync()
    return out, parts


def bench_distributed(args, cfg, rank, world, metric, unit, workload_config, ClockSampler):
    """bench.py --gpus N (N > 1): weak scaling, cfg.n points PER GPU, Morton-partitioned"""
    import torch
    import torch.distributed as dist

    from . import HfmmCuda
    from .workloads import charges, make_points

    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = torch.device("cuda", local)
    n_total = (args.n or cfg.n) * world
    xyz = make_points(cfg, n_total)              # every rank builds the same global tree
    op = HfmmCuda(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max,
                  leaf_cap=cfg.leaf_cap, device=local)
    op.set_partition(rank, world)
    t0 = time.perf_counter()
    op.set_points(xyz)
    setup = time.perf_counter() - t0
    sh = ShardedFmm(op, dist, rank, world, device, pruned=True)
    order = op.body_order()
    q = charges(n_total, cfg.seed)[order[sh.first:sh.first + sh.count]]
    q_local = torch.from_numpy(np.stack([q.real, q.imag], 1).astype(np.float32)).to(device)

    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    for _ in range(args.warmup):
        sh.matvec(q_local)
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(args.steps):
        y = sh.matvec(q_local)
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    wall_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    ms = torch.tensor([max(e0.elapsed_time(e1) / args.steps, 0.0), wall_ms], device=device)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    # end to end: owned charges come from / results go to pinned host memory every step
    qh = torch.from_numpy(np.stack([q.real, q.imag], 1).astype(np.float32)).pin_memory()
    oh = torch.empty_like(qh).pin_memory()
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        q_local.copy_(qh, non_blocking=True)
        oh.copy_(sh.matvec(q_local), non_blocking=True)
        torch.cuda.synchronize()
    e2e = torch.tensor([(time.perf_counter() - t0) / args.steps], device=device)
    dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    st = op.stats()
    work = torch.tensor([float(sh.owned_m2l_pairs), float(sh.owned_p2p_body_pairs), float(sh.count)],
                        device=device)
    allw = torch.empty(world * 3, device=device)
    dist.all_gather_into_tensor(allw, work)
    clocks = sampler.stop() if rank == 0 else None
    dist.destroy_process_group()
    if rank != 0:
        return None
    ms_step = float(ms[1])     # wall clock between barriers bounds the max over ranks
    allw = allw.reshape(world, 3).cpu().numpy()
    return {
        "metric": metric, "value": n_total / ms_step * 1e-3, "unit": unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": workload_config(cfg, n_total, world),
        "e2e": {"value": n_total / float(e2e[0]) * 1e-6, "unit": unit,
                "ms_per_step": float(e2e[0]) * 1e3,
                "h2d_bytes_per_step": int(sh.count) * 8, "d2h_bytes_per_step": int(sh.count) * 8},
        "gpu_launches": int(st["kernel_launches"]) * args.steps,
        # rank 0's receive volume per matvec: locally essential rows only (full gather in brackets)
        "exchange": {"kind": "locally essential tree, all_to_all" if sh.pruned else "all-gather",
                     "charges_bytes_per_rank": sh.let_bytes["charges"] if sh.pruned else n_total * 8,
                     "multipole_bytes_per_rank": sh.let_bytes["multipoles"] if sh.pruned else
                     int(sum(c for rr in sh.cell_ranges for _, c in rr)) * sh.stride * 8,
                     "full_gather_bytes_per_rank": n_total * 8 + int(sum(c for rr in sh.cell_ranges for _, c in rr)) * sh.stride * 8},
        "balance": {"m2l_pairs": allw[:, 0].tolist(), "p2p_body_pairs": allw[:, 1].tolist(),
                    "bodies": allw[:, 2].tolist()},
        "device_ms_rank_max": float(ms[0]), "setup_seconds": setup, "clocks": clocks,
    }
