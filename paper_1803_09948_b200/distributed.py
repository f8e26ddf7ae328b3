"""Multi-GPU FMM matvec: one process per GPU, Morton-partitioned targets.  The data plane lives in the
library (csrc/comm.cu: pack kernel -> one grouped ncclSend / ncclRecv -> unpack kernel on a communication
stream, device-side all-reduce of the GMRES scalars); this module is the LAUNCHER around it:

  * bootstrap        torch.distributed (the process group torchrun or bench.py set up) carries the 128-byte
                     NCCL unique id from rank 0 to its peers, then is used for timing reductions only
  * ShardedFmm       set_partition + communicator + owned slices of the Morton-ordered vectors
  * host transport   the same exchanges staged through pinned host memory and performed with gloo on CPU
                     tensors: what lets two processes share ONE GPU in the tests (NCCL refuses that)
  * emulation        R handles in one process, one host thread per rank, the host transport between them

Data flow of one matvec on rank r (stands in for the reference's simulated
part::distributed_matvec, let.cpp:320-362): halo charges and the multipoles of the cells this rank
translates from arrive through the two locally-essential-tree exchanges (sender-initiated like the
reference's extract_let); P2M + M2M of the owned cells overlap the first, the near field the second.
"""
from __future__ import annotations

import os
import threading
import time

import numpy as np


class DevicePointerTensor:
    """exposes a raw device allocation of the library to torch through __cuda_array_interface__"""

    def __init__(self, ptr: int, n_float32: int):
        self.__cuda_array_interface__ = {"shape": (n_float32,), "typestr": "<f4",
                                         "data": (int(ptr), False), "version": 3, "strides": None}


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


def init_nccl(op, dist, rank: int):
    """ncclCommInitRank inside the library: rank 0 creates the unique id, the process group hands it on"""
    box = [op.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    op.comm_init_nccl(box[0])


def init_host_transport(op, dist, group=None):
    """The host-staged transport over a gloo process group (CPU tensors): all_to_all_single with uneven
    splits on bytes, all_reduce on doubles."""
    import torch

    def alltoallv(send, send_bytes, recv, recv_bytes):
        s = torch.from_numpy(send) if send.size else torch.zeros(0, dtype=torch.uint8)
        r = torch.from_numpy(recv) if recv.size else torch.zeros(0, dtype=torch.uint8)
        dist.all_to_all_single(r, s, output_split_sizes=[int(v) for v in recv_bytes],
                               input_split_sizes=[int(v) for v in send_bytes], group=group)

    def allreduce_sum(values):
        t = torch.from_numpy(values)
        dist.all_reduce(t, group=group)

    op.comm_init_host(alltoallv, allreduce_sum)


class ShardedFmm:
    """The FMM operator of one rank.  Vectors are sharded by Morton range: rank r holds
    q[first_r : first_r + count_r] of the Morton-ordered charge vector and produces the same slice
    of the potential.  transport: "nccl" (one GPU per rank) or "host" (gloo; ranks may share a GPU)."""

    def __init__(self, op, dist, rank: int, world: int, device, transport: str = "nccl", group=None):
        import torch

        self.op, self.dist, self.rank, self.world, self.device = op, dist, rank, world, device
        if transport == "nccl":         # also in a world of one: the same code path, one rank
            init_nccl(op, dist, rank)
        elif transport == "host":
            init_host_transport(op, dist, group)
        elif transport is not None:
            raise ValueError("transport must be 'nccl', 'host' or None (world of one, no communicator)")
        p = op.partition()
        self.n = int(p.n_bodies)
        self.first, self.count = int(p.body_first), int(p.body_count)
        self.out = torch.zeros(max(self.count, 1), 2, dtype=torch.float32, device=device)
        self.owned_m2l_pairs = int(p.owned_m2l_pairs)
        self.owned_p2p_body_pairs = int(p.owned_p2p_body_pairs)
        self.let_bytes = dict(zip(("charges", "multipoles"), op.exchange_volume())) if transport else \
            {"charges": 0, "multipoles": 0}

    def matvec(self, q_local):
        """q_local: (count, 2) float32 device tensor, the owned Morton slice -> same slice of A q
        (asynchronous on the library's streams; the caller synchronises the handle)"""
        self.op.dist_matvec(q_local.data_ptr(), self.out.data_ptr())
        return self.out[:self.count]

    def gmres(self, rhs_local, rtol=1e-4, restart=30, max_iterations=500, precondition=True):
        """Distributed GMRES: rhs_local / the returned solution are the owned
        Morton slices (complex128 numpy).  Krylov vectors stay sharded on the GPUs, the inner products are
        all-reduced on the device by the library's communicator."""
        return self.op.dist_solve(rhs_local, rtol=rtol, restart=restart, max_iterations=max_iterations,
                                  precondition=precondition)


class ThreadTransport:
    """The host transport between R handles of ONE process (one host thread per rank): a mailbox and a
    barrier.  No kernel ever waits on another rank's kernel — every exchange happens on the host side of
    a stream synchronise — so this is safe on a single device (B200_PROFILING.md)."""

    def __init__(self, nranks: int, timeout: float = 180.0):
        self.R = nranks
        self.barrier = threading.Barrier(nranks, timeout=timeout)
        self.send = [None] * nranks
        self.sbytes = [None] * nranks
        self.vals = [None] * nranks

    def callbacks(self, r: int):
        def alltoallv(send, send_bytes, recv, recv_bytes):
            self.send[r], self.sbytes[r] = send, send_bytes
            self.barrier.wait()
            off = 0
            for p in range(self.R):
                nb = int(recv_bytes[p])
                if nb:
                    start = int(self.sbytes[p][:r].sum())
                    assert int(self.sbytes[p][r]) == nb, "send and receive lists disagree"
                    recv[off:off + nb] = self.send[p][start:start + nb]
                off += nb
            self.barrier.wait()

        def allreduce_sum(values):
            self.vals[r] = values.copy()
            self.barrier.wait()
            total = sum(self.vals[p] for p in range(self.R))   # same order on every rank: identical bits
            self.barrier.wait()
            values[:] = total

        return alltoallv, allreduce_sum


def run_ranks_in_threads(ops, fn, timeout: float = 180.0):
    """fn(rank, op) on one host thread per handle, the handles joined by a ThreadTransport;
    returns the per-rank results"""
    import torch

    R = len(ops)
    tr = ThreadTransport(R, timeout)
    dev = torch.cuda.current_device()
    for r, op in enumerate(ops):
        op.comm_init_host(*tr.callbacks(r))
    results, errors = [None] * R, []

    def run(r):
        torch.cuda.set_device(dev)
        try:
            results[r] = fn(r, ops[r])
        except BaseException as e:
            errors.append(e)
            tr.barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(R)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        real = [e for e in errors if not isinstance(e, threading.BrokenBarrierError)]
        raise (real or errors)[0]
    return results


def emulate_gmres_on_one_device(ops, rhs_morton, timeout=180.0, **kw):
    """Distributed GMRES of `len(ops)` ranks on ONE GPU through the library's own sharded solver and
    exchanges (host transport between threads).  Returns the per-rank (x_owned, report) list."""
    def solve(r, op):
        p = op.partition()
        f, c = int(p.body_first), int(p.body_count)
        return op.dist_solve(rhs_morton[f:f + c], **kw)

    return run_ranks_in_threads(ops, solve, timeout)


def emulate_matvec_on_one_device(ops, q_morton, timeout=180.0):
    """hfmm_cuda_dist_matvec of `len(ops)` ranks on ONE GPU (threads + host transport): the assembled
    Morton-ordered result as a (n, 2) float32 device tensor"""
    import torch

    out = torch.zeros_like(q_morton)

    def mv(r, op):
        p = op.partition()
        f, c = int(p.body_first), int(p.body_count)
        qi = q_morton[f:f + c].contiguous()
        yo = torch.zeros(max(c, 1), 2, dtype=torch.float32, device=q_morton.device)
        op.dist_matvec(qi.data_ptr(), yo.data_ptr())
        op.sync()
        out[f:f + c] = yo[:c]
        return c

    run_ranks_in_threads(ops, mv, timeout)
    return out


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


def repartitioned_gmres_emulated(make_ops, rhs_morton, rtol=1e-4, restart=30, max_iterations=500,
                                 precondition=True, alpha_max: float = 2.0, timeout=180.0):
    """GMRES(restart) over Morton-sharded vectors with the reference's repartitioning loop acting at the restart
    boundaries (partition.cpp:143-227), ranks emulated on ONE GPU.

    make_ops(alpha) -> the handles of all ranks, partitioned with w = l + alpha r (set_partition +
    set_partition_alpha before set_points).  Every restart cycle is one hfmm_cuda_dist_solve of the residual
    equation Z d = r with max_iterations = restart (x += d, r <- hfmm_cuda_get_solve_residual): the same
    iteration as the monolithic restarted solver — the absolute target rtol ||b|| is kept by rescaling rtol —
    but the handles may change between two cycles.  A cycle's matvec time per iteration (max over ranks) is
    what update_alpha sees; when it moves alpha the Morton cuts are redrawn (make_ops) and iterate and residual,
    held in global Morton order here, are simply sliced again.  Returns (x_morton, report)."""
    rp = Repartitioner(make_ops, alpha_max)
    rhs = np.asarray(rhs_morton, dtype=np.complex128)
    bnorm = float(np.linalg.norm(rhs))
    x, r = np.zeros_like(rhs), rhs.copy()
    rep = {"iterations": 0, "converged": bnorm == 0.0, "residuals": [], "alphas": [], "cuts": [], "recuts": 0,
           "final_residual": 0.0 if bnorm == 0.0 else 1.0}
    target = rtol * bnorm
    while not rep["converged"] and rep["iterations"] < max_iterations:
        ops = rp.operator
        parts = [op.partition() for op in ops]
        rep["alphas"].append(rp.alpha)
        rep["cuts"].append([int(p.body_first) for p in parts])
        rnorm = float(np.linalg.norm(r))
        res = emulate_gmres_on_one_device(ops, r, timeout, rtol=min(target / rnorm, 0.999999), restart=restart,
                                          max_iterations=min(restart, max_iterations - rep["iterations"]),
                                          precondition=precondition)
        x += np.concatenate([d for d, _ in res])
        r = np.concatenate([op.solve_residual() for op in ops])
        r0 = res[0][1]
        assert len({q["iterations"] for _, q in res}) == 1, "ranks left lock step"
        rep["iterations"] += int(r0["iterations"])
        rep["residuals"] += [float(v) * rnorm / bnorm for v in r0["residuals"]]
        rep["final_residual"] = float(np.linalg.norm(r)) / bnorm
        if rep["final_residual"] <= rtol or (rep["residuals"] and rep["residuals"][-1] <= rtol) or r0["breakdown"]:
            rep["converged"] = rep["final_residual"] <= rtol or rep["residuals"][-1] <= rtol
            break
        per_it = max(float(q["matvec_seconds"]) for _, q in res) / max(int(r0["iterations"]), 1)
        if rp.record(per_it):
            rep["recuts"] += 1
    return x, rep


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
    """bench.py --gpus N (N > 1), one rank per GPU.  --scaling strong (default): the configuration's points
    (BASELINE cfg 5: 33,554,432) are shared out over the ranks; weak: cfg.n points per GPU.  Rank 0 also times
    the same total problem as ONE domain on its own GPU (when it fits) so that every line carries its own
    single-GPU baseline."""
    import torch
    import torch.distributed as dist

    from . import HfmmCuda
    from .workloads import charges, make_points

    local = int(os.environ.get("LOCAL_RANK", rank))
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench.py --gpus {world}: rank {rank} needs cuda:{local}, "
                         f"this node has {torch.cuda.device_count()} GPU(s)")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    # the process group is bootstrap and timing plumbing only (gloo); the data plane is the library's NCCL
    dist.init_process_group("gloo")
    strong = args.scaling == "strong"
    n_total = (args.n or cfg.n) if strong else (args.n or cfg.n) * world
    xyz = make_points(cfg, n_total)              # every rank builds the same global tree
    op = HfmmCuda(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max,
                  leaf_cap=cfg.leaf_cap, device=local)
    op.set_partition(rank, world)
    t0 = time.perf_counter()
    op.set_points(xyz)
    setup = time.perf_counter() - t0
    sh = ShardedFmm(op, dist, rank, world, device, transport=args.transport)
    order = op.body_order()
    q_all = charges(n_total, cfg.seed)
    q = q_all[order[sh.first:sh.first + sh.count]]
    q_local = torch.from_numpy(np.stack([q.real, q.imag], 1).astype(np.float32)).to(device)

    def barrier():
        op.sync()
        torch.cuda.synchronize()
        dist.barrier()

    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    for _ in range(args.warmup):
        sh.matvec(q_local)
    barrier()
    t0 = time.perf_counter()
    op.timer_record(0)
    for _ in range(args.steps):
        sh.matvec(q_local)
    op.timer_record(1)
    dev_ms = op.timer_elapsed_ms(0, 1) / args.steps
    barrier()
    wall_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    ms = torch.tensor([dev_ms, wall_ms], dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    # end to end: owned charges come from / results go to pinned host memory every step
    qh = torch.from_numpy(np.stack([q.real, q.imag], 1).astype(np.float32)).pin_memory()
    oh = torch.empty_like(qh).pin_memory()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        q_local.copy_(qh, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        y = sh.matvec(q_local)
        op.sync()
        oh.copy_(y, non_blocking=True)
        torch.cuda.synchronize()
    e2e = torch.tensor([(time.perf_counter() - t0) / args.steps], dtype=torch.float64)
    dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    st = op.stats()
    work = torch.tensor([float(sh.owned_m2l_pairs), float(sh.owned_p2p_body_pairs), float(sh.count),
                         float(sh.let_bytes["charges"]), float(sh.let_bytes["multipoles"])], dtype=torch.float64)
    allw = [torch.zeros_like(work) for _ in range(world)]
    dist.all_gather(allw, work)
    clocks = sampler.stop() if rank == 0 else None
    # the same total problem as one domain on rank 0's GPU: the baseline of this line
    single = None
    if rank == 0 and not args.no_single_domain:
        del sh
        op.close()
        torch.cuda.empty_cache()
        try:
            one = HfmmCuda(k=cfg.k, order=cfg.order, ncrit=cfg.ncrit, theta=cfg.theta, kd_max=cfg.kd_max,
                           leaf_cap=cfg.leaf_cap, device=local)
            one.set_points(xyz)
            qd = torch.from_numpy(np.stack([q_all.real, q_all.imag], 1).astype(np.float32)).to(device)
            od = torch.empty_like(qd)
            for _ in range(min(args.warmup, 2)):
                one.matvec_device(qd.data_ptr(), od.data_ptr())
            one.sync()
            ks = max(1, min(args.steps, 5))
            one.timer_record(0)
            for _ in range(ks):
                one.matvec_device(qd.data_ptr(), od.data_ptr())
            one.timer_record(1)
            t1 = one.timer_elapsed_ms(0, 1) / ks
            single = {"n_points": n_total, "ms_per_step": t1, "value": n_total / t1 * 1e-3, "unit": unit, "steps": ks}
            one.close()
        except Exception as e:        # e.g. out of memory for a problem sized for N GPUs
            single = {"unavailable": str(e)[:200]}
    dist.barrier()
    dist.destroy_process_group()
    if rank != 0:
        return None
    ms_step = float(ms[1])     # wall clock between barriers bounds the max over ranks
    allw = torch.stack(allw).numpy()
    line = {
        "metric": metric, "value": n_total / ms_step * 1e-3, "unit": unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": workload_config(cfg, n_total, world),
        "e2e": {"value": n_total / float(e2e[0]) * 1e-6, "unit": unit,
                "ms_per_step": float(e2e[0]) * 1e3,
                "h2d_bytes_per_step": int(allw[0, 2]) * 8, "d2h_bytes_per_step": int(allw[0, 2]) * 8},
        "gpu_launches": (int(st["kernel_launches"]) + 4) * args.steps,
        # per rank receive volume per matvec: locally essential rows only
        "exchange": {"kind": f"locally essential tree: pack kernel, grouped send/recv ({args.transport}), unpack kernel",
                     "charges_bytes_per_rank": allw[:, 3].astype(int).tolist(),
                     "multipole_bytes_per_rank": allw[:, 4].astype(int).tolist()},
        "balance": {"m2l_pairs": allw[:, 0].tolist(), "p2p_body_pairs": allw[:, 1].tolist(),
                    "bodies": allw[:, 2].tolist()},
        "device_ms_rank_max": float(ms[0]), "setup_seconds": setup, "clocks": clocks,
    }
    if getattr(args, "share_gpu", False):
        line["invalid_as_scaling"] = "all ranks shared cuda:0 (--share-gpu): plumbing check, not a measurement"
    if single is not None:
        line["single_domain_same_problem"] = single
        if "ms_per_step" in single:
            line["speedup_vs_single_domain"] = single["ms_per_step"] / ms_step
    return line
