"""Multi-GPU form of the hot path (DESIGN.md §5/§7).

One process per GPU (torchrun; RANK / LOCAL_RANK / WORLD_SIZE from the
environment).  Trajectories are independent ("natural
independence"), so the path shards with no data-path collective: rank r
simulates the aligned id shard r of the canonical reduction tree
(`shard_bounds`, R26) up to its device-resident moment root
(`ssa_run_shard`).  The exchange step is the paper's two-level "systolic"
reduction (§3.2: workers reduce locally, the collector
reduces their partials) made deterministic:

1. an all-gather of one status/counter word per rank (status, events,
   near-ties, errors, first erroring id and reaction) -- every rank then
   holds the same job-wide counters and the same error, and no rank raises
   before the collectives, so an error on one rank cannot leave the others
   blocked in the next collective;
2. an all-gather of the W moment roots (NCCL over NVLink on the GPU box;
   gloo in the CPU tests, staged through host memory when the roots live on
   a GPU), merged by every rank as the top log2(W) levels of the same tree in
   rank order (`ssa_merge_roots`);
3. optionally, the raw-trajectory dumps concatenated in rank order
   (`gather_dump`) -- the shards are contiguous, so that is id order.

Because the RNG is keyed by the global trajectory id, every trajectory and
hence the merged grids are bitwise independent of W.  torch is used only for
device buffers and the process group; every step of the method runs in
libssa.so.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Callable, Optional, Tuple

import numpy as np
import torch
import torch.distributed as dist

from .ssa import SSAError, shard_bounds  # noqa: F401  (aligned-subtree shards, R26)

# status word layout (int64): status, events, near_ties, n_errors, first_error_id, first_error_reaction
_WORD = 6
_NO_ERROR_ID = (1 << 63) - 1


def env_rank() -> Tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment (1 process = 1 GPU)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _world(group=None) -> int:
    return dist.get_world_size(group) if dist.is_initialized() else 1


def _host_staged(t: torch.Tensor, group=None) -> bool:
    """gloo cannot read device memory: device tensors are staged through the host."""
    return t.is_cuda and dist.is_initialized() and dist.get_backend(group) == "gloo"


def _all_gather(out: torch.Tensor, inp: torch.Tensor, group=None):
    """all_gather_into_tensor in rank order (out = [W * inp.numel()])."""
    if _host_staged(inp, group):
        o = torch.empty(out.shape, dtype=out.dtype)
        dist.all_gather_into_tensor(o, inp.cpu(), group=group)
        out.copy_(o)
    else:
        dist.all_gather_into_tensor(out, inp, group=group)


def gather_roots(root: torch.Tensor, roots: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather the per-rank moment roots into `roots[W, ...]` in rank order
    (roots[r] = rank r's root).  `root` and `roots[r]` have the same shape;
    both live on the rank's device (CPU tensors under gloo, or device tensors
    staged through the host under gloo)."""
    world = _world(group)
    if roots.shape[0] != world or roots.shape[1:] != root.shape:
        raise ValueError(f"roots must be [{world}, {tuple(root.shape)}], got {tuple(roots.shape)}")
    if world == 1:
        roots[0].copy_(root)
    else:
        _all_gather(roots.view(-1), root.contiguous().view(-1), group)
    return roots


def max_and_sum(values, device, group=None):
    """Max over ranks of values[0] (a device time) and the sum of the rest
    (counters): the bench's max-over-ranks timing."""
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    if _world(group) > 1:
        tmax = t.clone()
        if _host_staged(t, group):
            t, tmax = t.cpu(), tmax.cpu()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        t[0] = tmax[0]
    return [float(v) for v in t.tolist()]


@dataclass
class StepResult:
    """Job-wide outcome of one sharded step, identical on every rank."""
    status: int              # 0, or the status of the first error by trajectory id (else the lowest rank's)
    events: int              # applied events over all ranks
    near_ties: int
    n_errors: int            # trajectories that ended in SSA_ERR_NUMERIC / OVERFLOW, all ranks
    first_error_id: int      # smallest erroring trajectory id (if n_errors > 0)
    first_error_reaction: int
    error_rank: int          # rank that reported `status` (-1 if OK)
    message: str = ""
    local: Optional[object] = None   # this rank's RunResult (None for an empty shard or a failed call)


def exchange_status(word, device, group=None):
    """All-gather the [W, 6] int64 status words (rank order) and combine them
    into one StepResult, the same on every rank."""
    w = torch.tensor(list(word), dtype=torch.int64, device=device)
    world = _world(group)
    allw = torch.empty((world, _WORD), dtype=torch.int64, device=device)
    if world == 1:
        allw[0].copy_(w)
    else:
        _all_gather(allw.view(-1), w, group)
    a = allw.cpu().numpy()
    events, ties, nerr = (int(a[:, i].sum()) for i in (1, 2, 3))
    status, err_rank, fid, frx = 0, -1, 0, -1
    bad = [r for r in range(world) if a[r, 0] != 0]
    if bad:
        # trajectory errors: the one with the smallest id (as a single-GPU ssa_run); any
        # other failure (argument, CUDA, ...): the lowest failing rank's
        traj = [r for r in bad if a[r, 0] in (3, 4) and a[r, 3] > 0]
        other = [r for r in bad if r not in traj]
        err_rank = min(other) if other else min(traj, key=lambda r: a[r, 4])
        status = int(a[err_rank, 0])
    if nerr:
        r0 = min((r for r in range(world) if a[r, 3] > 0), key=lambda r: a[r, 4])
        fid, frx = int(a[r0, 4]), int(a[r0, 5])
    return StepResult(status, events, ties, nerr, fid, frx, err_rank)


class ShardedEnsemble:
    """One rank's share of a W-GPU ensemble run: `step()` = ssa_run_shard on
    this rank's shard -> all-gather of the status words -> all-gather of the
    roots -> ssa_merge_roots in rank order.  `for_model` wires
    `run_shard(b, e, root)` and `merge(roots, out)` to the C-ABI calls; the
    CPU tests pass stand-ins to exercise the same orchestration under gloo."""

    def __init__(self, n_total: int, cells: int, device, run_shard: Callable, merge: Callable, group=None):
        self.world = _world(group)
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.group = group
        self.device = device
        self.n_total, self.cells = n_total, cells
        self.begin, self.end = shard_bounds(n_total, self.world, self.rank)
        self.root = torch.zeros((3, cells), dtype=torch.float64, device=device)
        self.roots = torch.zeros((self.world, 3, cells), dtype=torch.float64, device=device)
        self.out = torch.zeros((4, cells), dtype=torch.float64, device=device)
        self._run_shard = run_shard
        self._merge = merge
        self.last: Optional[StepResult] = None

    @classmethod
    def for_model(cls, model, n_total: int, t_end: float, sample_dt: float, seed: int, device, *,
                  path: int = 0, stream=None, group=None, dump_ids=None, **opts) -> "ShardedEnsemble":
        """dump_ids: the job's sorted global dump ids (each rank dumps those in its
        shard; `gather_dump(ens.last.local.dump, ...)` concatenates them)."""
        from . import ssa as S
        cells = S.grid_size(t_end, sample_dt) * model.S
        dev = torch.device(device)
        if stream is None and dev.type == "cuda":
            # the library must run on the stream the collectives are ordered on: torch's
            # current stream (an all-gather with async_op=False does not block the host)
            stream = torch.cuda.current_stream(dev).cuda_stream
        ids = None if dump_ids is None else np.asarray(dump_ids, dtype=np.uint64)

        def run_shard(b, e, root):
            mine = None if ids is None else ids[(ids >= b) & (ids < e)]
            return S.run_shard(model, b, e, t_end, sample_dt, seed, root, path=path, stream=stream,
                               raise_on_error=False, dump_ids=mine, **opts)

        def merge(roots, out):
            S.merge_roots(roots, roots.shape[0], cells, stream=stream, out=out)

        return cls(n_total, cells, dev, run_shard, merge, group)

    def step(self, raise_on_error: bool = True) -> StepResult:
        """Run this rank's shard and the exchange.  Returns the job-wide
        StepResult (the same on every rank); the merged (mean, var, M2, n)
        grids are left in `self.out`.  With raise_on_error, every rank raises
        the same SSAError after the collectives when any rank failed."""
        res, status, msg = None, 0, ""
        if self.end > self.begin:
            try:
                res = self._run_shard(self.begin, self.end, self.root)
                status = int(getattr(res, "status", 0) or 0) if res is not None else 0
            except SSAError as ex:            # no rank leaves before the collectives
                status, msg = ex.status, str(ex)
                self.root.fill_(float("nan"))
                self.root[0].zero_()
        else:
            self.root.zero_()                 # an empty shard is the identity leaf (n = 0)
        get = (lambda k, d=0: int(res.get(k, d)) if isinstance(res, dict) else int(getattr(res, k, d))) \
            if res is not None else (lambda k, d=0: d)
        word = [status, get("events"), get("near_ties"), get("n_errors"),
                get("first_error_id", _NO_ERROR_ID) if get("n_errors") else _NO_ERROR_ID,
                get("first_error_reaction", -1)]
        word_dev = self.device if not _host_staged(self.root, self.group) else torch.device("cpu")
        out = exchange_status(word, word_dev, self.group)
        out.local = res
        if out.status and out.error_rank == self.rank and msg:
            out.message = msg
        gather_roots(self.root, self.roots, self.group)
        self._merge(self.roots, self.out)
        self.last = out
        if raise_on_error and out.status:
            raise SSAError(out.status, f"rank {out.error_rank}: " + (
                out.message or (f"trajectory {out.first_error_id} (reaction {out.first_error_reaction})"
                                if out.n_errors else "shard failed")))
        return out


def gather_dump(dump, device, group=None, dst: Optional[int] = 0):
    """Concatenate the ranks' raw-trajectory dumps (ssa.Dump, host arrays) in
    rank order -- contiguous shards, so ascending id order.  Ranks may hold
    different numbers of dumped ids (or none: dump=None).  Returns the
    combined ssa.Dump on `dst` (every rank with dst=None), None elsewhere.
    The bytes travel through the process group (device tensors under NCCL)."""
    from .ssa import SUMMARY_DTYPE, Dump
    world = _world(group)
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if dump is not None:
        arrays = [dump.ids, dump.states, dump.events_at, dump.time_at, dump.summary]
        n = len(dump.ids)
        shape_gs = dump.states.shape[1:]
    else:
        arrays, n, shape_gs = None, 0, None
    # per-rank counts and the (G, S) shape
    meta = torch.tensor([n, *(shape_gs if shape_gs else (0, 0))], dtype=torch.int64)
    metas = torch.empty((world, 3), dtype=torch.int64)
    if world > 1:
        mdev = device if (dist.get_backend(group) != "gloo") else torch.device("cpu")
        m_all = metas.to(mdev)
        dist.all_gather_into_tensor(m_all.view(-1), meta.to(mdev), group=group)
        metas = m_all.cpu()
    else:
        metas[0] = meta
    counts = [int(c) for c in metas[:, 0]]
    G, S = (int(v) for v in metas[int(np.argmax(counts)), 1:])
    nmax = max(counts)
    if nmax == 0:
        return None
    dtypes = [np.dtype(np.uint64), np.dtype(np.int32), np.dtype(np.uint64), np.dtype(np.float64), SUMMARY_DTYPE]
    row_bytes = [8, 4 * G * S, 8 * G, 8 * G, SUMMARY_DTYPE.itemsize]
    stride = sum(row_bytes)
    buf = np.zeros((nmax, stride), np.uint8)     # one padded record per dumped id
    if n:
        off = 0
        for a, rb in zip(arrays, row_bytes):
            buf[:n, off:off + rb] = np.ascontiguousarray(a).view(np.uint8).reshape(n, rb)
            off += rb
    local = torch.from_numpy(buf.reshape(-1))
    if world > 1:
        cdev = device if dist.get_backend(group) != "gloo" else torch.device("cpu")
        allb = torch.empty(world * local.numel(), dtype=torch.uint8, device=cdev)
        dist.all_gather_into_tensor(allb, local.to(cdev), group=group)
        allb = allb.cpu().numpy().reshape(world, nmax, stride)
    else:
        allb = buf.reshape(1, nmax, stride)
    if dst is not None and rank != dst:
        return None
    rows = np.concatenate([allb[r, :counts[r]] for r in range(world)])
    tot = rows.shape[0]
    outs, off = [], 0
    for dt_, rb in zip(dtypes, row_bytes):
        outs.append(np.ascontiguousarray(rows[:, off:off + rb]).view(dt_).reshape(tot, -1))
        off += rb
    return Dump(outs[0].reshape(tot), outs[1].reshape(tot, G, S), outs[2].reshape(tot, G),
                outs[3].reshape(tot, G), outs[4].reshape(tot))
