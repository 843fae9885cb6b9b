"""Multi-GPU form of the hot path (DESIGN.md §5/§7).

One process per GPU (torchrun; RANK / LOCAL_RANK / WORLD_SIZE from the
environment).  Trajectories are independent ("natural
independence"), so the path shards with no data-path collective: rank r
simulates the aligned id shard r of the canonical reduction tree
(`shard_bounds`, R26) up to its device-resident moment root
(`ssa_run_shard`).  The one exchange step is an all-gather of the W roots
(NCCL over NVLink on the GPU box; gloo in the CPU tests), after which every
rank merges them as the top log2(W) levels of the same tree in rank order
(`ssa_merge_roots`) -- the paper's two-level "systolic" reduction
(§3.2) made deterministic.  Because the RNG is keyed by the
global trajectory id, every trajectory and hence the merged grids are bitwise
independent of W.

torch is used only for device buffers and the process group; every step of
the method runs in libssa.so.
"""
from __future__ import annotations

import os
from typing import Callable, Tuple

import torch
import torch.distributed as dist

from .ssa import shard_bounds  # noqa: F401  (aligned-subtree shards, R26)


def env_rank() -> Tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment (1 process = 1 GPU)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def gather_roots(root: torch.Tensor, roots: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather the per-rank moment roots into `roots[W, ...]` in rank order
    (roots[r] = rank r's root).  `root` and `roots[r]` have the same shape;
    both live on the rank's device (CPU tensors under gloo)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if roots.shape[0] != world or roots.shape[1:] != root.shape:
        raise ValueError(f"roots must be [{world}, {tuple(root.shape)}], got {tuple(roots.shape)}")
    if world == 1:
        roots[0].copy_(root)
    else:
        dist.all_gather_into_tensor(roots.view(-1), root.contiguous().view(-1), group=group)
    return roots


def max_and_sum(values, device, group=None):
    """Max over ranks of values[0] (a device time) and the sum of the rest
    (counters): the bench's max-over-ranks timing."""
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        t[0] = tmax[0]
    return [float(v) for v in t.tolist()]


class ShardedEnsemble:
    """One rank's share of a W-GPU ensemble run: `step()` = ssa_run_shard on
    this rank's shard -> all-gather of the roots -> ssa_merge_roots in rank
    order.  `for_model` wires `run_shard(b, e, root)` and `merge(roots, out)`
    to the C-ABI calls; the CPU tests pass stand-ins to exercise the same
    orchestration under gloo."""

    def __init__(self, n_total: int, cells: int, device, run_shard: Callable, merge: Callable, group=None):
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.group = group
        self.n_total, self.cells = n_total, cells
        self.begin, self.end = shard_bounds(n_total, self.world, self.rank)
        self.root = torch.zeros((3, cells), dtype=torch.float64, device=device)
        self.roots = torch.zeros((self.world, 3, cells), dtype=torch.float64, device=device)
        self.out = torch.zeros((4, cells), dtype=torch.float64, device=device)
        self._run_shard = run_shard
        self._merge = merge

    @classmethod
    def for_model(cls, model, n_total: int, t_end: float, sample_dt: float, seed: int, device, *,
                  path: int = 0, stream=None, group=None, **opts) -> "ShardedEnsemble":
        from . import ssa as S
        cells = S.grid_size(t_end, sample_dt) * model.S

        def run_shard(b, e, root):
            return S.run_shard(model, b, e, t_end, sample_dt, seed, root, path=path, stream=stream, **opts)

        def merge(roots, out):
            S.merge_roots(roots, roots.shape[0], cells, stream=stream, out=out)

        return cls(n_total, cells, device, run_shard, merge, group)

    def step(self):
        """Returns this rank's run_shard result (None for an empty shard);
        the merged (mean, var, M2, n) grids are left in `self.out`."""
        res = None
        if self.end > self.begin:
            res = self._run_shard(self.begin, self.end, self.root)
        else:
            self.root.zero_()            # an empty shard is the identity leaf (n = 0)
        gather_roots(self.root, self.roots, self.group)
        self._merge(self.roots, self.out)
        return res
