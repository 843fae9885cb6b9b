"""The N>1 path's host logic under gloo on CPU (world sizes 2 and 4).

The product's multi-GPU orchestration (`paper_1007_1768_b200/dist.py`:
shard_bounds -> per-rank shard run -> all-gather of roots in rank order ->
merge) is exercised with real torch.distributed process groups.  The per-shard
compute is a CPU stand-in (the oracle's exact integer sums n, Σx, Σx² over the
shard's trajectories), so the test checks the orchestration -- which ids each
rank owns, that roots land at index = rank, that empty shards are identities,
and max-over-ranks timing -- against a single-process oracle run over all ids.
The CUDA merge itself is covered by tests/test_gpu_parity.py
(test_shard_merge_equals_single_run)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

import inputs

T_END, DT, SEED, N_TOTAL = 20.0, 1.0, 11, 300      # ragged: next_pow2 = 512


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard_sums(b, e, root):
    """CPU stand-in for ssa_run_shard: exact (n, Σx, Σx²) per grid cell of
    ids [b, e), from the oracle."""
    from oracle import oracle as O
    net = inputs.immigration_death()
    r = O.run(O.OracleModel(net), np.arange(b, e, dtype=np.uint64), SEED, T_END, DT, 0)
    x = r.grid_x.reshape(e - b, -1).astype(np.float64)     # small counts: sums are exact in fp64
    root[0] = float(e - b)
    root[1] = torch.from_numpy(x.sum(axis=0))
    root[2] = torch.from_numpy((x * x).sum(axis=0))
    return {"ids": (b, e), "events": int(r.summaries["events"].sum())}


def _sum_merge(roots, out):
    """CPU stand-in for ssa_merge_roots: roots combined in rank order."""
    acc = torch.zeros_like(roots[0])
    for w in range(roots.shape[0]):
        acc += roots[w]
    out[:3] = acc


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_1007_1768_b200 import dist as D
    r, w, lr = D.env_rank()
    assert (r, w, lr) == (rank, world, rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1007_1768_b200.ssa import grid_size as _g  # noqa: F401  (binding importable without a GPU)
        G = int(np.floor(T_END / DT + 1e-9)) + 1
        ens = D.ShardedEnsemble(N_TOTAL, G * 1, torch.device("cpu"), _shard_sums, _sum_merge)
        res = ens.step()
        t_ms, events = D.max_and_sum([10.0 * (rank + 1), res.local["events"] if res.local else 0],
                                     torch.device("cpu"))
        assert res.events == events and res.status == 0 and res.n_errors == 0
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), roots=ens.roots.numpy(), out=ens.out.numpy(),
                 bounds=np.array([ens.begin, ens.end]), t_ms=t_ms, events=events)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_ensemble_under_gloo(tmp_path, world):
    from oracle import oracle as O
    O.build()
    tmp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="fork")
    outs = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]

    # one single-process oracle run over all ids
    ref = O.run(O.OracleModel(inputs.immigration_death()), np.arange(N_TOTAL, dtype=np.uint64), SEED, T_END, DT, 0)
    x = ref.grid_x.reshape(N_TOTAL, -1).astype(np.float64)
    ev_ref = int(ref.summaries["events"].sum())

    bounds = [tuple(o["bounds"]) for o in outs]
    span = 512 // world
    assert bounds == [(min(r * span, N_TOTAL), min((r + 1) * span, N_TOTAL)) for r in range(world)]
    for o in outs:
        roots = o["roots"]
        for r, (b, e) in enumerate(bounds):
            # root r is rank r's shard (all-gather in rank order); empty shards are identities
            assert roots[r, 0, 0] == e - b
            assert np.array_equal(roots[r, 1], x[b:e].sum(axis=0))
        # every rank holds the same merged grids, equal to the single run
        assert np.array_equal(o["out"][0], np.full(x.shape[1], float(N_TOTAL)))
        assert np.array_equal(o["out"][1], x.sum(axis=0))
        assert np.array_equal(o["out"][2], (x * x).sum(axis=0))
        assert float(o["t_ms"]) == 10.0 * world                 # max over ranks
        assert int(o["events"]) == ev_ref                       # counters summed over ranks
    mean = outs[0]["out"][1] / N_TOTAL
    assert np.allclose(mean, ref.mean.reshape(-1), rtol=1e-12, atol=0)


def test_shard_bounds_rejects_bad_world():
    from paper_1007_1768_b200 import dist as D
    with pytest.raises(ValueError):
        D.shard_bounds(100, 3, 0)
    with pytest.raises(ValueError):
        D.shard_bounds(100, 4, 4)


# ------------------------------------------------------------ fail-safe exchange
def _fail_worker(rank, world, port, outdir):
    """Rank 1's shard fails outright (a library error raised before any
    collective) and rank 2's shard reports trajectory errors; every rank must
    still reach the root all-gather and raise the same error afterwards."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    from paper_1007_1768_b200 import dist as D
    from paper_1007_1768_b200.ssa import SSAError
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def run_shard(b, e, root):
            root[0] = float(e - b)
            root[1:] = 1.0
            if rank == 1:
                raise SSAError(6, "injected CUDA failure")
            n_err = 5 if rank == 2 else 0
            return {"events": 100 + rank, "near_ties": rank, "n_errors": n_err, "status": 3 if n_err else 0,
                    "first_error_id": b + 7 if n_err else 0, "first_error_reaction": 4 if n_err else -1}

        ens = D.ShardedEnsemble(64, 3, torch.device("cpu"), run_shard, _sum_merge)
        try:
            ens.step()
            raised = None
        except SSAError as ex:
            raised = (ex.status, str(ex))
        res = ens.last
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), raised=np.array(raised is not None),
                 status=raised[0] if raised else 0, msg=raised[1] if raised else "",
                 word=np.array([res.status, res.events, res.near_ties, res.n_errors, res.first_error_id,
                                res.first_error_reaction, res.error_rank]), out=ens.out.numpy())
    finally:
        dist.destroy_process_group()


def test_error_on_one_rank_reaches_every_rank(tmp_path):
    world = 4
    tmp.start_processes(_fail_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="fork")
    outs = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    w0 = outs[0]["word"]
    for o in outs:
        assert bool(o["raised"]) and int(o["status"]) == 6          # the non-trajectory failure wins
        assert np.array_equal(o["word"], w0)                      # identical job-wide result on every rank
    # events/ties summed over the ranks that ran; the trajectory errors of rank 2 are still counted
    assert list(w0[:4]) == [6, 100 + 0 + 102 + 103, 0 + 2 + 3, 5]
    assert int(w0[4]) == 32 + 7 and int(w0[5]) == 4 and int(w0[6]) == 1
    # the failed rank's root is NaN (n = 0), so the merged moments are NaN everywhere
    assert np.all(np.isnan(outs[0]["out"][1]))


def _dump_worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    from paper_1007_1768_b200 import dist as D
    from paper_1007_1768_b200.ssa import SUMMARY_DTYPE, Dump
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        G, S = 5, 3
        n = [3, 0, 1, 4][rank]            # uneven, one rank with nothing dumped
        d = None
        if n:
            ids = np.arange(n, dtype=np.uint64) + 100 * rank
            st = (ids[:, None, None] * 1000 + np.arange(G * S).reshape(1, G, S)).astype(np.int32)
            ev = (ids[:, None] + np.arange(G)).astype(np.uint64)
            tm = ev.astype(np.float64) * 0.5
            sm = np.zeros(n, SUMMARY_DTYPE)
            sm["events"] = ids * 3
            sm["hash"] = ids ^ 0xABCDEF
            d = Dump(ids, st, ev, tm, sm)
        for dst in (0, None):
            g = D.gather_dump(d, torch.device("cpu"), dst=dst)
            if g is not None:
                np.savez(os.path.join(outdir, f"rank{rank}_{dst}.npz"), ids=g.ids, states=g.states,
                         events_at=g.events_at, time_at=g.time_at, ev=g.summary["events"], hash=g.summary["hash"])
    finally:
        dist.destroy_process_group()


def test_gather_dump_rank_order(tmp_path):
    world = 4
    tmp.start_processes(_dump_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="fork")
    ids = np.concatenate([np.arange(n, dtype=np.uint64) + 100 * r for r, n in enumerate([3, 0, 1, 4])])
    files = sorted(os.listdir(tmp_path))
    assert files == ["rank0_0.npz", "rank0_None.npz", "rank1_None.npz", "rank2_None.npz", "rank3_None.npz"]
    for f in files:
        g = np.load(tmp_path / f)
        assert np.array_equal(g["ids"], ids)
        assert np.array_equal(g["states"][:, 2, 1], (ids * 1000 + 7).astype(np.int32))
        assert np.array_equal(g["events_at"][:, 4], ids + 4)
        assert np.array_equal(g["time_at"], g["events_at"].astype(np.float64) * 0.5)
        assert np.array_equal(g["ev"], ids * 3) and np.array_equal(g["hash"], ids ^ 0xABCDEF)
