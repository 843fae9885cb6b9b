"""The N>1 path with the REAL libssa.so in several processes (
PAPER.md:133-135 §3.2, the two-level "systolic" reduction).

Two (and four) processes share the one GPU of the test box; the process group
is gloo and the device roots, status words and dumps are staged through host
memory (dist.py).  No kernel of one rank waits on another rank: each rank runs
its own shard through ssa_run_shard and the exchange is host-side, so this is
the multi-GPU orchestration exactly as it runs over NCCL, minus the transport.
Checked: the merged grids on every rank are bitwise those of one ssa_run over
all ids; the job-wide counters equal the single run's; the rank-order dump
gather equals the single run's dump; and a numeric error is reported
identically by every rank (and matches the single run's first error)."""
import os
import socket

import numpy as np
import pytest

import inputs
from inputs.networks import Network, _rx

pytestmark = pytest.mark.gpu

THREAD = 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _error_net():
    """X immigrates and decays; the modified rate of a zero-propensity
    reaction Y -> Y is k^ = 0 + 1e308 * X, which overflows to +inf once X
    reaches 2, and inf * C(Y=0, 1) = NaN is a non-finite propensity
     -- so only the trajectories that reach X = 2 fail."""
    return Network(("X", "Y"), (0, 0), (
        _rx([], [(0, 1)], 0.4),
        _rx([(0, 1)], [], 1.0),
        _rx([(1, 1)], [(1, 1)], 0.0, mod=(0, 1e308)),
    ), "error-injection")


CASES = {
    # name: (network, n_total, t_end, dt, seed, dump every k-th id)
    "c1": (lambda: inputs.config(1).network, 3000, 20.0, 0.1, 2, 7),
    "hiv": (lambda: inputs.config(2).network, 200, 4.0, 1.0, 3, 3),
    "err": (_error_net, 1000, 3.0, 0.5, 9, 0),
}


def _worker(rank, world, port, outdir, case):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK="0")
    import torch
    import torch.distributed as dist
    from paper_1007_1768_b200 import dist as D
    from paper_1007_1768_b200 import ssa as S
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mk, n, t_end, dt, seed, every = CASES[case]
        net = mk()
        m = S.Model(net)
        ids = np.arange(0, n, every, dtype=np.uint64) if every else None
        ens = D.ShardedEnsemble.for_model(m, n, t_end, dt, seed, "cuda:0", path=THREAD, dump_ids=ids)
        raised = None
        try:
            res = ens.step()
        except S.SSAError as ex:
            raised = (ex.status, str(ex))
            res = ens.last
        g = D.gather_dump(res.local.dump if res.local is not None else None, torch.device("cuda:0"), dst=None)
        out = ens.out.cpu().numpy()
        np.savez(os.path.join(outdir, f"{case}_{world}_{rank}.npz"), out=out,
                 word=np.array([res.status, res.events, res.near_ties, res.n_errors, res.first_error_id,
                                res.first_error_reaction]), raised=np.array(raised is not None),
                 status=raised[0] if raised else 0,
                 gids=g.ids if g is not None else np.zeros(0, np.uint64),
                 gstates=g.states if g is not None else np.zeros(0, np.int32),
                 gev=g.events_at if g is not None else np.zeros(0, np.uint64),
                 gt=g.time_at if g is not None else np.zeros(0),
                 ghash=g.summary["hash"] if g is not None else np.zeros(0, np.uint64))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def S():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1007_1768_b200 import build
    build.build()
    from paper_1007_1768_b200 import ssa
    return ssa


def _spawn(case, world, tmp_path):
    import torch.multiprocessing as tmp
    tmp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), case), nprocs=world,
                        start_method="spawn")
    return [np.load(tmp_path / f"{case}_{world}_{r}.npz") for r in range(world)]


@pytest.mark.parametrize("case,world", [("c1", 2), ("c1", 4), ("hiv", 2)])
def test_real_lib_sharded_equals_single_run(S, tmp_path, case, world):
    mk, n, t_end, dt, seed, every = CASES[case]
    net = mk()
    ids = np.arange(0, n, every, dtype=np.uint64)
    ref = S.run(S.Model(net), n, t_end, dt, seed, path=THREAD, dump_ids=ids)
    G = S.grid_size(t_end, dt)
    outs = _spawn(case, world, tmp_path)
    for o in outs:
        out = o["out"].reshape(4, G, net.S)
        assert np.array_equal(out[0], ref.mean) and np.array_equal(out[1], ref.var)     # bitwise, every rank
        assert np.array_equal(out[2], ref.m2) and np.array_equal(out[3], ref.count)
        w = o["word"]
        assert int(w[0]) == 0 and int(w[1]) == ref.events and int(w[2]) == ref.near_ties and int(w[3]) == 0
        # the rank-order dump gather is the single run's dump
        assert np.array_equal(o["gids"], ids)
        assert np.array_equal(o["gstates"], ref.dump.states)
        assert np.array_equal(o["gev"], ref.dump.events_at)
        assert np.array_equal(o["gt"], ref.dump.time_at)
        assert np.array_equal(o["ghash"], ref.dump.summary["hash"])


def test_real_lib_numeric_error_on_every_rank(S, tmp_path):
    """Trajectory errors (SSA_ERR_NUMERIC) in the shards: no rank blocks, every
    rank raises the same status with the single run's first erroring id,
    reaction and error count, and the merged moments are NaN."""
    mk, n, t_end, dt, seed, _ = CASES["err"]
    net = mk()
    ref = S.run(S.Model(net), n, t_end, dt, seed, path=THREAD, raise_on_error=False)
    assert ref.status == 3 and 0 < ref.n_errors < n              # the injection hits some trajectories only
    assert np.all(np.isnan(ref.mean)) and np.all(ref.count == n)
    outs = _spawn("err", 2, tmp_path)
    for o in outs:
        assert bool(o["raised"]) and int(o["status"]) == 3
        w = o["word"]
        assert int(w[0]) == 3 and int(w[3]) == ref.n_errors
        assert int(w[4]) == ref.first_error_id and int(w[5]) == ref.first_error_reaction == 2
        assert int(w[1]) == ref.events
        assert np.all(np.isnan(o["out"][0]))
