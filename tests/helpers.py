"""Test helpers: parallel oracle replay and comparison rules."""
from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

REL_MOMENTS = 1e-9   # north_star: mean/variance grids within 1e-9 relative


def _oracle_chunk(args):
    net, ids, seed, t_end, dt, mode = args
    from oracle import oracle as O
    r = O.run(O.OracleModel(net), ids, seed, t_end, dt, mode)
    return r.grid_x, r.grid_e, r.grid_t, r.summaries, r.status


_CTX = None


def _pool_context():
    """Worker processes come from a fork server started before any CUDA or torch threads exist in
    it (forking the multi-threaded test process itself is unsafe once CUDA is initialised)."""
    global _CTX
    if _CTX is None:
        _CTX = mp.get_context("forkserver")
        _CTX.set_forkserver_preload(["numpy", "oracle.oracle", "tests.helpers"])
    return _CTX


def oracle_replay(net, ids, seed, t_end, dt, mode, procs=None):
    """Run the oracle on `ids` in parallel worker processes; returns
    (grid_x [n,G,S], grid_e [n,G], grid_t [n,G], summaries [n])."""
    ids = np.asarray(ids, dtype=np.uint64)
    procs = procs or max(1, min(len(ids), os.cpu_count() or 1))
    parts = [p for p in np.array_split(ids, procs * 4) if len(p)]
    if procs == 1 or len(parts) == 1:
        outs = [_oracle_chunk((net, p, seed, t_end, dt, mode)) for p in parts]
    else:
        with _pool_context().Pool(procs) as pool:
            outs = pool.map(_oracle_chunk, [(net, p, seed, t_end, dt, mode) for p in parts])
    gx = np.concatenate([o[0] for o in outs])
    ge = np.concatenate([o[1] for o in outs])
    gt = np.concatenate([o[2] for o in outs])
    sm = np.concatenate([o[3] for o in outs])
    return gx, ge, gt, sm


def exact_moments(grid_x):
    from oracle import oracle as O
    n = grid_x.shape[0]
    mean, var = O.moments(grid_x.reshape(n, -1))
    return mean.reshape(grid_x.shape[1:]), var.reshape(grid_x.shape[1:])


def assert_moments_close(gpu_mean, gpu_var, ref_mean, ref_var, rel=REL_MOMENTS):
    for name, g, r in (("mean", gpu_mean, ref_mean), ("var", gpu_var, ref_var)):
        zero = r == 0
        assert np.all(g[zero] == 0), f"{name}: exact zeros not reproduced"
        err = np.abs(g - r) / np.maximum(np.abs(r), 1e-300)
        err[zero] = 0
        assert err.max() <= rel, f"{name}: max rel err {err.max():.3e} at {np.unravel_index(err.argmax(), err.shape)}"


def assert_dump_equal(dump, gx, ge, gt, sm, check_times=True):
    assert np.array_equal(dump.states, gx), f"states differ at {np.argwhere(dump.states != gx)[:5]}"
    assert np.array_equal(dump.events_at, ge), "events_at differ"
    assert np.array_equal(dump.summary["events"], sm["events"]), "event totals differ"
    assert np.array_equal(dump.summary["hash"], sm["hash"]), "firing hashes differ"
    assert np.array_equal(dump.summary["absorbed"], sm["absorbed"]), "absorbed flags differ"
    assert np.array_equal(dump.summary["near_ties"], sm["near_ties"]), "near-tie counts differ"
    if check_times:
        # plog is pinned on both sides: event times are bit-identical
        assert np.array_equal(dump.time_at, gt), "event times differ"
        assert np.array_equal(dump.summary["t_last"], sm["t_last"]), "t_last differ"
