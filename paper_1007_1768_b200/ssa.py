"""Thin Python binding of libssa.so (include/ssa.h) -- argument marshalling only.

Every step of the method runs in the library's CUDA kernels; this module only
packs arguments into the C structs, calls the C ABI with the same names, and
wraps outputs as numpy arrays (or torch device tensors for the shard/merge
form).  There is no CPU fallback: if libssa.so is missing or no CUDA device is
present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libssa.so")

SSA_OK = 0
SSA_PATH_AUTO, SSA_PATH_THREAD, SSA_PATH_WARP, SSA_PATH_HALFWARP = 0, 1, 2, 3
SSA_REDUCE_MEAN, SSA_REDUCE_VAR = 1, 2
STATUS_NAMES = {0: "SSA_OK", 1: "SSA_ERR_INVALID_ARG", 2: "SSA_ERR_MODEL", 3: "SSA_ERR_NUMERIC",
                4: "SSA_ERR_OVERFLOW", 5: "SSA_ERR_OOM", 6: "SSA_ERR_CUDA", 7: "SSA_ERR_JIT",
                8: "SSA_ERR_UNSUPPORTED"}


class SSAError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class ssa_term(C.Structure):
    _fields_ = [("species", C.c_int32), ("coef", C.c_int32)]


class ssa_reaction(C.Structure):
    _fields_ = [("n_reactants", C.c_int32), ("reactants", C.POINTER(ssa_term)),
                ("n_products", C.c_int32), ("products", C.POINTER(ssa_term)),
                ("rate", C.c_double), ("modifier_species", C.c_int32), ("modifier_coef", C.c_double)]


class ssa_gate(C.Structure):
    _fields_ = [("species", C.c_int32), ("kind", C.c_int32)]


class ssa_reaction_ext(C.Structure):
    _fields_ = [("mass_action", C.c_int32), ("n_gates", C.c_int32), ("gates", C.POINTER(ssa_gate))]


class ssa_traj_summary(C.Structure):
    _fields_ = [("events", C.c_uint64), ("hash", C.c_uint64), ("t_last", C.c_double),
                ("near_ties", C.c_uint64), ("absorbed", C.c_int32), ("status", C.c_int32),
                ("err_reaction", C.c_int32), ("pad", C.c_int32)]


SUMMARY_DTYPE = np.dtype([("events", "<u8"), ("hash", "<u8"), ("t_last", "<f8"), ("near_ties", "<u8"),
                          ("absorbed", "<i4"), ("status", "<i4"), ("err_reaction", "<i4"), ("pad", "<i4")])


class ssa_dump(C.Structure):
    _fields_ = [("n", C.c_uint64), ("ids", C.POINTER(C.c_uint64)), ("states", C.c_void_p),
                ("events_at", C.c_void_p), ("time_at", C.c_void_p), ("summary", C.c_void_p)]


class ssa_run_options(C.Structure):
    _fields_ = [("path", C.c_int32), ("device", C.c_int32), ("stream", C.c_void_p), ("chunk", C.c_uint64),
                ("staging_budget_bytes", C.c_uint64), ("block", C.c_int32), ("blocks_per_sm", C.c_int32),
                ("dump", C.POINTER(ssa_dump)), ("outputs_on_device", C.c_int32), ("tail_lanes", C.c_int32)]


class ssa_result(C.Structure):
    _fields_ = [("mean", C.c_void_p), ("var", C.c_void_p), ("m2", C.c_void_p), ("count", C.c_void_p),
                ("events", C.c_uint64), ("near_ties", C.c_uint64), ("n_errors", C.c_uint64),
                ("first_error_id", C.c_uint64), ("first_error_reaction", C.c_int32), ("path_used", C.c_int32),
                ("device_ms", C.c_double), ("ssa_ms", C.c_double), ("jit_ms", C.c_double),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64), ("kernel_launches", C.c_int32),
                ("pad2", C.c_int32), ("reduce_ms", C.c_double), ("reduce_bytes", C.c_uint64),
                ("dump_ms", C.c_double), ("dump_bytes", C.c_uint64)]


_lib = None


def lib():
    """Load libssa.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run `python -m paper_1007_1768_b200.build`")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        L.ssa_model_create.argtypes = [C.c_int32, P(C.c_int64), C.c_int32, P(ssa_reaction), P(C.c_void_p)]
        L.ssa_model_create.restype = C.c_int
        L.ssa_model_create_ex.argtypes = [C.c_int32, P(C.c_int64), C.c_int32, P(ssa_reaction), P(ssa_reaction_ext),
                                          P(C.c_void_p)]
        L.ssa_model_create_ex.restype = C.c_int
        L.ssa_model_set_names.argtypes = [C.c_void_p, P(C.c_char_p)]
        L.ssa_model_set_names.restype = C.c_int
        L.ssa_model_species_name.argtypes = [C.c_void_p, C.c_int32]
        L.ssa_model_species_name.restype = C.c_char_p
        L.ssa_model_destroy.argtypes = [C.c_void_p]
        L.ssa_model_destroy.restype = None
        L.ssa_model_n_species.argtypes = [C.c_void_p]
        L.ssa_model_n_reactions.argtypes = [C.c_void_p]
        L.ssa_grid_size.argtypes = [C.c_double, C.c_double]
        L.ssa_grid_size.restype = C.c_uint64
        L.ssa_run.argtypes = [C.c_void_p, C.c_uint64, C.c_double, C.c_double, C.c_uint64, C.c_uint32,
                              P(ssa_run_options), P(ssa_result)]
        L.ssa_run.restype = C.c_int
        L.ssa_run_shard.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_uint64,
                                    C.c_void_p, P(ssa_run_options), P(ssa_result)]
        L.ssa_run_shard.restype = C.c_int
        L.ssa_run_sweep.argtypes = [C.c_void_p, C.c_int32, P(C.c_double), P(C.c_double), C.c_uint64, C.c_double,
                                    C.c_double, C.c_uint64, C.c_uint32, P(ssa_run_options), P(ssa_result)]
        L.ssa_run_sweep.restype = C.c_int
        L.ssa_run_union.argtypes = [C.c_void_p, C.c_uint64, C.c_double, C.c_uint64, C.c_uint32, C.c_uint64,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, P(C.c_uint64),
                                    P(ssa_run_options), P(ssa_result)]
        L.ssa_run_union.restype = C.c_int
        L.ssa_run_trajectories.argtypes = [C.c_void_p, C.c_uint64, C.c_double, C.c_uint64, C.c_uint64, C.c_uint64,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, P(C.c_uint64),
                                           P(ssa_run_options), P(ssa_result)]
        L.ssa_run_trajectories.restype = C.c_int
        L.ssa_merge_roots.argtypes = [C.c_void_p, C.c_int32, C.c_uint64, P(ssa_run_options), P(ssa_result)]
        L.ssa_merge_roots.restype = C.c_int
        L.ssa_model_prepare.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
        L.ssa_model_prepare.restype = C.c_int
        L.ssa_status_string.argtypes = [C.c_int]
        L.ssa_status_string.restype = C.c_char_p
        L.ssa_last_error.argtypes = []
        L.ssa_last_error.restype = C.c_char_p
        L.ssa_abi_version.restype = C.c_int32
        L.ssa_debug_k1_source.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int64]
        L.ssa_debug_k1_source.restype = C.c_char_p
        L.ssa_debug_model_hot.argtypes = [C.c_void_p, P(C.c_int32), C.c_int32]
        L.ssa_debug_model_hot.restype = C.c_int32
        L.ssa_debug_k1_compile.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_char_p, C.c_uint64,
                                           P(C.c_uint64)]
        L.ssa_debug_k1_compile.restype = C.c_int
        L.ssa_debug_k2_source.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
        L.ssa_debug_k2_source.restype = C.c_char_p
        L.ssa_debug_k2_compile.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_char_p, C.c_uint64, P(C.c_uint64)]
        L.ssa_debug_k2_compile.restype = C.c_int
        _lib = L
    return _lib


def _check(st: int):
    if st != SSA_OK:
        raise SSAError(st, lib().ssa_last_error().decode(errors="replace"))


def grid_size(t_end: float, dt: float) -> int:
    return int(lib().ssa_grid_size(t_end, dt))


class Model:
    """ssa_model_create over a network description (species, initial counts,
    reactions with reactant/product stoichiometry, rate, optional modifier)."""

    def __init__(self, network):
        self.network = network
        self.S, self.R = network.S, network.R
        keep = []
        rx = (ssa_reaction * max(self.R, 1))()
        for j, r in enumerate(network.reactions):
            reac = (ssa_term * max(len(r.reactants), 1))(*[ssa_term(s, m) for s, m in r.reactants])
            prod = (ssa_term * max(len(r.products), 1))(*[ssa_term(s, m) for s, m in r.products])
            keep += [reac, prod]
            rx[j] = ssa_reaction(len(r.reactants), reac, len(r.products), prod, r.rate,
                                 r.modifier_species, r.modifier_coef)
        x0 = np.ascontiguousarray(np.array(network.x0, dtype=np.int64))
        h = C.c_void_p()
        # gated propensities (NEXT 3): per-reaction extensions only when used
        ext = None
        if any((not getattr(r, "mass_action", True)) or getattr(r, "gates", ()) for r in network.reactions):
            ext = (ssa_reaction_ext * max(self.R, 1))()
            for j, r in enumerate(network.reactions):
                gates = getattr(r, "gates", ())
                garr = (ssa_gate * max(len(gates), 1))(*[ssa_gate(sp, kind) for sp, kind in gates])
                keep.append(garr)
                ext[j] = ssa_reaction_ext(1 if getattr(r, "mass_action", True) else 0, len(gates), garr)
        _check(lib().ssa_model_create_ex(self.S, x0.ctypes.data_as(C.POINTER(C.c_int64)), self.R, rx, ext,
                                         C.byref(h)))
        self.handle = h
        names = getattr(network, "species", None)
        if names:
            arr = (C.c_char_p * self.S)(*[str(n).encode() for n in names])
            _check(lib().ssa_model_set_names(self.handle, arr))

    def species_names(self):
        """The species names attached to the model (ssa_model_species_name)."""
        out = []
        for s in range(self.S):
            v = lib().ssa_model_species_name(self.handle, s)
            out.append(None if v is None else v.decode())
        return out

    def close(self):
        if getattr(self, "handle", None):
            lib().ssa_model_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prepare(self, device: int = -1, path: int = SSA_PATH_AUTO):
        _check(lib().ssa_model_prepare(self.handle, device, path))

    def k1_source(self, block: int = 128, minb: int = 4, dump: bool = False, seed: int = -1, record: int = 0,
                  sweep: bool = False) -> str:
        """Generated K1 source (dump=True: the variant with raw-trajectory dump + hash;
        seed >= 0: the variant with that seed's Philox key schedule compiled in; record 1/2:
        the event-recording / stride-point variants)."""
        flags = int(dump) | (record << 1) | (8 if sweep else 0)
        return lib().ssa_debug_k1_source(self.handle, block, minb, flags, seed).decode()

    def hot_set(self):
        """The K1 hot set measured by this model's first plain thread-path run (None: not yet)."""
        buf = (C.c_int32 * 8)()
        n = lib().ssa_debug_model_hot(self.handle, buf, 8)
        return None if n < 0 else [int(buf[i]) for i in range(min(n, 8))]

    def k2_source(self, block: int = 256, dump: bool = False, half: bool = False) -> str:
        """Generated K2 (warp path; half=True: two trajectories per warp) source."""
        return _k2_source(self, block, int(dump) | (2 if half else 0))

    def k2_compile(self, block: int = 256, dump: bool = False, half: bool = False, minb: int = 1):
        """NVRTC-compile the model's K2 kernel (no device needed); returns (status, log, cubin bytes)."""
        return _k2_compile(self, block, int(dump) | (2 if half else 0) | (min(max(minb, 1), 15) << 4))

    def k1_compile(self, block: int = 128, minb: int = 4, dump: bool = False):
        """NVRTC-compile the model's K1 kernel (no device needed); returns (status, log, cubin bytes)."""
        buf = C.create_string_buffer(1 << 16)
        nb = C.c_uint64()
        st = lib().ssa_debug_k1_compile(self.handle, block, minb, int(dump), buf, len(buf), C.byref(nb))
        return st, buf.value.decode(errors="replace"), nb.value


def _k2_source(model, block: int = 256, flags: int = 0) -> str:
    return lib().ssa_debug_k2_source(model.handle, block, int(flags)).decode()


def _k2_compile(model, block: int = 256, flags: int = 0):
    buf = C.create_string_buffer(1 << 16)
    nb = C.c_uint64()
    st = lib().ssa_debug_k2_compile(model.handle, block, int(flags), buf, len(buf), C.byref(nb))
    return st, buf.value.decode(errors="replace"), nb.value


@dataclass
class Dump:
    ids: np.ndarray            # [n] uint64, sorted
    states: np.ndarray         # [n, G, S] int32
    events_at: np.ndarray      # [n, G] uint64
    time_at: np.ndarray        # [n, G] float64
    summary: np.ndarray        # [n] SUMMARY_DTYPE


@dataclass
class RunResult:
    mean: np.ndarray
    var: np.ndarray
    m2: np.ndarray
    count: np.ndarray
    events: int
    near_ties: int
    n_errors: int
    first_error_id: int
    first_error_reaction: int
    path_used: int
    device_ms: float
    ssa_ms: float
    jit_ms: float
    h2d_bytes: int
    d2h_bytes: int
    kernel_launches: int
    status: int
    dump: Optional[Dump] = None
    reduce_ms: float = 0.0           # device time of the chunk reductions (K3)
    reduce_bytes: int = 0            # staged bytes they read
    dump_ms: float = 0.0             # device time of the dump's D2H copies (host dump arrays)
    dump_bytes: int = 0              # raw-trajectory dump bytes produced


def _options(path=SSA_PATH_AUTO, device=-1, stream=None, chunk=0, staging_budget_bytes=0, block=0,
             blocks_per_sm=0, dump=None, outputs_on_device=False, tail_lanes=0) -> ssa_run_options:
    o = ssa_run_options()
    o.path, o.device, o.chunk, o.staging_budget_bytes = path, device, chunk, staging_budget_bytes
    o.tail_lanes = tail_lanes
    o.stream = stream
    o.block, o.blocks_per_sm = block, blocks_per_sm
    o.outputs_on_device = 1 if outputs_on_device else 0
    if dump is not None:
        o.dump = C.pointer(dump)
    return o


def _host_array(shape, dtype, pinned: bool) -> np.ndarray:
    """Zeroed host array; pinned=True places it in page-locked memory (torch's pinned allocator) so
    the library's device->host copies run at full link speed."""
    dtype = np.dtype(dtype)
    if not pinned:
        return np.zeros(shape, dtype)
    import torch
    nbytes = int(np.prod(shape)) * dtype.itemsize
    buf = torch.zeros(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
    return buf.numpy()[:nbytes].view(dtype).reshape(shape)   # the view keeps the tensor alive


def _make_dump(ids, G, S, pinned: bool = False):
    ids = np.ascontiguousarray(np.asarray(ids, dtype=np.uint64))
    n = len(ids)
    d = Dump(ids, _host_array((n, G, S), np.int32, pinned), _host_array((n, G), np.uint64, pinned),
             _host_array((n, G), np.float64, pinned), _host_array(n, SUMMARY_DTYPE, pinned))
    cd = ssa_dump(n, ids.ctypes.data_as(C.POINTER(C.c_uint64)), d.states.ctypes.data, d.events_at.ctypes.data,
                  d.time_at.ctypes.data, d.summary.ctypes.data)
    return d, cd


def _result_from(r: ssa_result, st: int, mean, var, m2, count, dump=None) -> RunResult:
    return RunResult(mean, var, m2, count, r.events, r.near_ties, r.n_errors, r.first_error_id,
                     r.first_error_reaction, r.path_used, r.device_ms, r.ssa_ms, r.jit_ms, r.h2d_bytes,
                     r.d2h_bytes, r.kernel_launches, st, dump, r.reduce_ms, r.reduce_bytes, r.dump_ms,
                     r.dump_bytes)


def run(model: Model, n_trajectories: int, t_end: float, sample_dt: float, seed: int, *,
        reducers: int = SSA_REDUCE_MEAN | SSA_REDUCE_VAR, path: int = SSA_PATH_AUTO, dump_ids=None,
        dump_pinned: bool = False, raise_on_error: bool = True, **opts) -> RunResult:
    """ssa_run with host outputs: mean/var/m2/count as [G, S] numpy arrays (the dump's arrays in
    page-locked memory with dump_pinned=True)."""
    G = grid_size(t_end, sample_dt)
    S = model.S
    mean = np.zeros((G, S)); var = np.zeros((G, S)); m2 = np.zeros((G, S)); count = np.zeros((G, S))
    dump = cdump = None
    if dump_ids is not None and len(dump_ids):
        dump, cdump = _make_dump(dump_ids, G, S, dump_pinned)
    o = _options(path=path, dump=cdump, **opts)
    r = ssa_result()
    r.mean, r.var, r.m2, r.count = mean.ctypes.data, var.ctypes.data, m2.ctypes.data, count.ctypes.data
    st = lib().ssa_run(model.handle, n_trajectories, t_end, sample_dt, seed, reducers, C.byref(o), C.byref(r))
    if st != SSA_OK and (raise_on_error or st not in (3, 4)):
        _check(st)
    return _result_from(r, st, mean, var, m2, count, dump)


def run_sweep(model: Model, rates, n_per_point: int, t_end: float, sample_dt: float, seed: int, *,
              mod_coefs=None, reducers: int = SSA_REDUCE_MEAN | SSA_REDUCE_VAR, dump_ids=None,
              raise_on_error: bool = True, **opts) -> RunResult:
    """ssa_run_sweep: `rates` is [n_points, R] (and `mod_coefs`, if given);
    returns mean/var/m2/count as [n_points, G, S] numpy arrays.  Dump ids are
    virtual ids p * n_per_point + i."""
    rates = np.ascontiguousarray(np.asarray(rates, dtype=np.float64))
    assert rates.ndim == 2 and rates.shape[1] == model.R
    P = rates.shape[0]
    mc = None
    if mod_coefs is not None:
        mc = np.ascontiguousarray(np.asarray(mod_coefs, dtype=np.float64))
        assert mc.shape == rates.shape
    G = grid_size(t_end, sample_dt)
    S = model.S
    mean, var, m2, count = (np.zeros((P, G, S)) for _ in range(4))
    dump = cdump = None
    if dump_ids is not None and len(dump_ids):
        dump, cdump = _make_dump(dump_ids, G, S)
    o = _options(dump=cdump, **opts)
    r = ssa_result()
    r.mean, r.var, r.m2, r.count = mean.ctypes.data, var.ctypes.data, m2.ctypes.data, count.ctypes.data
    dp = C.POINTER(C.c_double)
    st = lib().ssa_run_sweep(model.handle, P, rates.ctypes.data_as(dp), mc.ctypes.data_as(dp) if mc is not None else None,
                             n_per_point, t_end, sample_dt, seed, reducers, C.byref(o), C.byref(r))
    if st != SSA_OK and (raise_on_error or st not in (3, 4)):
        _check(st)
    return _result_from(r, st, mean, var, m2, count, dump)


@dataclass
class UnionResult:
    times: np.ndarray     # [P]
    mean: np.ndarray      # [P, S]
    var: np.ndarray       # [P, S]
    count: np.ndarray     # [P]
    result: RunResult


def run_union(model: Model, n_trajectories: int, t_end: float, seed: int, thin_kx: int = 1, *,
              capacity: Optional[int] = None, **opts) -> UnionResult:
    """ssa_run_union (selective memory at union times, Avg-Y / Avg-XY).  With
    capacity None the call is made twice: once to learn the number of output
    points, once to fetch them."""
    S = model.S
    if capacity is None:
        n = C.c_uint64()
        r = ssa_result()
        o = _options(**opts)
        st = lib().ssa_run_union(model.handle, n_trajectories, t_end, seed, thin_kx, 0, None, None, None, None,
                                 C.byref(n), C.byref(o), C.byref(r))
        if st not in (SSA_OK, 1):
            _check(st)
        capacity = n.value
    times = np.zeros(max(capacity, 1)); count = np.zeros(max(capacity, 1))
    mean = np.zeros((max(capacity, 1), S)); var = np.zeros((max(capacity, 1), S))
    n = C.c_uint64()
    r = ssa_result()
    o = _options(**opts)
    st = lib().ssa_run_union(model.handle, n_trajectories, t_end, seed, thin_kx, capacity, times.ctypes.data,
                             mean.ctypes.data, var.ctypes.data, count.ctypes.data, C.byref(n), C.byref(o), C.byref(r))
    _check(st)
    P = n.value
    return UnionResult(times[:P], mean[:P], var[:P], count[:P],
                       _result_from(r, st, None, None, None, None))


@dataclass
class TrajectoryPoints:
    traj: np.ndarray      # [P] uint32
    event: np.ndarray     # [P] uint64
    time: np.ndarray      # [P] float64
    states: np.ndarray    # [P, S] int32
    result: RunResult


def run_trajectories(model: Model, n_trajectories: int, t_end: float, seed: int, stride: int = 10, *,
                     capacity: Optional[int] = None, **opts) -> TrajectoryPoints:
    """ssa_run_trajectories (stride-sampled full trajectories).  With capacity
    None the call is made twice: once to learn the number of points."""
    S = model.S
    if capacity is None:
        n = C.c_uint64()
        r = ssa_result()
        o = _options(**opts)
        st = lib().ssa_run_trajectories(model.handle, n_trajectories, t_end, seed, stride, 0, None, None, None, None,
                                        C.byref(n), C.byref(o), C.byref(r))
        if st not in (SSA_OK, 1):
            _check(st)
        capacity = n.value
    cap = max(capacity, 1)
    traj = np.zeros(cap, np.uint32); event = np.zeros(cap, np.uint64); time = np.zeros(cap)
    states = np.zeros((cap, S), np.int32)
    n = C.c_uint64()
    r = ssa_result()
    o = _options(**opts)
    st = lib().ssa_run_trajectories(model.handle, n_trajectories, t_end, seed, stride, capacity, traj.ctypes.data,
                                    event.ctypes.data, time.ctypes.data, states.ctypes.data, C.byref(n), C.byref(o),
                                    C.byref(r))
    _check(st)
    P = n.value
    return TrajectoryPoints(traj[:P], event[:P], time[:P], states[:P], _result_from(r, st, None, None, None, None))


def run_device(model: Model, n_trajectories: int, t_end: float, sample_dt: float, seed: int, out, *,
               path: int = SSA_PATH_AUTO, stream=None, **opts) -> RunResult:
    """ssa_run with device outputs: `out` is a torch CUDA float64 tensor [4, G, S]
    receiving mean, var, m2, count (torch used only for device memory)."""
    o = _options(path=path, stream=stream, outputs_on_device=True, **opts)
    r = ssa_result()
    base = out.data_ptr()
    cells = out.shape[1] * out.shape[2]
    r.mean, r.var, r.m2, r.count = base, base + 8 * cells, base + 16 * cells, base + 24 * cells
    st = lib().ssa_run(model.handle, n_trajectories, t_end, sample_dt, seed, SSA_REDUCE_MEAN | SSA_REDUCE_VAR,
                       C.byref(o), C.byref(r))
    _check(st)
    return _result_from(r, st, None, None, None, None)


def run_shard(model: Model, id_begin: int, id_end: int, t_end: float, sample_dt: float, seed: int, d_root, *,
              path: int = SSA_PATH_AUTO, stream=None, dump_ids=None, raise_on_error: bool = True,
              dump_pinned: bool = False, **opts) -> RunResult:
    """ssa_run_shard: d_root is a torch CUDA float64 tensor [3, G*S] (n, mean, M2).  With
    raise_on_error=False a trajectory error (SSA_ERR_NUMERIC / OVERFLOW) is returned in
    .status instead of raised (the root's mean and M2 are then NaN)."""
    G = grid_size(t_end, sample_dt)
    dump = cdump = None
    if dump_ids is not None and len(dump_ids):
        dump, cdump = _make_dump(dump_ids, G, model.S, dump_pinned)
    o = _options(path=path, stream=stream, dump=cdump, **opts)
    r = ssa_result()
    st = lib().ssa_run_shard(model.handle, id_begin, id_end, t_end, sample_dt, seed, C.c_void_p(d_root.data_ptr()),
                             C.byref(o), C.byref(r))
    if st != SSA_OK and (raise_on_error or st not in (3, 4)):
        _check(st)
    return _result_from(r, st, None, None, None, None, dump)


def merge_roots(d_roots, n_roots: int, cells: int, *, device: int = -1, stream=None, out=None):
    """ssa_merge_roots over [n_roots, 3, cells] device roots.  With `out` (a torch
    CUDA float64 tensor [4, cells]) the outputs stay on the device; otherwise
    numpy arrays (mean, var, m2, count) are returned."""
    o = _options(device=device, stream=stream, outputs_on_device=out is not None)
    r = ssa_result()
    if out is not None:
        base = out.data_ptr()
        r.mean, r.var, r.m2, r.count = base, base + 8 * cells, base + 16 * cells, base + 24 * cells
        _check(lib().ssa_merge_roots(C.c_void_p(d_roots.data_ptr()), n_roots, cells, C.byref(o), C.byref(r)))
        return out
    mean, var, m2, count = (np.zeros(cells) for _ in range(4))
    r.mean, r.var, r.m2, r.count = mean.ctypes.data, var.ctypes.data, m2.ctypes.data, count.ctypes.data
    _check(lib().ssa_merge_roots(C.c_void_p(d_roots.data_ptr()), n_roots, cells, C.byref(o), C.byref(r)))
    return mean, var, m2, count


def shard_bounds(n_total: int, world: int, rank: int):
    """Aligned-subtree shards of the canonical reduction tree (R26):
    span = next_pow2(n_total) / world (world a power of two).  Shards are
    contiguous, in rank order, cover [0, n_total) exactly once, and each is a
    whole subtree of the canonical perfect binary tree over ids."""
    if world < 1 or (world & (world - 1)) != 0:
        raise ValueError("world size must be a power of two (shards are subtrees of a binary tree)")
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    p = 1
    while p < n_total:
        p <<= 1
    span = max(p // world, 1)
    b = min(rank * span, n_total)
    e = min((rank + 1) * span, n_total)
    return b, e
