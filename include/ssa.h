/*
 * ssa.h -- C ABI of the B200 ensemble-SSA engine (libssa.so).
 *
 * The hot path of StochKit-FF (arxiv/paper_1007_1768): many independent
 * Gillespie direct-method trajectories of a mass-action reaction network
 * (§2, "The Gillespie's algorithm determines the next transition
 * and the time at which it occurs"), each aligned online to a common sample
 * grid and reduced across trajectories to per-species mean and variance --
 * the paper's "selective memory" (§3.2.1), here on a fixed grid
 * (BASELINE.json north_star).  The call names follow the paper's statement of
 * the problem: a model is parameters + integer state vector + stoichiometric
 * matrix + propensity vector (§3.2), StochRxn_ff() runs copies of
 * one simulation and reduces them online (§3.2).
 *
 * Conventions for every entry point:
 *  - No exceptions cross the ABI; every call returns an ssa_status.  On error,
 *    ssa_last_error() returns a thread-local message with the detail
 *    (validation message, trajectory id and reaction of a numeric error,
 *    CUDA/NVRTC error string).
 *  - Host pointers are only read during the call; the library keeps no
 *    reference to caller memory after returning (ssa_model_create deep-copies).
 *  - All compute runs on the CUDA device in hand-written sm_100a kernels; the
 *    library has no CPU fallback.  Without a usable CUDA device ssa_run
 *    returns SSA_ERR_CUDA.
 *  - Results are bitwise deterministic for a given (model, N, t_end, dt,
 *    seed, path): independent of chunk size, block size, scheduling and of how
 *    trajectories are sharded over GPUs.
 */
#ifndef SSA_H
#define SSA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SSA_OK = 0,
    SSA_ERR_INVALID_ARG = 1,  /* bad argument (null pointer, t_end <= 0, dt <= 0, N == 0, ...) */
    SSA_ERR_MODEL = 2,        /* invalid model (bad species index, coef < 1, rate < 0 or non-finite, ...) */
    SSA_ERR_NUMERIC = 3,      /* a trajectory met a non-finite propensity */
    SSA_ERR_OVERFLOW = 4,     /* a sampled species count exceeded INT32_MAX */
    SSA_ERR_OOM = 5,          /* device allocation failed */
    SSA_ERR_CUDA = 6,         /* CUDA runtime error (no device, launch failure, ...) */
    SSA_ERR_JIT = 7,          /* NVRTC compilation of the model-specialised kernel failed */
    SSA_ERR_UNSUPPORTED = 8   /* valid model the requested path cannot run */
} ssa_status;

/* ------------------------------------------------------------------ model */
/* One stoichiometric term: `coef` molecules of species `species` (coef >= 1). */
typedef struct {
    int32_t species;
    int32_t coef;
} ssa_term;

/* One reaction (a column of the stoichiometric matrix + its propensity,
 * PAPER.md:157).  Mass action: a_j = k^_j * prod_reactants C(x_s, coef)
 * (unordered combinations, R1); the total reactant order is <= 3 and
 * each species appears at most once among the reactants (and once among the
 * products).  Optional linear modifier (beta_R5 = beta - K*F):
 *   k^_j = max(0, rate + modifier_coef * x[modifier_species]),
 * modifier_species = -1 for none. */
typedef struct {
    int32_t n_reactants;
    const ssa_term* reactants;
    int32_t n_products;
    const ssa_term* products;
    double rate;
    int32_t modifier_species;
    double modifier_coef;
} ssa_reaction;

typedef struct ssa_model ssa_model;

/* Validate and deep-copy a model.  initial_counts: [n_species], each in
 * [0, INT32_MAX].  n_species in [1, 16383]; n_reactions in [0, 65535] (0 is
 * valid: the state is held).  On success *out owns the model;
 * release it with ssa_model_destroy.  Errors: SSA_ERR_INVALID_ARG (null
 * pointers), SSA_ERR_MODEL (with the reason in ssa_last_error()).  The model
 * is immutable and may be used from several threads at once.  (The library
 * caches compiled kernels and a dispatch profile per model -- the reactions
 * that dominate its event stream, measured by its first thread-path run; they
 * change speed only, never results.) */
ssa_status ssa_model_create(int32_t n_species, const int64_t* initial_counts, int32_t n_reactions,
                            const ssa_reaction* reactions, ssa_model** out);
/* Gated propensities (the paper's time-triggered
 * mutation, "a stochastic event expected to occur at about a
 * given time", as SPEC.md:424's mu*step(V5)*(1-step(V4)); R33).
 * Per reaction: mass_action = 1 keeps h = prod C(x_s, m_s) over the
 * reactants; 0 makes h = 1 (the reactants then only set the stoichiometry).
 * Each gate multiplies the propensity by an indicator: SSA_GATE_POSITIVE is
 * [x_species > 0] (step), SSA_GATE_ZERO is [x_species == 0] (1 - step).  A
 * closed gate makes a_j exactly 0; an open one leaves k^ * h unchanged. */
enum { SSA_GATE_POSITIVE = 0, SSA_GATE_ZERO = 1 };
typedef struct {
    int32_t species;
    int32_t kind;          /* SSA_GATE_POSITIVE or SSA_GATE_ZERO */
} ssa_gate;
typedef struct {
    int32_t mass_action;   /* 1 (default) or 0 */
    int32_t n_gates;       /* 0..4 */
    const ssa_gate* gates; /* [n_gates], may be NULL when n_gates == 0 */
} ssa_reaction_ext;

/* ssa_model_create with optional per-reaction extensions: ext is NULL (every
 * reaction mass action, no gates: the same as ssa_model_create) or an array
 * of n_reactions entries (deep-copied).  Errors as ssa_model_create, plus
 * SSA_ERR_MODEL for a gate species out of range, an unknown gate kind or more
 * than 4 gates. */
ssa_status ssa_model_create_ex(int32_t n_species, const int64_t* initial_counts, int32_t n_reactions,
                               const ssa_reaction* reactions, const ssa_reaction_ext* ext, ssa_model** out);
/* Species names (SURVEY.md §8(b)'s nullable `names`; the paper's models name their species,
 * e.g. Table 1's U0, U, T, Z4, Z5, I4, I5, V4, V5, F): attach n_species
 * NUL-terminated names (deep-copied) to a model, or NULL to clear them.  Names are labels
 * only; no computation reads them.  Errors: SSA_ERR_INVALID_ARG (null model, a null name). */
ssa_status ssa_model_set_names(ssa_model* model, const char* const* names);
/* The name of species `index`, or NULL if none was set or index is out of range.  The
 * pointer stays valid until the model is destroyed or its names are set again. */
const char* ssa_model_species_name(const ssa_model* model, int32_t index);
void ssa_model_destroy(ssa_model* model);
int32_t ssa_model_n_species(const ssa_model* model);
int32_t ssa_model_n_reactions(const ssa_model* model);

/* Number of grid points G = K + 1, K = floor(t_end/sample_dt + 1e-9); grid
 * times s_k = k * sample_dt (R15).  Returns 0 for invalid input. */
uint64_t ssa_grid_size(double t_end, double sample_dt);

/* --------------------------------------------------------------- options */
/* THREAD: one trajectory per thread, sequential summation order; WARP: one
 * trajectory per warp, order warp32; HALFWARP: two trajectories per warp
 * (16 lanes each), order warp16s (R34; the oracle's mode 3).  The order
 * fixes the rounding of the total and of the selection, so results are bitwise
 * reproducible per path (result->path_used reports it). */
enum { SSA_PATH_AUTO = 0, SSA_PATH_THREAD = 1, SSA_PATH_WARP = 2, SSA_PATH_HALFWARP = 3 };
enum { SSA_REDUCE_MEAN = 1, SSA_REDUCE_VAR = 2 };

/* Per-trajectory record of a dumped trajectory (a11). */
typedef struct {
    uint64_t events;       /* applied events (event time <= s_K) */
    uint64_t hash;         /* h = (h ^ j) * 0x100000001b3 over fired reactions j, from 0xcbf29ce484222325 */
    double t_last;         /* time of the last applied event (0 if none) */
    uint64_t near_ties;    /* grid crossings with an event within 1e-9 relative of s_k */
    int32_t absorbed;      /* 1 if a0 == 0 was reached before s_K */
    int32_t status;        /* SSA_OK, SSA_ERR_NUMERIC or SSA_ERR_OVERFLOW */
    int32_t err_reaction;  /* reaction index of a non-finite propensity, else -1 */
    int32_t pad;
} ssa_traj_summary;

/* Optional raw-trajectory dump for checking ("the worker can
 * directly write the full simulation results").  ids: host array, sorted
 * ascending, unique, each < N (or inside [id_begin, id_end) for a shard).
 * Output arrays are caller-allocated, host or device memory according to
 * ssa_run_options.outputs_on_device; any may be NULL. Layouts:
 *   states    [n][G][S] int32  held state at s_k
 *   events_at [n][G]   uint64  events applied up to s_k
 *   time_at   [n][G]   double  time of the last applied event <= s_k (0 if none)
 *   summary   [n]              per-trajectory record */
typedef struct {
    uint64_t n;
    const uint64_t* ids;
    int32_t* states;
    uint64_t* events_at;
    double* time_at;
    ssa_traj_summary* summary;
} ssa_dump;

typedef struct {
    int32_t path;                  /* SSA_PATH_*: AUTO picks THREAD for R <= 160, HALFWARP for R <= 256, else WARP */
    int32_t device;                /* CUDA device ordinal; -1 = the calling thread's current device */
    void* stream;                  /* cudaStream_t to run on; NULL = a library-owned stream */
    uint64_t chunk;                /* trajectories per chunk (power of two); 0 = auto */
    uint64_t staging_budget_bytes; /* cap on the per-chunk staging buffer; 0 = 32 GiB */
    int32_t block;                 /* threads per block for K1 / K2; 0 = default */
    int32_t blocks_per_sm;         /* resident blocks per SM for K1 / K2; 0 = occupancy maximum */
    const ssa_dump* dump;          /* NULL = no dump */
    int32_t outputs_on_device;     /* 1: ssa_result arrays and dump arrays are device pointers */
    int32_t tail_lanes;            /* thread path, end of a launch: once no ids are left, the trajectories of a
                                      warp with at most this many live lanes are suspended at their next grid
                                      point and resumed packed into whole warps by a follow-up launch (tail
                                      compaction); 0 = default (off), -1 = off.  Speed only: results are
                                      bitwise the same for every value. */
} ssa_run_options;

/* Result.  The caller sets the output arrays (any may be NULL), each [G*S]
 * with cell (k, s) at k*S + s; the call fills the rest. */
typedef struct {
    double* mean;              /* ensemble mean */
    double* var;               /* population variance M2/n (R18) */
    double* m2;                /* sum of squared deviations */
    double* count;             /* n per cell */
    uint64_t events;           /* applied events over all trajectories */
    uint64_t near_ties;        /* grid crossings flagged as near ties (informational) */
    uint64_t n_errors;         /* trajectories that ended in SSA_ERR_NUMERIC / OVERFLOW */
    uint64_t first_error_id;   /* smallest erroring trajectory id (if n_errors > 0) */
    int32_t first_error_reaction; /* its reaction (numeric errors), else -1 */
    int32_t path_used;         /* SSA_PATH_THREAD, _WARP or _HALFWARP (fixes the summation order) */
    double device_ms;          /* device time of simulation + reduction (CUDA events) */
    double ssa_ms;             /* device time inside the SSA kernels (K1/K2) */
    double jit_ms;             /* host time spent compiling the K1 kernel in this call (0 if cached) */
    uint64_t h2d_bytes;        /* host->device bytes copied by this call (model tables, dump ids) */
    uint64_t d2h_bytes;        /* device->host bytes copied by this call (results, dump, counters) */
    int32_t kernel_launches;   /* kernels this call launched (SSA + reduction + finalize) */
    int32_t pad2;
    double reduce_ms;          /* device time of the chunk reductions (K3 + tile merges, CUDA events) */
    uint64_t reduce_bytes;     /* staged sample bytes those reductions read (4 per trajectory x grid cell) */
    double dump_ms;            /* device time of the dump's device->host copies (CUDA events; 0 when the dump
                                  arrays are device memory or there is no dump) */
    uint64_t dump_bytes;       /* bytes of raw-trajectory dump produced (states, events_at, time_at, summaries) */
} ssa_result;

/* StochRxn_ff on one GPU: simulate trajectories 0..n_trajectories-1 on
 * [0, t_end], align each to the grid, reduce to mean/variance.  seed keys the
 * Philox stream: trajectory i's event e uses counter (e, i) and key seed, so
 * any trajectory is reproducible in isolation.  reducers: SSA_REDUCE_MEAN |
 * SSA_REDUCE_VAR (both are always computed; the flags only gate the copies).
 * Returns the first error by trajectory id: SSA_ERR_NUMERIC/OVERFLOW (detail
 * in result->first_error_*), or an argument/CUDA/JIT error.  When any
 * trajectory ends in SSA_ERR_NUMERIC/OVERFLOW the whole ensemble has no
 * defined moments: mean, var and m2 are written as NaN (count is still
 * written, the counters and the dump are valid). */
ssa_status ssa_run(const ssa_model* model, uint64_t n_trajectories, double t_end, double sample_dt,
                   uint64_t seed, uint32_t reducers, const ssa_run_options* opts, ssa_result* result);

/* Multi-process form (one process per GPU; the workers of the paper's
 * two-level "systolic" reduction, §3.2 -- each reduces its
 * own simulations before the collector merges the partials): simulate ids
 * [id_begin, id_end) and write their subtree root of the canonical reduction
 * tree to d_root (DEVICE memory, caller-owned, [3][G*S] doubles: n, mean,
 * M2).  (id_end - id_begin) must be >= 1 and id_begin a multiple of the next
 * power of two >= (id_end - id_begin), so the shard is an aligned subtree
 * (R26).  result's output arrays are ignored; its counters are
 * filled (this shard's only: the caller exchanges them, paper_1007_1768_b200/
 * dist.py).  Errors as ssa_run; on SSA_ERR_NUMERIC/OVERFLOW the root's mean
 * and M2 rows are NaN, so any merge that includes it is NaN. */
ssa_status ssa_run_shard(const ssa_model* model, uint64_t id_begin, uint64_t id_end, double t_end,
                         double sample_dt, uint64_t seed, double* d_root, const ssa_run_options* opts,
                         ssa_result* result);

/* Parameter sweep: StochRxn_ff's "set of parameter-swept simulations"
 * (§3.2), e.g. the delta_t sensitivity analysis of Fig. 4 panels
 * 2-4.  n_points parameter points, each a full vector of
 * rate constants: rates[p*R + j] (HOST, finite, >= 0) and, optionally,
 * modifier coefficients mod_coefs[p*R + j] (HOST, finite; NULL = the model's).
 * The model supplies species, stoichiometry, modifier species and initial
 * counts.  Every point simulates trajectories 0..n_per_point-1 with the same
 * seed (common random numbers across points, R31), so point p's
 * grids are bitwise those of ssa_run (thread path) on the model with point
 * p's constants.
 * result->mean/var/m2/count are [n_points][G*S] (host, or device with
 * opts->outputs_on_device); the counters are totals over all points.  Dump ids
 * (opts->dump) are virtual ids p*n_per_point + i.  Runs on the thread path
 * at any size (AUTO included; an explicit WARP or HALFWARP path is
 * SSA_ERR_UNSUPPORTED); the points whose staging fits the
 * budget run in one kernel launch.  Errors as ssa_run (first_error_id is the
 * virtual id). */
ssa_status ssa_run_sweep(const ssa_model* model, int32_t n_points, const double* rates, const double* mod_coefs,
                         uint64_t n_per_point, double t_end, double sample_dt, uint64_t seed, uint32_t reducers,
                         const ssa_run_options* opts, ssa_result* result);

/* Selective memory at union times (PAPER.md:143-149
 * §3.2.1, Fig. 3): simulate trajectories 0..n-1 on
 * [0, t_end] (thread path), align them at EVERY distinct event time of the
 * ensemble (the union times, plus 0 and t_end) by zero-order hold -- Avg-Y,
 * with equal union times collapsed into one slice -- and reduce thin_kx
 * successive aligned slices along time -- Avg-XY (thin_kx = 1: Avg-Y itself).
 * Output point p: times[p] = mean of its slices' times (left-to-right sum /
 * count), mean[p*S + s], var[p*S + s] (population), count[p] = n * slices.
 * The output has ceil(slices / thin_kx) points; capacity is the number of
 * points the caller's arrays hold (host, or device with
 * opts->outputs_on_device).  *n_points always receives the number of points;
 * if it exceeds capacity the call returns SSA_ERR_INVALID_ARG and writes
 * nothing (call again with a larger capacity).  Work: the ensemble runs
 * twice (event counts, then recording) and every event is stored (~24 B)
 * and sorted; n is at most 2^24.  DESIGN.md §8d. */
ssa_status ssa_run_union(const ssa_model* model, uint64_t n_trajectories, double t_end, uint64_t seed,
                         uint32_t thin_kx, uint64_t capacity, double* times, double* mean, double* var,
                         double* count, uint64_t* n_points, const ssa_run_options* opts, ssa_result* result);

/* Full-trajectory output with stride sampling (
 * PAPER.md:133 "the worker can directly write the full simulation results",
 * PAPER.md:175 "a 1:10 sampling (outputting 1 simulation point every 10)";
 * SPEC.md:162 Stride(s)): simulate trajectories 0..n-1 on [0, t_end] (thread
 * path) and return, ordered by trajectory then time, the points (0, x0), the
 * state after every stride-th applied event, and the horizon point (t_end,
 * held state) unless the last point is already at t_end.  Row p: traj[p],
 * event[p] (events applied up to the point; the horizon point carries the
 * total), time[p], states[p*S + s] (int32).  capacity, n_points and errors
 * as ssa_run_union (host arrays, or device with opts->outputs_on_device);
 * result->d2h_bytes counts the output copied to the host, result->reduce_ms
 * the sort + gather.  n is at most 2^23. */
ssa_status ssa_run_trajectories(const ssa_model* model, uint64_t n_trajectories, double t_end, uint64_t seed,
                                uint64_t stride, uint64_t capacity, uint32_t* traj, uint64_t* event, double* time,
                                int32_t* states, uint64_t* n_points, const ssa_run_options* opts,
                                ssa_result* result);

/* The collector of the paper's two-level reduction (§3.2: "a
 * systolic reduction of partial results"), made deterministic: merge n_roots
 * shard roots (DEVICE memory, contiguous [n_roots][3][cells], in rank order,
 * each an aligned subtree of equal span) as the top levels of the canonical
 * tree, then finalize into result->mean/var/m2/count (host or device per
 * opts->outputs_on_device).  Every rank obtains bitwise identical output.
 * Reads d_roots only during the call, on opts->stream (NULL: a library
 * stream, synchronised with the device before reading -- pass the stream the
 * all-gather was ordered on).  Errors: SSA_ERR_INVALID_ARG (null pointer,
 * n_roots < 1, cells == 0), SSA_ERR_CUDA. */
ssa_status ssa_merge_roots(const double* d_roots, int32_t n_roots, uint64_t cells, const ssa_run_options* opts,
                           ssa_result* result);

/* Compile (NVRTC) and load the model's seed-independent kernel for a device
 * ahead of time (K2, or K1 with the Philox keys as launch parameters) and
 * check that it builds.  path as in ssa_run_options.  The thread path still
 * compiles, once per model, device and seed, a variant with the seed's Philox
 * round keys as instruction immediates, and after a model's first plain run a
 * variant specialised on its measured dispatch profile; both are cached. */
ssa_status ssa_model_prepare(const ssa_model* model, int32_t device, int32_t path);

const char* ssa_status_string(ssa_status status);
const char* ssa_last_error(void);
int32_t ssa_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SSA_H */
