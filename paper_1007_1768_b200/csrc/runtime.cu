// runtime.cu -- the C-ABI library (include/ssa.h): model validation and
// packing, NVRTC specialisation of K1, chunked launch of the SSA kernels and
// of the canonical-tree reduction, shard/merge entry points.
//
// Host code only (compiled by nvcc so that it can share the device record
// layouts of ssa_device.cuh); all arithmetic of the method runs in the
// kernels (k1_thread.cuh via NVRTC, kernels.cu).
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <tuple>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/ssa.h"
#include "embedded_src.h"
#include "ssa_device.cuh"
#include "ssa_kernels.h"

static_assert(sizeof(ssa_dev_summary) == sizeof(ssa_traj_summary), "summary layout");

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;

static ssa_status fail(ssa_status st, const char* fmt, ...)
{
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

#define CU(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return fail(e_ == cudaErrorMemoryAllocation ? SSA_ERR_OOM : SSA_ERR_CUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(e_), __FILE__, __LINE__);                        \
    } while (0)

#define TRY(expr)                                                                                  \
    do {                                                                                           \
        ssa_status s_ = (expr);                                                                    \
        if (s_ != SSA_OK) return s_;                                                               \
    } while (0)

// ------------------------------------------------------------------ model
// K1 phases per trajectory (time slicing, k1_thread.cuh); profiles/r2z_seg_ab.txt
#define SSA_TSLICES 32

struct RxI {
    std::vector<std::pair<int, int>> reac;   // (species, coef) in declared order
    std::vector<std::pair<int, long long>> nu; // nonzero net change, species ascending
    double rate = 0.0;
    int mod_sp = -1;
    double mod_coef = 0.0;
    bool mass_action = true;                   // false: h = 1 (gated propensities, NEXT 3)
    std::vector<std::pair<int, int>> gates;    // (species, SSA_GATE_POSITIVE | SSA_GATE_ZERO)
};

struct K1Entry {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t fn = nullptr;
    int block = 0, minb = 0;
    int blocks_per_sm = 0;
    void *c_k = nullptr, *c_x0 = nullptr;  // module constant memory
    std::string log;
};

struct K2Kernel {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t fn = nullptr;
    size_t smem = 0;
    size_t rxd_offset = 0;
    size_t rec_offset = 0, dent_offset = 0;   // half-warp layout
    int blocks_per_sm = 0;
};

struct K2Dev {
    bool ready = false;
    int P = 0, n_ent = 0, n_dep = 0;
    void* dev_image = nullptr;   // one device block holding the tables below
    void* host_image = nullptr;  // its page-locked host image
    size_t image_bytes = 0;
    ssa_u64* pk = nullptr;
    ssa_u64* gw = nullptr;
    double *rate = nullptr, *modc = nullptr, *x0 = nullptr;
    int *nu_off = nullptr, *nu_ent = nullptr;
    int *dep_off = nullptr, *dep_ent = nullptr;
    int4* rec = nullptr;                    // half-warp path: per-reaction {nu b, nu e, dep b, dep e}
    ssa_u64* dent = nullptr;                // half-warp path: resolved dependency entries
    ssa_u64* rfe = nullptr;                 // half-warp path: fast-evaluator terms per reaction
    std::map<std::string, K2Kernel> kern;   // "block/dump" -> NVRTC-compiled K2
};

struct DevCache {
    std::map<std::string, K1Entry> k1;  // k1_key(block, minb, dump, sweep layout)
    K2Dev k2;
    double* prof = nullptr;             // [R] propensity-share sums of a profiling run (device)
};

struct ssa_model {
    int S = 0, R = 0;
    std::vector<long long> x0;
    std::vector<std::string> names;   // optional species labels (ssa_model_set_names)
    std::vector<RxI> rx;
    mutable std::mutex mu;
    mutable std::map<int, DevCache> dev;
    mutable double* pinned_const = nullptr;  // [constant pool][x0 S], page-locked, for per-run uploads
    // K1 dispatch profile (results are identical with or without it): the
    // reactions that dominate the event stream, measured by the first thread-path
    // run (propensity shares sampled at grid crossings) and applied by predicated
    // adds ahead of the update's jump table in later runs
    mutable std::vector<int> hot;
    mutable bool hot_known = false;
    // parameter sweeps: events per trajectory of each point, from an earlier run of
    // the same sweep (keyed by its points, sizes and horizon), used to hand out the
    // costliest points first
    mutable std::map<std::string, std::vector<double>> sweep_cost;
};

struct PoolLayout;
static PoolLayout make_pool(const ssa_model& m, int points, const double* rates, const double* modcs);

// K1 constant-memory image of the model's numbers (its constant pool, then
// the initial counts), staged once in page-locked host memory and copied to
// the device at the start of every run (the run's inputs).  *n_pool receives
// the pool size.
static ssa_status pinned_constants(const ssa_model& m, double** out, size_t* bytes, size_t* n_pool);

extern "C" ssa_status ssa_model_create(int32_t n_species, const int64_t* initial_counts, int32_t n_reactions,
                                       const ssa_reaction* reactions, ssa_model** out)
{
    return ssa_model_create_ex(n_species, initial_counts, n_reactions, reactions, nullptr, out);
}

extern "C" ssa_status ssa_model_create_ex(int32_t n_species, const int64_t* initial_counts, int32_t n_reactions,
                                          const ssa_reaction* reactions, const ssa_reaction_ext* ext, ssa_model** out)
{
    if (!out) return fail(SSA_ERR_INVALID_ARG, "out is null");
    *out = nullptr;
    if (n_species < 1 || n_species > 16383) return fail(SSA_ERR_MODEL, "n_species %d not in [1, 16383]", n_species);
    if (n_reactions < 0 || n_reactions > 65535)
        return fail(SSA_ERR_MODEL, "n_reactions %d not in [0, 65535]", n_reactions);
    if (!initial_counts) return fail(SSA_ERR_INVALID_ARG, "initial_counts is null");
    if (n_reactions > 0 && !reactions) return fail(SSA_ERR_INVALID_ARG, "reactions is null");
    std::unique_ptr<ssa_model> m(new ssa_model);
    m->S = n_species;
    m->R = n_reactions;
    for (int s = 0; s < n_species; ++s) {
        const int64_t v = initial_counts[s];
        if (v < 0 || v > 2147483647LL)
            return fail(SSA_ERR_MODEL, "initial count of species %d is %lld (must be in [0, 2^31-1])", s, (long long)v);
        m->x0.push_back(v);
    }
    for (int j = 0; j < n_reactions; ++j) {
        const ssa_reaction& r = reactions[j];
        RxI q;
        if (r.n_reactants < 0 || r.n_reactants > 3 || r.n_products < 0)
            return fail(SSA_ERR_MODEL, "reaction %d: bad term counts", j);
        if ((r.n_reactants && !r.reactants) || (r.n_products && !r.products))
            return fail(SSA_ERR_INVALID_ARG, "reaction %d: null term array", j);
        if (!std::isfinite(r.rate) || r.rate < 0.0) return fail(SSA_ERR_MODEL, "reaction %d: rate must be finite and >= 0", j);
        std::map<int, long long> net;
        int order = 0;
        for (int t = 0; t < r.n_reactants; ++t) {
            const ssa_term& tm = r.reactants[t];
            if (tm.species < 0 || tm.species >= n_species)
                return fail(SSA_ERR_MODEL, "reaction %d: unknown reactant species %d", j, tm.species);
            if (tm.coef < 1) return fail(SSA_ERR_MODEL, "reaction %d: reactant coefficient %d < 1", j, tm.coef);
            for (auto& pr : q.reac)
                if (pr.first == tm.species)
                    return fail(SSA_ERR_MODEL, "reaction %d: species %d listed twice among reactants", j, tm.species);
            order += tm.coef;
            q.reac.push_back({tm.species, tm.coef});
            net[tm.species] -= tm.coef;
        }
        if (order > 3) return fail(SSA_ERR_MODEL, "reaction %d: total reactant order %d > 3", j, order);
        for (int t = 0; t < r.n_products; ++t) {
            const ssa_term& tm = r.products[t];
            if (tm.species < 0 || tm.species >= n_species)
                return fail(SSA_ERR_MODEL, "reaction %d: unknown product species %d", j, tm.species);
            if (tm.coef < 1 || tm.coef > 1000000)
                return fail(SSA_ERR_MODEL, "reaction %d: product coefficient %d not in [1, 1e6]", j, tm.coef);
            net[tm.species] += tm.coef;
        }
        for (auto& kv : net)
            if (kv.second != 0) q.nu.push_back({kv.first, kv.second});
        q.rate = r.rate;
        q.mod_sp = r.modifier_species;
        q.mod_coef = r.modifier_coef;
        if (q.mod_sp != -1) {
            if (q.mod_sp < 0 || q.mod_sp >= n_species)
                return fail(SSA_ERR_MODEL, "reaction %d: unknown modifier species %d", j, q.mod_sp);
            if (!std::isfinite(q.mod_coef)) return fail(SSA_ERR_MODEL, "reaction %d: non-finite modifier coefficient", j);
        } else {
            q.mod_coef = 0.0;
        }
        if (ext) {
            const ssa_reaction_ext& x = ext[j];
            if (x.mass_action != 0 && x.mass_action != 1)
                return fail(SSA_ERR_MODEL, "reaction %d: mass_action must be 0 or 1", j);
            q.mass_action = x.mass_action == 1;
            if (x.n_gates < 0 || x.n_gates > 4) return fail(SSA_ERR_MODEL, "reaction %d: %d gates (0..4)", j, x.n_gates);
            if (x.n_gates > 0 && !x.gates) return fail(SSA_ERR_INVALID_ARG, "reaction %d: gates is null", j);
            for (int g = 0; g < x.n_gates; ++g) {
                const ssa_gate& gt = x.gates[g];
                if (gt.species < 0 || gt.species >= n_species)
                    return fail(SSA_ERR_MODEL, "reaction %d: unknown gate species %d", j, gt.species);
                if (gt.kind != SSA_GATE_POSITIVE && gt.kind != SSA_GATE_ZERO)
                    return fail(SSA_ERR_MODEL, "reaction %d: unknown gate kind %d", j, gt.kind);
                q.gates.push_back({gt.species, gt.kind});
            }
        }
        m->rx.push_back(q);
    }
    *out = m.release();
    return SSA_OK;
}

extern "C" void ssa_model_destroy(ssa_model* m)
{
    if (!m) return;
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess) {
        for (auto& kv : m->dev) {
            if (cudaSetDevice(kv.first) != cudaSuccess) continue;
            K2Dev& k = kv.second.k2;
            if (k.dev_image) cudaFree(k.dev_image);
            if (k.host_image) cudaFreeHost(k.host_image);
            for (auto& e : k.kern)
                if (e.second.lib) cudaLibraryUnload(e.second.lib);
            for (auto& e : kv.second.k1)
                if (e.second.lib) cudaLibraryUnload(e.second.lib);
            if (kv.second.prof) cudaFree(kv.second.prof);
        }
        cudaSetDevice(cur);
    }
    if (m->pinned_const) cudaFreeHost(m->pinned_const);
    delete m;
}

extern "C" ssa_status ssa_model_set_names(ssa_model* m, const char* const* names)
{
    if (!m) return fail(SSA_ERR_INVALID_ARG, "model is null");
    std::vector<std::string> v;
    if (names) {
        for (int s = 0; s < m->S; ++s) {
            if (!names[s]) return fail(SSA_ERR_INVALID_ARG, "name of species %d is null", s);
            v.emplace_back(names[s]);
        }
    }
    std::lock_guard<std::mutex> lk(m->mu);
    m->names.swap(v);
    return SSA_OK;
}

extern "C" const char* ssa_model_species_name(const ssa_model* m, int32_t index)
{
    if (!m || index < 0 || index >= m->S || m->names.empty()) return nullptr;
    return m->names[(size_t)index].c_str();
}

extern "C" int32_t ssa_model_n_species(const ssa_model* m) { return m ? m->S : 0; }
extern "C" int32_t ssa_model_n_reactions(const ssa_model* m) { return m ? m->R : 0; }

static long long grid_K(double t_end, double dt) { return (long long)std::floor(t_end / dt + 1e-9); }

extern "C" uint64_t ssa_grid_size(double t_end, double dt)
{
    if (!(t_end > 0.0) || !(dt > 0.0) || !std::isfinite(t_end) || !std::isfinite(dt)) return 0;
    const double kk = std::floor(t_end / dt + 1e-9);
    if (!(kk < 1e12)) return 0;
    return (uint64_t)kk + 1;
}

// ------------------------------------------------------------------ K1 JIT
static std::string factor_expr(int s, int m)
{
    std::ostringstream o;
    if (m == 1) o << "x[" << s << "]";
    else if (m == 2) o << "__dmul_rn(__dmul_rn(x[" << s << "], __dadd_rn(x[" << s << "], -1.0)), 0.5)";
    else o << "__ddiv_rn(__dmul_rn(__dmul_rn(x[" << s << "], __dadd_rn(x[" << s << "], -1.0)), __dadd_rn(x[" << s << "], -2.0)), 6.0)";
    return o.str();
}

// Layout of the K1 constants: the model's rate and modifier constants,
// deduplicated into slots.  For a parameter sweep each reaction's constant
// is a column over the sweep points and two reactions share a slot only if
// their columns are bitwise equal at every point; a plain run is the
// one-point case.  K1 reads slot i as SSA_K(i): c_k[i] from __constant__
// memory (one uniform load fetches two), or kp[i] from the per-point rows in
// shared memory in the sweep variant.  The clamp max(0, k + d*x) of P:93 is
// emitted only if d < 0 at some point (k >= 0 and d >= 0 give k + d*x >= 0 for
// counts x >= 0, so there it is a no-op).
struct PoolLayout {
    int n = 0;                       // slots
    std::vector<int> rate_slot, mod_slot;
    std::vector<char> clamp;
    std::vector<double> values;      // [points][n]
};

static PoolLayout make_pool(const ssa_model& m, int points, const double* rates, const double* modcs)
{
    PoolLayout L;
    const int R = m.R;
    auto rate = [&](int p, int j) { return rates ? rates[(size_t)p * R + j] : m.rx[j].rate; };
    auto modc = [&](int p, int j) { return modcs ? modcs[(size_t)p * R + j] : m.rx[j].mod_coef; };
    std::vector<std::vector<double>> cols;
    auto slot_of = [&](const std::vector<double>& col) {
        for (size_t i = 0; i < cols.size(); ++i)
            if (memcmp(cols[i].data(), col.data(), sizeof(double) * col.size()) == 0) return (int)i;
        cols.push_back(col);
        return (int)cols.size() - 1;
    };
    L.rate_slot.assign(R, -1);
    L.mod_slot.assign(R, -1);
    L.clamp.assign(R, 0);
    std::vector<double> col(points);
    for (int j = 0; j < R; ++j) {
        for (int p = 0; p < points; ++p) col[p] = rate(p, j);
        L.rate_slot[j] = slot_of(col);
        if (m.rx[j].mod_sp >= 0) {
            bool neg = false;
            for (int p = 0; p < points; ++p) {
                col[p] = modc(p, j);
                neg = neg || !(col[p] >= 0.0);
            }
            L.mod_slot[j] = slot_of(col);
            L.clamp[j] = neg;
        }
    }
    if (cols.empty()) cols.push_back(std::vector<double>(points, 0.0));
    L.n = (int)cols.size();
    L.values.resize((size_t)points * L.n);
    for (int p = 0; p < points; ++p)
        for (int i = 0; i < L.n; ++i) L.values[(size_t)p * L.n + i] = cols[i][p];
    return L;
}

static ssa_status pinned_constants(const ssa_model& m, double** out, size_t* bytes, size_t* n_pool)
{
    const PoolLayout L = make_pool(m, 1, nullptr, nullptr);
    *n_pool = (size_t)L.n;
    *bytes = sizeof(double) * ((size_t)L.n + (size_t)m.S);
    if (!m.pinned_const) {
        CU(cudaMallocHost(&m.pinned_const, *bytes));
        double* p = m.pinned_const;
        for (int i = 0; i < L.n; ++i) p[i] = L.values[i];
        for (int s = 0; s < m.S; ++s) p[L.n + s] = (double)m.x0[s];
    }
    *out = m.pinned_const;
    return SSA_OK;
}

// a3 for reaction j: k^ (rate, or the clamped linear modifier of P:93), then
// a = k^ * h.
// kh >= 0: the reaction's modified rate k^ is the cached register kh[kh] (K1)
static std::string prop_stmts(const RxI& q, int j, const PoolLayout& L, int kh = -1)
{
    std::ostringstream o;
    const std::string rate = "SSA_K(" + std::to_string(L.rate_slot[j]) + ")";
    if (kh >= 0) {
        o << "k = kh[" << kh << "]; ";
    } else if (q.mod_sp >= 0) {
        const std::string modc = "SSA_K(" + std::to_string(L.mod_slot[j]) + ")";
        o << "k = __dadd_rn(" << rate << ", __dmul_rn(" << modc << ", x[" << q.mod_sp << "])); ";
        if (L.clamp[j]) o << "k = (k < 0.0) ? 0.0 : k; ";
    } else {
        o << "k = " << rate << "; ";
    }
    if (q.reac.empty() || !q.mass_action) {
        o << "a = k;";
    } else {
        o << "h = " << factor_expr(q.reac[0].first, q.reac[0].second) << "; ";
        for (size_t t = 1; t < q.reac.size(); ++t)
            o << "h = __dmul_rn(h, " << factor_expr(q.reac[t].first, q.reac[t].second) << "); ";
        o << "a = __dmul_rn(k, h);";
    }
    if (!q.gates.empty()) {   // a closed gate makes the propensity exactly 0
        o << " a = (";
        for (size_t g = 0; g < q.gates.size(); ++g)
            o << (g ? " && " : "") << "x[" << q.gates[g].first << "]" << (q.gates[g].second == SSA_GATE_ZERO ? " == 0.0" : " > 0.0");
        o << ") ? a : 0.0;";
    }
    return o.str();
}

// K1 code-generation variants (tuning; the arithmetic is identical in all of
// them).  SSA_K1_GEN is read once per process:
//   upd=brx|switch   a8 as one brx.idx jump table (default) or a C++ switch
//   hot=a:b:...      override the measured hot set (K1Spec; run_range measures
//                    it on a model's first plain thread-path run): the listed
//                    reactions are applied by predicated adds and only the other
//                    lanes take the jump table
//   nospread32       small ensembles run the (128, minb) variant instead of a
//                    (32, 1) one
// (Measured and dropped: int64-pattern selection compares on the ALU pipe,
// species counts in shared memory with a table update, and a warp-vote
// pruning of the selection compares at static anchors were all slower.)
// Dispatch specialisation of one K1 variant (the arithmetic is the same in all).
struct K1Spec {
    std::vector<int> hot;   // reactions applied by predicated adds ahead of the jump table
    bool prof = false;      // sample the propensity shares at grid crossings
};

struct K1Gen {
    bool flat_switch = true;
    bool seed_imm = true;   // keys=imm|param: Philox round keys as instruction immediates (kernel per seed)
    int sel = 0;   // sel=f64|i64|mix: selection compares as fp64 (FP64 pipe), int64 patterns (ALU), or alternating
    std::vector<int> hot;   // hot=a:b:...: reactions updated by predicated adds ahead of the jump table
    bool spread32 = true;   // small-ensemble launches use a (32, 1) launch-bounds variant (nospread32: off)
    int plog = 0;           // plog=div: round 1's division-based log (speed A/B only, breaks parity);
                            // plog=global: the table read through L1 instead of shared memory
    bool no_cskip = true;   // cskip: reuse the cold prefix (measured 1.6% slower on HIV: the warp-uniform
                            // branch splits the event loop's basic block; off by default)
};

static K1Gen k1_gen()
{
    static const K1Gen g = [] {
        K1Gen r;
        const char* e = getenv("SSA_K1_GEN");
        const std::string s = e ? e : "";
        if (s.find("upd=switch") != std::string::npos) r.flat_switch = false;
        if (s.find("keys=param") != std::string::npos) r.seed_imm = false;
        if (s.find("sel=i64") != std::string::npos) r.sel = 1;
        if (s.find("sel=mix") != std::string::npos) r.sel = 2;
        if (s.find("sel=hi32") != std::string::npos) r.sel = 3;   // speed A/B only (no tie fallback)
        if (s.find("sel=hi32x") != std::string::npos) r.sel = 4;  // high words + exact tie fallback
        if (s.find("nospread32") != std::string::npos) r.spread32 = false;
        if (s.find("plog=div") != std::string::npos) r.plog = 1;
        if (s.find("plog=global") != std::string::npos) r.plog = 2;
        if (s.find("cskip") != std::string::npos && s.find("nocskip") == std::string::npos) r.no_cskip = false;
        const size_t h = s.find("hot=");
        if (h != std::string::npos) {
            size_t q = h + 4;
            while (q < s.size() && isdigit((unsigned char)s[q])) {
                size_t e = q;
                while (e < s.size() && isdigit((unsigned char)s[e])) ++e;
                r.hot.push_back(atoi(s.substr(q, e - q).c_str()));
                q = (e < s.size() && s[e] == ':') ? e + 1 : e;
            }
        }
        return r;
    }();
    return g;
}

// sweep: the parameter-sweep variant (constants per sweep point, read from
// shared memory through kp); L: the constant layout the code indexes.
// seed >= 0: the run's Philox key schedule is compiled in as immediates.
static std::string gen_k1_model(const ssa_model& m, int block, int minb, bool dump, bool sweep, const PoolLayout& L,
                                long long seed_bits, bool use_seed, int record = 0, const K1Spec* spec = nullptr)
{
    const int S = m.S, R = m.R;
    const K1Gen g = k1_gen();
    std::ostringstream o;
    if (record == 1) {
        // event recording: the pre-event counts of the species reaction j changes, in nu order
        size_t U = 1;
        for (int j = 0; j < R; ++j) U = std::max(U, m.rx[j].nu.size());
        o << "#define SSA_K1_RECORD 1\n#define SSA_REC_U " << U << "\n";
    } else if (record == 2) {
        // stride-sampled points: the full state (S counts) per point
        o << "#define SSA_K1_RECORD 2\n#define SSA_REC_U " << S << "\n";
    } else {
        o << "#define SSA_K1_RECORD 0\n";
    }
    o << "#define SSA_K1_PROF " << (spec && spec->prof ? 1 : 0) << "\n";
    o << "#define SSA_PLOG_DIV " << (g.plog == 1 ? 1 : 0) << "\n#define SSA_PLOG_GLOBAL " << (g.plog == 2 ? 1 : 0) << "\n";
    if (g.plog == 1) o << "__constant__ double c_plog_div[14] = SSA_PLOG_DIV_COEF_INIT;\n";
    // tail compaction (k1_thread.cuh): plain, dump and profiling variants
    o << "#define SSA_K1_MIG " << ((!sweep && record == 0) ? 1 : 0) << "\n";
    // time-sliced trajectories (k1_thread.cuh): plain, dump and profiling variants (not sweeps: their
    // costliest-first order hands out the long trajectories' phases ~1 round of lanes apart, so
    // phase p + 1 would often wait for phase p -- 13% slower on the Fig. 4 sweep with 32 phases)
    o << "#define SSA_K1_SEG " << ((!sweep && record == 0) ? 1 : 0) << "\n";
    std::vector<int> hot;   // the dispatch profile's hot reactions (K1Spec, or the knob)
    for (int hj : (!g.hot.empty() ? g.hot : (spec ? spec->hot : std::vector<int>())))
        if (hj >= 0 && hj < R) hot.push_back(hj);
    o << "#define SSA_S " << S << "\n#define SSA_R " << R << "\n#define SSA_K1_BLOCK " << block
      << "\n#define SSA_K1_MINB " << minb << "\n#define SSA_K1_SEL " << g.sel << "\n#define SSA_K1_DUMP "
      << (dump ? 1 : 0) << "\n#define SSA_K1_SWEEP " << (sweep ? 1 : 0) << "\n";
    if (use_seed) {
        const ssa_u32 k0 = (ssa_u32)(unsigned long long)seed_bits, k1 = (ssa_u32)((unsigned long long)seed_bits >> 32);
        // Philox4x32-10 (a2) with this seed's round keys as literals
        o << "#define SSA_KS_IMM 1\n"
          << "static __device__ __forceinline__ ssa_philox_out ssa_philox_seeded(ssa_u32 c0, ssa_u32 c1, ssa_u32 c2, "
             "ssa_u32 c3) {\n  ssa_u32 lo0, hi0, lo1, hi1;\n";
        for (int r = 0; r < 10; ++r) {
            const ssa_u32 rk0 = k0 + (ssa_u32)r * 0x9E3779B9u, rk1 = k1 + (ssa_u32)r * 0xBB67AE85u;
            o << "  lo0 = 0xD2511F53u * c0; hi0 = __umulhi(0xD2511F53u, c0); lo1 = 0xCD9E8D57u * c2; "
                 "hi1 = __umulhi(0xCD9E8D57u, c2);\n"
              << "  c0 = hi1 ^ c1 ^ " << rk0 << "u; c1 = lo1; c2 = hi0 ^ c3 ^ " << rk1 << "u; c3 = lo0;\n";
        }
        o << "  ssa_philox_out o; o.o0 = c0; o.o1 = c1; o.o2 = c2; o.o3 = c3; return o;\n}\n";
    } else {
        o << "#define SSA_KS_IMM 0\n";
    }
    if (sweep) {
        o << "#define SSA_K(i) kp[i]\n#define SSA_KP_PARAM , const double* __restrict__ kp\n#define SSA_KP_ARG , kp\n";
    } else {
        o << "__constant__ double c_k[" << L.n << "];\n";
        o << "#define SSA_K(i) c_k[i]\n#define SSA_KP_PARAM\n#define SSA_KP_ARG\n";
    }
    o << "__constant__ double c_x0[" << S << "];\n";
    o << "__constant__ double c_plog[8] = SSA_PLOG_COEF_INIT;\n";
    // a3's modified rates k^ = max(0, k + d x_m) (R4) depend on x_m alone: each
    // distinct (k, d, m) is kept in a register (kh) and recomputed only after
    // an event that changes a modifier species (and at the start of a
    // trajectory).  Same expression, same bits as evaluating it every event.
    std::vector<int> kh_of(R, -1);
    std::vector<int> kh_first;   // a reaction that defines each cached term
    for (int j = 0; j < R; ++j) {
        if (m.rx[j].mod_sp < 0) continue;
        for (size_t i = 0; i < kh_first.size() && kh_of[j] < 0; ++i) {
            const int f = kh_first[i];
            if (L.rate_slot[f] == L.rate_slot[j] && L.mod_slot[f] == L.mod_slot[j] &&
                m.rx[f].mod_sp == m.rx[j].mod_sp && L.clamp[f] == L.clamp[j])
                kh_of[j] = (int)i;
        }
        if (kh_of[j] < 0) {
            kh_of[j] = (int)kh_first.size();
            kh_first.push_back(j);
        }
    }
    if (kh_first.size() > 8) {   // register budget: evaluate inline instead
        kh_first.clear();
        std::fill(kh_of.begin(), kh_of.end(), -1);
    }
    const int NKH = (int)kh_first.size();
    o << "#define SSA_NKH " << NKH << "\n";
    o << "static __device__ __forceinline__ void ssa_khat(const double (&x)[SSA_S], double (&kh)[SSA_NKH > 0 ? SSA_NKH : 1] SSA_KP_PARAM) {\n";
    o << "  double k; (void)k; (void)x; (void)kh;\n";
    for (int i = 0; i < NKH; ++i) {
        const int j = kh_first[i];
        o << "  { k = __dadd_rn(SSA_K(" << L.rate_slot[j] << "), __dmul_rn(SSA_K(" << L.mod_slot[j] << "), x["
          << m.rx[j].mod_sp << "])); ";
        if (L.clamp[j]) o << "k = (k < 0.0) ? 0.0 : k; ";
        o << "kh[" << i << "] = k; }\n";
    }
    o << "}\n";
    {
        // reactions whose net change touches a modifier species of a cached term
        std::vector<int> dirty;
        for (int j = 0; j < R; ++j) {
            bool d = false;
            for (auto& nu : m.rx[j].nu)
                for (int f : kh_first) d = d || (nu.second != 0 && nu.first == m.rx[f].mod_sp);
            if (d) dirty.push_back(j);
        }
        o << "static __device__ __forceinline__ bool ssa_khat_dirty(int j) { (void)j; return ";
        if (dirty.empty()) {
            o << "false";
        } else if (dirty.size() <= 4) {
            for (size_t i = 0; i < dirty.size(); ++i) o << (i ? " || " : "") << "j == " << dirty[i];
        } else if (R <= 64) {
            unsigned long long mask = 0;
            for (int j : dirty) mask |= 1ull << j;
            o << "((0x" << std::hex << mask << std::dec << "ull >> j) & 1ull) != 0";
        } else {
            o << "true";
        }
        o << "; }\n";
    }
    o << "static __device__ __forceinline__ double ssa_prefix(const double (&x)[SSA_S], const double (&kh)[SSA_NKH > 0 ? SSA_NKH : 1], double (&c)[SSA_R > 0 ? SSA_R : 1] SSA_KP_PARAM) {\n";
    o << "  double a, h, k, acc = 0.0; (void)a; (void)h; (void)k; (void)x; (void)c; (void)kh;\n";
    for (int j = 0; j < R; ++j) {
        o << "  { " << prop_stmts(m.rx[j], j, L, kh_of[j]) << " "
          << (j == 0 ? "acc = a;" : "acc = __dadd_rn(acc, a);") << " c[" << j << "] = acc; }\n";
    }
    o << "  return acc;\n}\n";
    // Cold-prefix reuse (K1Spec::hot): the profile's hot reactions change a few
    // species (HIV's V4 -> 0 and V5 -> 0 change V4, V5); every propensity before
    // the first one that reads such a species -- indices [0, f) -- and hence the
    // prefix c_0..c_{f-1} is unchanged by a hot event.  K1 keeps c_0..c_{f-1} across
    // iterations and recomputes them only when some lane of the warp applied a
    // reaction that changes a species they read (a warp-uniform branch); the
    // values are the same expressions of the same counts, so the bits are those
    // of the full recompute.  ssa_prefix_lo computes c_0..c_{f-1}, ssa_prefix_hi
    // the rest from c_{f-1}; ssa_lo_clean(j) says reaction j leaves [0, f) alone.
    int cskip = 0;
    if (!hot.empty() && !(spec && spec->prof) && !sweep && !g.no_cskip) {
        std::vector<char> hot_sp(S, 0), lo_reads(S, 0);
        for (int hj : hot)
            for (auto& d : m.rx[hj].nu) hot_sp[d.first] = 1;
        auto reads = [&](int j, const std::vector<char>& set) {
            const RxI& q = m.rx[j];
            bool r = q.mod_sp >= 0 && set[q.mod_sp];
            if (q.mass_action) for (auto& t : q.reac) r = r || set[t.first];
            for (auto& gt : q.gates) r = r || set[gt.first];
            return r;
        };
        int f = R;
        for (int j = 0; j < R && f == R; ++j)
            if (reads(j, hot_sp)) f = j;
        std::vector<int> clean;
        if (f >= 2 && f < R) {
            for (int j = 0; j < f; ++j) {
                const RxI& q = m.rx[j];
                if (q.mod_sp >= 0) lo_reads[q.mod_sp] = 1;
                if (q.mass_action) for (auto& t : q.reac) lo_reads[t.first] = 1;
                for (auto& gt : q.gates) lo_reads[gt.first] = 1;
            }
            for (int j = 0; j < R; ++j) {
                bool touches = false;
                for (auto& d : m.rx[j].nu) touches = touches || lo_reads[d.first];
                if (!touches) clean.push_back(j);
            }
            if (R <= 64 || clean.size() <= 4) cskip = f;
        }
        if (cskip) {
            o << "static __device__ __forceinline__ void ssa_prefix_lo(const double (&x)[SSA_S], const double (&kh)[SSA_NKH > 0 ? SSA_NKH : 1], double (&c)[SSA_R > 0 ? SSA_R : 1] SSA_KP_PARAM) {\n";
            o << "  double a, h, k, acc = 0.0; (void)a; (void)h; (void)k; (void)x; (void)kh;\n";
            for (int j = 0; j < cskip; ++j)
                o << "  { " << prop_stmts(m.rx[j], j, L, kh_of[j]) << " "
                  << (j == 0 ? "acc = a;" : "acc = __dadd_rn(acc, a);") << " c[" << j << "] = acc; }\n";
            o << "}\n";
            o << "static __device__ __forceinline__ double ssa_prefix_hi(const double (&x)[SSA_S], const double (&kh)[SSA_NKH > 0 ? SSA_NKH : 1], double (&c)[SSA_R > 0 ? SSA_R : 1] SSA_KP_PARAM) {\n";
            o << "  double a, h, k, acc = c[" << cskip - 1 << "]; (void)a; (void)h; (void)k; (void)x; (void)kh;\n";
            for (int j = cskip; j < R; ++j)
                o << "  { " << prop_stmts(m.rx[j], j, L, kh_of[j]) << " acc = __dadd_rn(acc, a); c[" << j
                  << "] = acc; }\n";
            o << "  return acc;\n}\n";
            o << "static __device__ __forceinline__ bool ssa_lo_clean(int j) { return ";
            if (clean.empty()) {
                o << "false";
            } else if (R <= 64) {
                unsigned long long mask = 0;
                for (int j : clean) mask |= 1ull << j;
                o << "((0x" << std::hex << mask << std::dec << "ull >> j) & 1ull) != 0";
            } else {
                for (size_t i = 0; i < clean.size(); ++i) o << (i ? " || " : "") << "j == " << clean[i];
            }
            o << "; }\n";
        }
    }
    o << "#define SSA_CSKIP " << cskip << "\n";
    // error path only: out of line, state passed by value so the caller's
    // counts never need an addressable (stack) copy
    o << "struct ssa_state_v { double v[SSA_S]; };\n";
    o << "static __device__ __noinline__ int ssa_first_bad_v(const ssa_state_v xs SSA_KP_PARAM) {\n";
    o << "  const double* x = xs.v;\n";
    o << "  double a, h, k; (void)a; (void)h; (void)k; (void)x;\n";
    for (int j = 0; j < R; ++j)
        o << "  { " << prop_stmts(m.rx[j], j, L) << " if (!(fabs(a) < __longlong_as_double(0x7FF0000000000000ll))) return " << j << "; }\n";
    o << "  return -1;\n}\n";
    o << "static __device__ __forceinline__ int ssa_first_bad(const double (&x)[SSA_S] SSA_KP_PARAM) {\n";
    o << "  ssa_state_v xs;\n#pragma unroll\n  for (int s = 0; s < SSA_S; ++s) xs.v[s] = x[s];\n";
    o << "  return ssa_first_bad_v(xs SSA_KP_ARG);\n}\n";
    bool any_nu = false;
    for (int j = 0; j < R; ++j) any_nu = any_nu || !m.rx[j].nu.empty();
    bool exact_imm = true;   // every delta is an exact fp64 immediate (|d| < 2^53)
    for (int j = 0; j < R; ++j)
        for (auto& d : m.rx[j].nu) exact_imm = exact_imm && std::llabs(d.second) < (1ll << 53);
    const bool use_brx = g.flat_switch && any_nu && exact_imm && S <= 28 && R <= 4096;
    // a8 as ONE indirect branch through a jump table (PTX brx.idx): the C++
    // switch compiles to a decision tree of small tables, several dependent
    // branches deep.  Operands: %0..%(S-1) = x, %S = j; with rec (event
    // recording), %(S+1) = the row's pre-event count slots (null: row dropped),
    // written in the same case as the update (the C++ switch of the record
    // costs another decision tree per event).
    auto emit_brx = [&](bool rec) {
        const std::string pfx = rec ? "ssa_applyr_" : "ssa_apply_";
        o << "  asm volatile(\"{\\n\\t";
        if (rec) o << ".reg .pred pst;\\n\\t.reg .s32 rr;\\n\\tsetp.ne.u64 pst, %" << S + 1 << ", 0;\\n\\t";
        o << pfx << "tab: .branchtargets ";
        for (int jj = 0; jj < R; ++jj) o << (jj ? ", " : "") << pfx << jj;
        o << ";\\n\\tbrx.idx %" << S << ", " << pfx << "tab;\\n\\t";
        for (int jj = 0; jj < R; ++jj) {
            o << pfx << jj << ":\\n\\t";
            if (rec) {
                int q = 0;
                for (auto& d : m.rx[jj].nu) {
                    o << "cvt.rzi.s32.f64 rr, %" << d.first << ";\\n\\t@pst st.global.s32 [%" << S + 1 << "+" << 4 * q
                      << "], rr;\\n\\t";
                    ++q;
                }
            }
            for (auto& d : m.rx[jj].nu) {
                double v = (double)d.second;
                unsigned long long bits;
                memcpy(&bits, &v, 8);
                char hx[32];
                snprintf(hx, sizeof hx, "0d%016llX", bits);
                o << "add.rn.f64 %" << d.first << ", %" << d.first << ", " << hx << ";\\n\\t";
            }
            o << "bra " << pfx << "end;\\n\\t";
        }
        o << pfx << "end:\\n\\t}\"\n    : ";
        for (int s2 = 0; s2 < S; ++s2) o << (s2 ? ", " : "") << "\"+d\"(x[" << s2 << "])";
        o << "\n    : \"r\"(j)" << (rec ? ", \"l\"(out)" : "") << (rec ? "\n    : \"memory\"" : "") << ");\n";
    };
    // a7 + a8 with the selection counted on the high words (K1Gen::sel 4, k1_thread.cuh
    // ssa_count_hi): j0 <= j*, equal unless hi(c_j0) == hi(r).  The hot reactions check that tie
    // in their predicate; every jump-table case checks it for its own c_j (the case R-1 cannot
    // tie: j0 = R-1 means c_j < r for all j <= R-2).  A tie skips the update, recounts in fp64
    // and applies through ssa_apply.  Operands: %0..%(S-1) = x, %S = tie, %(S+1) = j0,
    // %(S+2) = hi(r), %(S+3+q) = hi(c_q) for q <= R-2.
    const bool selx = g.sel == 4 && use_brx && record == 0 && S + R + 2 <= 120;
    o << "#define SSA_K1_SELX " << (selx ? 1 : 0) << "\n";
    auto emit_brx_sel = [&]() {
        const std::string pfx = "ssa_applys_";
        o << "  asm volatile(\"{\\n\\t.reg .pred pt;\\n\\t" << pfx << "tab: .branchtargets ";
        for (int jj = 0; jj < R; ++jj) o << (jj ? ", " : "") << pfx << jj;
        o << ";\\n\\tbrx.idx %" << S + 1 << ", " << pfx << "tab;\\n\\t";
        for (int jj = 0; jj < R; ++jj) {
            o << pfx << jj << ":\\n\\t";
            if (jj <= R - 2)
                o << "setp.eq.s32 pt, %" << S + 3 + jj << ", %" << S + 2 << ";\\n\\t@pt bra " << pfx << "tie;\\n\\t";
            for (auto& d : m.rx[jj].nu) {
                double v = (double)d.second;
                unsigned long long bits;
                memcpy(&bits, &v, 8);
                char hx[32];
                snprintf(hx, sizeof hx, "0d%016llX", bits);
                o << "add.rn.f64 %" << d.first << ", %" << d.first << ", " << hx << ";\\n\\t";
            }
            o << "bra " << pfx << "end;\\n\\t";
        }
        o << pfx << "tie:\\n\\tmov.u32 %" << S << ", 1;\\n\\t" << pfx << "end:\\n\\t}\"\n    : ";
        for (int s2 = 0; s2 < S; ++s2) o << "\"+d\"(x[" << s2 << "]), ";
        o << "\"+r\"(tie)\n    : \"r\"(j), \"r\"(hr)";
        for (int q = 0; q + 1 < R; ++q) o << ", \"r\"(__double2hiint(c[" << q << "]))";
        o << ");\n";
    };
    o << "static __device__ __forceinline__ void ssa_apply(int j, double (&x)[SSA_S]) {\n";
    if (use_brx) {
        if (!hot.empty()) {
            // the most frequent reactions as predicated adds; the jump table only
            // for the lanes whose reaction is not among them
            o << "  bool hot = false;\n";
            for (int hj : hot) {
                o << "  if (j == " << hj << ") { hot = true;";
                for (auto& d : m.rx[hj].nu)   // exact integer literal (as the switch path)
                    o << " x[" << d.first << "] = __dadd_rn(x[" << d.first << "], " << d.second << ".0);";
                o << " }\n";
            }
            o << "  if (!hot) {\n";
            emit_brx(false);
            o << "  }\n";
        } else {
            emit_brx(false);
        }
        o << "}\n";
    } else {
        o << "  switch (j) {\n";
        for (int jj = 0; jj < R; ++jj) {
            if (m.rx[jj].nu.empty()) continue;
            o << "  case " << jj << ":";
            for (auto& d : m.rx[jj].nu) o << " x[" << d.first << "] = __dadd_rn(x[" << d.first << "], " << d.second << ".0);";
            o << " break;\n";
        }
        o << "  default: break;\n  }\n  (void)x;\n}\n";
    }
    if (selx) {
        o << "static __device__ __forceinline__ int ssa_apply_sel(int j, double (&x)[SSA_S], "
             "const double (&c)[SSA_R], double r) {\n  const int hr = __double2hiint(r);\n  int tie = 0;\n";
        o << "  bool hot = false;\n";
        for (int hj : hot) {
            // one predicate, no short circuit (keeps the adds predicated, as in ssa_apply)
            o << "  if ((j == " << hj << ")";
            if (hj <= R - 2) o << " & (__double2hiint(c[" << hj << "]) != hr)";
            o << ") { hot = true;";
            for (auto& d : m.rx[hj].nu)
                o << " x[" << d.first << "] = __dadd_rn(x[" << d.first << "], " << d.second << ".0);";
            o << " }\n";
        }
        o << "  if (!hot) {\n";
        emit_brx_sel();
        o << "  }\n";
        // the tie (hi(c_j0) == hi(r)): j* = #{ q <= R-2 : c_q <= r } in fp64, as ssa_count_from
        o << "  if (tie) {\n    int js = 0;\n#pragma unroll\n    for (int q = 0; q < SSA_R - 1; ++q) js += c[q] <= r ? 1 : 0;\n"
             "    j = js;\n    ssa_apply(j, x);\n  }\n  return j;\n}\n";
    }
    if (record == 1) {
        // pre-event counts of the species reaction j changes, in nu order, then x += nu_j
        o << "static __device__ __forceinline__ void ssa_apply_rec(int j, double (&x)[SSA_S], int* out) {\n";
        if (use_brx) {
            if (!hot.empty()) {
                // hot reactions: the record's stores and the adds predicated, the jump
                // table only for the other lanes (as ssa_apply)
                o << "  bool hot = false;\n";
                for (int hj : hot) {
                    o << "  if (j == " << hj << ") { hot = true;";
                    o << " if (out) {";
                    for (size_t q = 0; q < m.rx[hj].nu.size(); ++q)
                        o << " out[" << q << "] = (int)x[" << m.rx[hj].nu[q].first << "];";
                    o << " }";
                    for (auto& d : m.rx[hj].nu)
                        o << " x[" << d.first << "] = __dadd_rn(x[" << d.first << "], " << d.second << ".0);";
                    o << " }\n";
                }
                o << "  if (!hot) {\n";
                emit_brx(true);
                o << "  }\n";
            } else {
                emit_brx(true);
            }
        } else {
            o << "  if (out) switch (j) {\n";
            for (int jj = 0; jj < R; ++jj) {
                if (m.rx[jj].nu.empty()) continue;
                o << "  case " << jj << ":";
                for (size_t q = 0; q < m.rx[jj].nu.size(); ++q) o << " out[" << q << "] = (int)x[" << m.rx[jj].nu[q].first << "];";
                o << " break;\n";
            }
            o << "  default: break;\n  }\n  ssa_apply(j, x);\n";
        }
        o << "}\n";
    }
    return o.str();
}

static std::mutex g_jit_mu;
static std::map<std::string, std::vector<char>> g_cubin_cache;  // source -> cubin

static ssa_status nvrtc_compile(const std::string& src, std::vector<char>& cubin, std::string& log)
{
    {
        std::lock_guard<std::mutex> lk(g_jit_mu);
        auto it = g_cubin_cache.find(src);
        if (it != g_cubin_cache.end()) {
            cubin = it->second;
            return SSA_OK;
        }
    }
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, src.c_str(), "ssa_k1.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
        return fail(SSA_ERR_JIT, "nvrtcCreateProgram failed");
    const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "--fmad=false", "-lineinfo",
                          "--ptxas-options=-v", "-DSSA_NVRTC=1"};
    nvrtcResult rc = nvrtcCompileProgram(prog, (int)(sizeof opts / sizeof opts[0]), opts);
    size_t log_size = 0;
    nvrtcGetProgramLogSize(prog, &log_size);
    log.assign(log_size, '\0');
    if (log_size) nvrtcGetProgramLog(prog, &log[0]);
    if (rc != NVRTC_SUCCESS) {
        nvrtcDestroyProgram(&prog);
        return fail(SSA_ERR_JIT, "NVRTC compile failed: %s\n%s", nvrtcGetErrorString(rc), log.c_str());
    }
    size_t n = 0;
    nvrtcGetCUBINSize(prog, &n);
    cubin.resize(n);
    nvrtcGetCUBIN(prog, cubin.data());
    nvrtcDestroyProgram(&prog);
    std::lock_guard<std::mutex> lk(g_jit_mu);
    g_cubin_cache[src] = cubin;
    return SSA_OK;
}

// dump: the variant that also records the raw-trajectory dump and the firing
// hash (a11); runs without dumped ids use the variant without them.
// sweep: the parameter-sweep variant indexing the layout *sweep (else the
// model's own constant pool).
// seed: the run's seed when the key schedule is compiled in (K1Gen::seed_imm),
// else -1 (keys from the launch parameters).
// SSA_DEBUG_CHECKS=1: the NVRTC kernels count out-of-range indices (ssa_device.cuh SSA_CHECK)
static const char* debug_checks_prefix()
{
    static const bool on = getenv("SSA_DEBUG_CHECKS") && atoi(getenv("SSA_DEBUG_CHECKS")) != 0;
    return on ? "#define SSA_DEBUG_CHECKS 1\n" : "";
}

static std::string k1_full_source(const ssa_model& m, int block, int minb, bool dump, const PoolLayout* sweep,
                                  long long seed = -1, int record = 0, const K1Spec* spec = nullptr)
{
    const PoolLayout L = sweep ? *sweep : make_pool(m, 1, nullptr, nullptr);
    return std::string(debug_checks_prefix()) + kSsaDeviceSrc + "\n" +
           gen_k1_model(m, block, minb, dump, sweep != nullptr, L, seed, seed != -1, record, spec) + "\n" +
           kK1ThreadSrc;
}

static std::string k1_key(int block, int minb, bool dump, const PoolLayout* sweep, long long seed, int record,
                          const K1Spec* spec = nullptr)
{
    std::ostringstream o;
    o << block << "/" << minb << "/" << (dump ? 1 : 0) << "/" << seed << "/" << record;
    if (spec) {
        o << "/prof:" << (spec->prof ? 1 : 0) << "/hot";
        for (int h : spec->hot) o << ":" << h;
    }
    if (sweep) {
        o << "/sweep:" << sweep->n;
        for (size_t j = 0; j < sweep->rate_slot.size(); ++j)
            o << "," << sweep->rate_slot[j] << ":" << sweep->mod_slot[j] << ":" << (int)sweep->clamp[j];
    }
    return o.str();
}

static int default_minb(const ssa_model& m, int block)
{
    // target <= 128 registers per thread (512 threads/SM) for small networks;
    // let larger networks spill less by asking for fewer resident blocks
    // (measured on synthetic networks, profiles/r1k_k1_blocks_per_sm.txt:
    // 4 x 128 threads best up to R = 48, 3 x 128 for R = 56..80, 2 x 128 beyond)
    const int threads = m.R <= 48 ? 512 : (m.R <= 80 ? 384 : 256);
    return std::max(1, threads / block);
}

// requires: current device == dev, m.mu held
static ssa_status ensure_k1(const ssa_model& m, int dev, int block, int minb, bool dump, const PoolLayout* sweep,
                            K1Entry** out, double* jit_ms, long long seed = -1, int record = 0,
                            const K1Spec* spec = nullptr)
{
    DevCache& dc = m.dev[dev];
    const std::string key = k1_key(block, minb, dump, sweep, seed, record, spec);
    auto it = dc.k1.find(key);
    if (it != dc.k1.end()) {
        *out = &it->second;
        return SSA_OK;
    }
    auto t0 = std::chrono::steady_clock::now();
    K1Entry e;
    e.block = block;
    e.minb = minb;
    std::vector<char> cubin;
    TRY(nvrtc_compile(k1_full_source(m, block, minb, dump, sweep, seed, record, spec), cubin, e.log));
    CU(cudaLibraryLoadData(&e.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    CU(cudaLibraryGetKernel(&e.fn, e.lib, "ssa_k1"));
    // constant pool (plain runs) and x0 into the module's constant memory
    {
        double* pc = nullptr;
        size_t bytes = 0, n_pool = 0, got = 0;
        TRY(pinned_constants(m, &pc, &bytes, &n_pool));
        if (!sweep) {
            CU(cudaLibraryGetGlobal(&e.c_k, &got, e.lib, "c_k"));
            CU(cudaMemcpy(e.c_k, pc, sizeof(double) * n_pool, cudaMemcpyHostToDevice));
        }
        CU(cudaLibraryGetGlobal(&e.c_x0, &got, e.lib, "c_x0"));
        CU(cudaMemcpy(e.c_x0, pc + n_pool, sizeof(double) * m.S, cudaMemcpyHostToDevice));
    }
    int nb = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)e.fn, block, 0));
    e.blocks_per_sm = std::max(nb, 1);
    auto t1 = std::chrono::steady_clock::now();
    if (jit_ms) *jit_ms += std::chrono::duration<double, std::milli>(t1 - t0).count();
    auto res = dc.k1.emplace(key, e);
    *out = &res.first->second;
    return SSA_OK;
}

// SSA_PATH_AUTO: the thread path for R <= 64 (registers hold the prefix),
// two trajectories per warp for R <= 256 (P = ceil(R/16) <= 16), else one
// trajectory per warp.
// Thresholds from the path A/B benchmark (scripts/path_ab.py): on synthetic networks
// the thread path leads up to R = 128 (even with its prefix spilled past R ~ 64) and the half-warp
// K2 from R = 192; the crossover lies near R = 160.
static int auto_path(const ssa_model& m)
{
    return m.R <= 160 ? SSA_PATH_THREAD : (m.R <= 256 ? SSA_PATH_HALFWARP : SSA_PATH_WARP);
}

// requires: current device == dev, m.mu held.  The K2 tables live in one
// device block whose image is kept in page-locked host memory; every run
// re-uploads it (the run's model inputs) with one async copy.  The kernel
// itself is NVRTC-compiled per (block, dump) with S, R and P baked in.
// dynamic shared memory of K2: rx[R] (32 B) | x0[S] | per warp (x[S] | a[32P]) |
// nu_off | nu_ent | dep_off | dep_ent | (16-byte aligned) decoded descriptors [R] (40 B)
static bool has_m3(const ssa_model& m)
{
    for (auto& q : m.rx)
        for (auto& t : q.reac)
            if (t.second == 3) return true;
    return false;
}

// Half-warp fast evaluator (k2_half.cuh, SSA_K2_FE): every propensity has the form
// k * ((x_a * (x_b - d)) * s) -- no modifier, no gates, and a reactant multiset that is
// empty, {i}, {i, j} with coefficients 1, or {2i} (x_S = 1.0 stands in for a missing
// factor).  Each form performs exactly the operations of the general evaluator.
static bool k2_fe_ok(const ssa_model& m)
{
    for (auto& q : m.rx) {
        if (q.mod_sp >= 0 || !q.gates.empty()) return false;
        if (!q.mass_action) continue;
        if (q.reac.size() > 2) return false;
        if (q.reac.size() == 2 && (q.reac[0].second != 1 || q.reac[1].second != 1)) return false;
        if (q.reac.size() == 1 && q.reac[0].second > 2) return false;
    }
    return true;
}

// (species a, species b, flag d = 1 / s = 1/2) of reaction j's fast-evaluator form
static void k2_fe_terms(const ssa_model& m, int j, ssa_u64* sa, ssa_u64* sb, ssa_u64* f)
{
    const RxI& q = m.rx[j];
    const ssa_u64 one = (ssa_u64)m.S;
    *sa = one; *sb = one; *f = 0;
    if (!q.mass_action || q.reac.empty()) return;
    if (q.reac.size() == 2) { *sa = (ssa_u64)q.reac[0].first; *sb = (ssa_u64)q.reac[1].first; return; }
    *sa = (ssa_u64)q.reac[0].first;
    if (q.reac[0].second == 2) { *sb = *sa; *f = 1; }
}

// rx: whether the packed table is staged (models with coefficient-3 reactants)
static size_t k2_rxd_offset(int S, int R, int P, int n_ent, int n_dep, int block, bool half = false, bool rx = true)
{
    const size_t warps = (size_t)(block / 32);
    const size_t per_warp = half ? 2 * ((size_t)S + 16 * (size_t)P) : ((size_t)S + 32 * (size_t)P);
    const size_t b = (rx ? 32 * (size_t)R : 0) + 8 * (size_t)S + warps * 8 * per_warp +
                     4 * ((size_t)R + 1 + (size_t)n_ent + (size_t)R + 1 + (size_t)n_dep);
    return (b + 15) & ~(size_t)15;
}

static size_t k2_smem_bytes(int S, int R, int P, int n_ent, int n_dep, int block, bool half = false, bool rx = true)
{
    return k2_rxd_offset(S, R, P, n_ent, n_dep, block, half, rx) + 40 * (size_t)R;
}

// half-warp layout (k2_half.cuh): rx[R] (coefficient-3 models) | x0[S] | (16-aligned) per warp, per
// half (a[16 x 18] | x[S + 1 rounded up to even] | (E, u2)[16]) | rec[R] (16 B) | nu_ent | dent[n_dep] (8 B) |
// (16-aligned) rxd[R] (40 B) -- or, with the fast evaluator, rate[R] (8 B)
struct K2HalfLayout {
    size_t rec = 0, dent = 0, rxd = 0, bytes = 0;
};
static K2HalfLayout k2_half_layout(int S, int R, int P, int n_ent, int n_dep, int block, bool rx, bool fe)
{
    (void)P;
    K2HalfLayout L;
    const size_t warps = (size_t)(block / 32);
    const size_t awin = 16 * 18 + (((size_t)S + 2) & ~(size_t)1) + 32;
    size_t b = (rx ? 32 * (size_t)R : 0) + 8 * (size_t)S;
    b = (b + 15) & ~(size_t)15;
    b += warps * 2 * 8 * awin;
    b = (b + 15) & ~(size_t)15;
    L.rec = b;
    b += 16 * (size_t)R + 4 * (size_t)std::max(n_ent, 1);
    b = (b + 7) & ~(size_t)7;
    L.dent = b;
    b += 8 * (size_t)std::max(n_dep, 1);
    b = (b + 15) & ~(size_t)15;
    L.rxd = b;
    L.bytes = b + (rx ? 0 : (fe ? 8 * (size_t)R : 40 * (size_t)R));
    return L;
}

static std::string gen_k2_model(const ssa_model& m, int P, int block, int minb, bool dump, bool half)
{
    // longest net-change list and longest per-reaction dependency list (as
    // built by ensure_k2), and whether any reactant has coefficient 3
    int nu_max = 0, dep_max = 0, m3 = 0, gates = 0, mods = 0;
    std::vector<std::vector<int>> readers(m.S);
    for (int j = 0; j < m.R; ++j) {
        nu_max = std::max(nu_max, (int)m.rx[j].nu.size());
        gates |= !m.rx[j].gates.empty();
        mods |= (m.rx[j].mod_sp >= 0);
        for (auto& t : m.rx[j].reac) {
            readers[t.first].push_back(j);
            m3 |= (t.second == 3);
        }
        if (m.rx[j].mod_sp >= 0) readers[m.rx[j].mod_sp].push_back(j);
        for (auto& g : m.rx[j].gates) readers[g.first].push_back(j);
    }
    for (int j = 0; j < m.R; ++j) {
        std::vector<int> d;
        for (auto& c : m.rx[j].nu) d.insert(d.end(), readers[c.first].begin(), readers[c.first].end());
        std::sort(d.begin(), d.end());
        d.erase(std::unique(d.begin(), d.end()), d.end());
        dep_max = std::max(dep_max, (int)d.size());
    }
    std::ostringstream o;
    o << "#define SSA_S " << m.S << "\n#define SSA_R " << m.R << "\n#define SSA_P " << P << "\n#define SSA_K2_BLOCK "
      << block << "\n#define SSA_K2_MINB " << minb << "\n#define SSA_K2_DUMP " << (dump ? 1 : 0)
      << "\n#define SSA_K2_HALF " << (half ? 1 : 0)
      << "\n#define SSA_K2_FE " << ((half && k2_fe_ok(m)) ? 1 : 0)
      << "\n#define SSA_HAS_M3 " << m3 << "\n#define SSA_HAS_GATES " << gates << "\n#define SSA_HAS_MODS " << mods << "\n#define SSA_NU_MAX " << nu_max << "\n#define SSA_DEP_MAX " << dep_max
      << "\n";
    o << "__constant__ double c_plog[8] = SSA_PLOG_COEF_INIT;\n";
    return o.str();
}

// half: two trajectories per warp (k2_half.cuh, order warp16), P = ceil(R/16)
static std::string k2_full_source(const ssa_model& m, int P, int block, int minb, bool dump, bool half = false)
{
    return std::string(debug_checks_prefix()) + kSsaDeviceSrc + "\n" + gen_k2_model(m, P, block, minb, dump, half) + "\n" + kK2WarpSrc +
           "\n" + kK2HalfSrc;
}

// minb: the __launch_bounds__ residency target (1 = let the compiler use the
// registers it wants)
static ssa_status ensure_k2(const ssa_model& m, int dev, int block, int minb, bool dump, K2Dev** out,
                            K2Kernel** kout, double* jit_ms, bool half = false)
{
    K2Dev& k = m.dev[dev].k2;
    const int R = m.R, S = m.S;
    if (!k.ready) {
        const int P = std::max(1, (R + 31) / 32);
        if (P > 16) return fail(SSA_ERR_UNSUPPORTED, "warp path supports at most 512 reactions (got %d)", R);
        if (S > 16383) return fail(SSA_ERR_UNSUPPORTED, "warp path supports at most 16383 species (got %d)", S);
        const size_t R1 = (size_t)std::max(R, 1);
        std::vector<ssa_u64> pk(R1, 0), gw(R1, 0);
        std::vector<double> rate(R1, 0.0), modc(R1, 0.0), x0(S);
        std::vector<int> nu_off(R + 1, 0), nu_ent;
        for (int j = 0; j < R; ++j) {
            const RxI& q = m.rx[j];
            // gate word: count (3 bits) | per gate 14-bit species, 1-bit kind
            ssa_u64 g = (ssa_u64)q.gates.size();
            for (size_t t = 0; t < q.gates.size(); ++t)
                g |= ((ssa_u64)(q.gates[t].first & 0x3FFF) | ((ssa_u64)q.gates[t].second << 14)) << (3 + 15 * t);
            gw[j] = g;
            // packed reactant word of the PROPENSITY (no terms when h = 1)
            const size_t nr = q.mass_action ? q.reac.size() : 0;
            ssa_u64 w = (ssa_u64)nr;
            for (size_t t = 0; t < nr; ++t) {
                w |= (ssa_u64)(q.reac[t].first & 0x3FFF) << (2 + 16 * t);
                w |= (ssa_u64)(q.reac[t].second & 3) << (16 + 16 * t);
            }
            w |= (ssa_u64)(q.mod_sp >= 0 ? q.mod_sp : 0x3FFF) << 50;
            pk[j] = w;
            rate[j] = q.rate;
            modc[j] = q.mod_coef;
            for (auto& d : q.nu) {
                if (d.second < -32768 || d.second > 32767)
                    return fail(SSA_ERR_UNSUPPORTED, "warp path: reaction %d changes species %d by %lld (|delta| > 32767)",
                                j, d.first, d.second);
                nu_ent.push_back((int)(d.first & 0xFFFF) | (int)((unsigned)(int)d.second << 16));
            }
            nu_off[j + 1] = (int)nu_ent.size();
        }
        for (int s2 = 0; s2 < S; ++s2) x0[s2] = (double)m.x0[s2];
        const int n_ent_real = (int)nu_ent.size();
        if (nu_ent.empty()) nu_ent.push_back(0);
        // dependency graph: reaction j -> the reactions whose propensity reads a
        // species j changes (as a reactant, the modifier species or a gate
        // species), unique, ascending
        std::vector<std::vector<int>> readers(S);
        for (int j = 0; j < R; ++j) {
            const RxI& q = m.rx[j];
            for (auto& t : q.reac) readers[t.first].push_back(j);
            if (q.mod_sp >= 0) readers[q.mod_sp].push_back(j);
            for (auto& g : q.gates) readers[g.first].push_back(j);
        }
        std::vector<int> dep_off(R + 1, 0), dep_ent;
        for (int j = 0; j < R; ++j) {
            std::vector<int> d;
            for (auto& c : m.rx[j].nu) d.insert(d.end(), readers[c.first].begin(), readers[c.first].end());
            std::sort(d.begin(), d.end());
            d.erase(std::unique(d.begin(), d.end()), d.end());
            dep_ent.insert(dep_ent.end(), d.begin(), d.end());
            dep_off[j + 1] = (int)dep_ent.size();
        }
        const int n_dep_real = (int)dep_ent.size();
        if (dep_ent.empty()) dep_ent.push_back(0);
        // half-warp path: per-reaction records and dependency entries resolved for its
        // propensity layout a[l*18 + q] (reaction l*PH + q, PH = ceil(R/16))
        const int PH = std::max(1, (R + 15) / 16);
        std::vector<int4> rec(R1);
        for (int j = 0; j < R; ++j) rec[j] = make_int4(nu_off[j], nu_off[j + 1], dep_off[j], dep_off[j + 1]);
        const bool fe = k2_fe_ok(m);
        std::vector<ssa_u64> dent(dep_ent.size(), 0), rfe(R1, 0);
        for (int j = 0; j < R; ++j) {
            for (int q = dep_off[j]; q < dep_off[j + 1]; ++q) {
                const int jj = dep_ent[q];
                const ssa_u64 row = (ssa_u64)(jj / PH);
                const ssa_u64 slot = row * 18 + (ssa_u64)(jj % PH);   // a[l*18 + q], reaction l*PH + q
                ssa_u64 w;
                if (fe) {
                    // sa | sb << 16 | slot << 32 | d << 41 | reaction << 48
                    ssa_u64 sa, sb, f;
                    k2_fe_terms(m, jj, &sa, &sb, &f);
                    w = sa | (sb << 16) | (f << 41);
                } else {
                    // sa | sb << 14 | ma << 28 | mb << 30 | slot << 32 | reaction << 48
                    const ssa_u64 pw = pk[jj];
                    const int n = (int)(pw & 3ull);
                    const ssa_u64 sa = n >= 1 ? (pw >> 2) & 0x3FFF : 0, sb = n >= 2 ? (pw >> 18) & 0x3FFF : 0;
                    const ssa_u64 ma = n >= 1 ? (pw >> 16) & 3 : 0, mb = n >= 2 ? (pw >> 32) & 3 : 0;
                    w = sa | (sb << 14) | (ma << 28) | (mb << 30);
                }
                dent[q] = w | (slot << 32) | ((ssa_u64)jj << 48);
            }
        }
        if (fe)
            for (int j = 0; j < R; ++j) {
                ssa_u64 sa, sb, f;
                k2_fe_terms(m, j, &sa, &sb, &f);
                rfe[j] = sa | (sb << 16) | (f << 41);
            }
        // image layout (8-byte aligned sections): pk | gw | rate | modc | x0 | nu_off | nu_ent | dep_off | dep_ent
        const size_t o_pk = 0, o_gw = o_pk + 8 * R1, o_rate = o_gw + 8 * R1, o_modc = o_rate + 8 * R1,
                     o_x0 = o_modc + 8 * R1;
        const size_t o_off = o_x0 + 8 * (size_t)std::max(S, 1);
        const size_t o_ent = o_off + ((4 * nu_off.size() + 7) & ~(size_t)7);
        const size_t o_doff = o_ent + ((4 * nu_ent.size() + 7) & ~(size_t)7);
        const size_t o_dent = o_doff + ((4 * dep_off.size() + 7) & ~(size_t)7);
        const size_t o_rec = (o_dent + 4 * dep_ent.size() + 15) & ~(size_t)15;
        const size_t o_hd = o_rec + 16 * R1;
        const size_t o_rfe = o_hd + 8 * dent.size();
        const size_t bytes = o_rfe + 8 * R1;
        CU(cudaMallocHost(&k.host_image, bytes));
        char* h = (char*)k.host_image;
        memcpy(h + o_pk, pk.data(), 8 * R1);
        memcpy(h + o_gw, gw.data(), 8 * R1);
        memcpy(h + o_rate, rate.data(), 8 * R1);
        memcpy(h + o_modc, modc.data(), 8 * R1);
        memcpy(h + o_x0, x0.data(), 8 * (size_t)S);
        memcpy(h + o_off, nu_off.data(), 4 * nu_off.size());
        memcpy(h + o_ent, nu_ent.data(), 4 * nu_ent.size());
        memcpy(h + o_doff, dep_off.data(), 4 * dep_off.size());
        memcpy(h + o_dent, dep_ent.data(), 4 * dep_ent.size());
        memcpy(h + o_rec, rec.data(), 16 * R1);
        memcpy(h + o_hd, dent.data(), 8 * dent.size());
        memcpy(h + o_rfe, rfe.data(), 8 * R1);
        CU(cudaMalloc(&k.dev_image, bytes));
        CU(cudaMemcpy(k.dev_image, k.host_image, bytes, cudaMemcpyHostToDevice));
        char* d = (char*)k.dev_image;
        k.pk = (ssa_u64*)(d + o_pk);
        k.gw = (ssa_u64*)(d + o_gw);
        k.rate = (double*)(d + o_rate);
        k.modc = (double*)(d + o_modc);
        k.x0 = (double*)(d + o_x0);
        k.nu_off = (int*)(d + o_off);
        k.nu_ent = (int*)(d + o_ent);
        k.dep_off = (int*)(d + o_doff);
        k.dep_ent = (int*)(d + o_dent);
        k.rec = (int4*)(d + o_rec);
        k.dent = (ssa_u64*)(d + o_hd);
        k.rfe = (ssa_u64*)(d + o_rfe);
        k.image_bytes = bytes;
        k.P = P;
        k.n_ent = n_ent_real;
        k.n_dep = n_dep_real;
        k.ready = true;
    }
    *out = &k;
    const std::string key = std::to_string(block) + "/" + std::to_string(minb) + "/" + (dump ? "1" : "0") + "/" +
                            (half ? "h" : "w");
    const int PL = half ? std::max(1, (R + 15) / 16) : k.P;
    auto it = k.kern.find(key);
    if (it == k.kern.end()) {
        auto t0 = std::chrono::steady_clock::now();
        K2Kernel kk;
        std::vector<char> cubin;
        std::string log;
        if (half && PL > 16) return fail(SSA_ERR_UNSUPPORTED, "half-warp path supports at most 256 reactions (got %d)", R);
        TRY(nvrtc_compile(k2_full_source(m, PL, block, minb, dump, half), cubin, log));
        CU(cudaLibraryLoadData(&kk.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
        CU(cudaLibraryGetKernel(&kk.fn, kk.lib, "ssa_k2"));
        const bool m3 = has_m3(m);
        if (half) {
            const K2HalfLayout hl = k2_half_layout(S, R, PL, k.n_ent, k.n_dep, block, m3, k2_fe_ok(m));
            kk.smem = hl.bytes;
            kk.rxd_offset = hl.rxd;
            kk.rec_offset = hl.rec;
            kk.dent_offset = hl.dent;
        } else {
            kk.smem = k2_smem_bytes(S, R, PL, k.n_ent, k.n_dep, block, half, m3);
            kk.rxd_offset = k2_rxd_offset(S, R, PL, k.n_ent, k.n_dep, block, half, m3);
        }
        if (kk.smem > 227 * 1024)
            return fail(SSA_ERR_UNSUPPORTED, "warp path: model needs %zu B of shared memory", kk.smem);
        CU(cudaFuncSetAttribute((const void*)kk.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kk.smem));
        int nb = 0;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)kk.fn, block, kk.smem));
        if (nb <= 0) return fail(SSA_ERR_CUDA, "warp path: kernel cannot be resident (block %d, smem %zu)", block, kk.smem);
        kk.blocks_per_sm = nb;
        auto t1 = std::chrono::steady_clock::now();
        if (jit_ms) *jit_ms += std::chrono::duration<double, std::milli>(t1 - t0).count();
        it = k.kern.emplace(key, kk).first;
    }
    *kout = &it->second;
    return SSA_OK;
}

// ------------------------------------------------------------------ run core
static ssa_u64 next_pow2(ssa_u64 v)
{
    ssa_u64 p = 1;
    while (p < v) p <<= 1;
    return p;
}

template <int N>
struct Events {   // CUDA events, destroyed on every exit path (including a failed create)
    cudaEvent_t e[N] = {};
    ~Events() { for (cudaEvent_t x : e) if (x) cudaEventDestroy(x); }
    cudaError_t create()
    {
        for (cudaEvent_t& x : e) {
            const cudaError_t r = cudaEventCreate(&x);
            if (r != cudaSuccess) return r;
        }
        return cudaSuccess;
    }
};

struct DevBuf {  // stream-ordered device allocation
    void* p = nullptr;
    cudaStream_t st = nullptr;
    ~DevBuf()
    {
        if (p) cudaFreeAsync(p, st);
    }
    cudaError_t alloc(size_t bytes, cudaStream_t s)
    {
        st = s;
        return cudaMallocAsync(&p, bytes ? bytes : 8, s);
    }
    template <class T> T* as() const { return (T*)p; }
    void reset()
    {
        if (p) cudaFreeAsync(p, st);
        p = nullptr;
    }
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

struct Ctx {
    int device = 0;
    int prev_device = -1;
    cudaStream_t st = nullptr;
    bool own_stream = false;
    ~Ctx()
    {
        if (own_stream && st) {
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
        if (prev_device >= 0) cudaSetDevice(prev_device);
    }
};

static ssa_status setup_ctx(const ssa_run_options* o, Ctx& c)
{
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return fail(SSA_ERR_CUDA, "no CUDA device available (%s)", cudaGetErrorString(e));
    CU(cudaGetDevice(&c.prev_device));
    c.device = (o && o->device >= 0) ? o->device : c.prev_device;
    if (c.device >= n) return fail(SSA_ERR_INVALID_ARG, "device %d out of range (%d devices)", c.device, n);
    CU(cudaSetDevice(c.device));
    static std::once_flag pool_once[64];
    if (c.device < 64) {
        std::call_once(pool_once[c.device], [&] {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, c.device) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
        });
    }
    if (o && o->stream) {
        c.st = (cudaStream_t)o->stream;
    } else {
        CU(cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking));
        c.own_stream = true;
    }
    return SSA_OK;
}

struct RangeOut {
    double *n, *mean, *m2;  // device root [cells] each
};

struct RunInfo {
    ssa_dev_stats stats;
    int path = 0;
    double device_ms = 0, ssa_ms = 0, jit_ms = 0, reduce_ms = 0, dump_ms = 0;
    uint64_t h2d = 0, d2h = 0, reduce_bytes = 0, dump_bytes = 0;
    int launches = 0;
    uint64_t lanes = 0;   // SSA lanes launched (K1 threads that take trajectories)
};

// Reduce `count` elements per row from `in` down to one, writing the final
// root into `fin`.  Intermediate passes ping-pong through scratch buffers.
static ssa_status reduce_partials(ssa_tree_in in, ssa_u64 count, ssa_u64 rows, const ssa_tree_out& fin, cudaStream_t st,
                                  int* launches)
{
    DevBuf bufs[2];
    int which = 0;
    while (count > SSA_TREE_SPAN) {
        const ssa_u64 nout = (count + SSA_TREE_SPAN - 1) / SSA_TREE_SPAN;
        DevBuf& b = bufs[which];
        if (b.p) cudaFreeAsync(b.p, st), b.p = nullptr;
        CU(b.alloc(sizeof(double) * 3 * rows * nout, st));
        ssa_tree_out o{b.as<double>(), b.as<double>() + rows * nout, b.as<double>() + 2 * rows * nout, nout, 1, 0};
        CU(ssa_tree_merge_launch(in, count, rows, o, st));
        *launches += 1;
        in = ssa_tree_in{o.n, o.mean, o.m2, nout, 1};
        count = nout;
        which ^= 1;
    }
    CU(ssa_tree_merge_launch(in, count, rows, fin, st));
    *launches += 1;
    return SSA_OK;
}

// Parameter sweep ("a set of parameter-swept simulations"):
// P points of N trajectories each, point p's constants in row p of L.values.
// The run covers virtual ids p * N + i; a chunk holds whole points.
struct SweepSpec {
    int P = 0;
    ssa_u64 N = 0;
    PoolLayout L;
    std::vector<RangeOut> roots;   // per point
    std::vector<double> cost;      // per point: events per trajectory of an earlier run (empty: unknown)
    mutable std::vector<ssa_u64> events;   // out: applied events per point in this run
};

// Event recording (union-time selective memory): every applied event is
// appended (in no particular order) at a row reserved from *count; rows
// >= cap are counted but not written.
struct RecordSpec {
    int mode;              // 1: events (time, reaction, pre-event counts); 2: stride points (key, time, state)
    ssa_u64 stride;        // mode 2
    ssa_u64* key;          // mode 2: device [cap] (trajectory << 41 | 2k or 2E+1)
    ssa_u64* count;        // device counter (zeroed by the caller)
    ssa_u64 cap;
    double* t;             // device [cap]
    int* j;                // device [cap]
    int* pre;              // device [cap][U]
};

static ssa_status run_range(const ssa_model* m, ssa_u64 id_begin, ssa_u64 id_end, double t_end, double dt,
                            uint64_t seed, const ssa_run_options* o, Ctx& c, RangeOut root, RunInfo& info,
                            const ssa_dump* dump, bool dump_on_device, const SweepSpec* sw = nullptr,
                            const RecordSpec* rec = nullptr)
{
    const long long K = grid_K(t_end, dt);
    const ssa_u64 G = (ssa_u64)K + 1, S = (ssa_u64)m->S, cells = G * S;
    const ssa_u64 n_ids = id_end - id_begin;
    const ssa_u64 span = next_pow2(n_ids);
    const ssa_u64 budget = (o && o->staging_budget_bytes) ? o->staging_budget_bytes : (32ull << 30);
    int path = o ? o->path : SSA_PATH_AUTO;
    if (path == SSA_PATH_AUTO) path = auto_path(*m);
    if (path != SSA_PATH_THREAD && path != SSA_PATH_WARP && path != SSA_PATH_HALFWARP)
        return fail(SSA_ERR_INVALID_ARG, "bad path %d", path);
    info.path = path;
    ssa_u64 C = span;
    if (rec && (path != SSA_PATH_THREAD || sw))
        return fail(SSA_ERR_UNSUPPORTED, "event recording runs on the thread path");
    if (sw) {
        // chunk = as many whole sweep points as the staging budget and the
        // shared-memory constant rows (<= 32 KiB) allow
        if (path != SSA_PATH_THREAD) return fail(SSA_ERR_UNSUPPORTED, "parameter sweeps run on the thread path");
        const ssa_u64 per_point = sw->N * cells * 4ull;
        ssa_u64 pts = std::min<ssa_u64>((ssa_u64)sw->P, budget / per_point);
        pts = std::min<ssa_u64>(pts, (32768 / 8) / (ssa_u64)sw->L.n);
        if (pts == 0)
            return fail(SSA_ERR_UNSUPPORTED, "sweep point staging (%llu B) exceeds the staging budget",
                        (unsigned long long)per_point);
        C = pts * sw->N;
    } else {
        // chunk size: a power of two (aligned subtree), staging within the budget
        if (o && o->chunk) {
            if (o->chunk & (o->chunk - 1)) return fail(SSA_ERR_INVALID_ARG, "chunk %llu is not a power of two", (unsigned long long)o->chunk);
            C = std::min<ssa_u64>(span, o->chunk);
        }
        while (C > 1 && C * cells * 4ull > budget) C >>= 1;
    }
    const ssa_u64 n_chunks = (n_ids + C - 1) / C;

    int sms = 0;
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));

    // kernels for this model on this device (JIT on first use)
    K1Entry* k1 = nullptr;
    K2Dev* k2 = nullptr;
    K2Kernel* k2k = nullptr;
    int block = (o && o->block > 0) ? o->block : (path == SSA_PATH_THREAD ? 128 : SSA_K2_BLOCK);
    if (block % 32 || block > 1024) return fail(SSA_ERR_INVALID_ARG, "block %d must be a multiple of 32 <= 1024", block);
    int grid = 0;
    bool spread = false;
    K1Spec spec;              // K1 dispatch profile: measured on the first plain run, then applied
    double* prof = nullptr;   // the profiling run's share sums (device, [R])
    {
        std::lock_guard<std::mutex> lk(m->mu);
        if (path == SSA_PATH_THREAD) {
            // blocks_per_sm > 0 also sets the K1 variant's __launch_bounds__ residency
            // target (its register budget is 64K / (block * blocks_per_sm))
            // small ensembles (at most one trajectory per SM sub-partition) are spread:
            // one working lane per block of one warp (knob spread32: a variant JIT'd for
            // that launch shape, __launch_bounds__(32, 1))
            const bool spread_n = n_ids <= (ssa_u64)sms * 4 && !(o && o->block > 0);
            const bool s32 = spread_n && k1_gen().spread32;
            const int kblock = s32 ? 32 : block;
            const int minb = (o && o->blocks_per_sm > 0) ? o->blocks_per_sm : (s32 ? 1 : default_minb(*m, block));
            // seed -1 is reserved for "keys from the parameters" (a seed of 2^64-1 takes that path)
            // (kernels per seed are cached; past 32 compiled variants of this model on
            // this device, new seeds take the launch-parameter keys to bound the cache)
            if (!sw) {
                if (m->hot_known) {
                    spec.hot = m->hot;
                } else if (k1_gen().hot.empty()) {
                    spec.prof = true;
                    DevCache& dc = m->dev[c.device];
                    if (!dc.prof) CU(cudaMalloc(&dc.prof, sizeof(double) * ((size_t)m->R + 1)));
                    prof = dc.prof;
                }
            }
            long long kseed = k1_gen().seed_imm ? (long long)seed : -1;
            if (kseed != -1 && m->dev[c.device].k1.size() >= 32 &&
                !m->dev[c.device].k1.count(k1_key(kblock, minb, dump && dump->n > 0, sw ? &sw->L : nullptr, kseed,
                                                  rec ? rec->mode : 0, &spec)))
                kseed = -1;
            TRY(ensure_k1(*m, c.device, kblock, minb, dump && dump->n > 0, sw ? &sw->L : nullptr, &k1, &info.jit_ms,
                          kseed, rec ? rec->mode : 0, &spec));
            int bps = k1->blocks_per_sm;
            if (o && o->blocks_per_sm > 0) bps = std::min(bps, o->blocks_per_sm);
            grid = sms * bps;
            grid = (int)std::min<ssa_u64>((ssa_u64)grid, (C + block - 1) / block);
            // small ensembles (at most one trajectory per SM sub-partition): one
            // working lane per block of one warp, spread over the SMs
            if (spread_n) {
                spread = true;
                grid = (int)n_ids;
            }
        } else {
            // default residency: 4 x 256 threads for one trajectory per warp (64
            // registers), 3 x 256 for two per warp (80 registers)
            const int minb = (o && o->blocks_per_sm > 0) ? o->blocks_per_sm : (path == SSA_PATH_HALFWARP ? 3 : 4);
            TRY(ensure_k2(*m, c.device, block, minb, dump && dump->n > 0, &k2, &k2k, &info.jit_ms,
                          path == SSA_PATH_HALFWARP));
            int bps = k2k->blocks_per_sm;
            if (o && o->blocks_per_sm > 0) bps = std::min(bps, o->blocks_per_sm);
            const int tpb = (block / 32) * (path == SSA_PATH_HALFWARP ? 2 : 1);   // trajectories per block
            grid = sms * bps;
            grid = (int)std::min<ssa_u64>((ssa_u64)grid, (C + tpb - 1) / tpb);
        }
    }
    grid = std::max(grid, 1);
    cudaStream_t st = c.st;

    // the run's model inputs: one async copy from page-locked host memory
    if (path == SSA_PATH_THREAD) {
        double* pc = nullptr;
        size_t bytes = 0, n_pool = 0;
        {
            std::lock_guard<std::mutex> lk(m->mu);
            TRY(pinned_constants(*m, &pc, &bytes, &n_pool));
        }
        if (!sw) {
            CU(cudaMemcpyAsync(k1->c_k, pc, 8 * n_pool, cudaMemcpyHostToDevice, st));
            info.h2d += 8 * n_pool;
        }
        CU(cudaMemcpyAsync(k1->c_x0, pc + n_pool, 8 * (size_t)m->S, cudaMemcpyHostToDevice, st));
        info.h2d += 8 * (size_t)m->S;
    } else {
        CU(cudaMemcpyAsync(k2->dev_image, k2->host_image, k2->image_bytes, cudaMemcpyHostToDevice, st));
        info.h2d += k2->image_bytes;
    }

    // buffers
    DevBuf staging, tiles, croots, statsb, work, dids, dstates, de, dt_, dsum, pconst, ptev, ptord;
    // staging is trajectory-major: trajectory rel's grid samples are one row of `stride` ints
    // (cells rounded up to 8: rows of whole 32-byte sectors), element (rel, k*S + s).  The SSA
    // kernels write a crossing's S counts contiguously, so a lane fills whole sectors over its
    // consecutive crossings (no partial-sector read-modify-writes in DRAM), and K3 reads each
    // trajectory's 8-cell groups as whole sectors.
    const ssa_u64 stride = (cells + 7) / 8 * 8;
    CU(staging.alloc(sizeof(int) * stride * C, st));
    const ssa_u64 seg = sw ? sw->N : C;                   // ids per reduced segment (a point, or the chunk)
    const ssa_u64 n_tiles = (seg + SSA_TREE_SPAN - 1) / SSA_TREE_SPAN;
    if (n_tiles > 1) CU(tiles.alloc(sizeof(double) * 3 * cells * n_tiles, st));
    if (n_chunks > 1 && !sw) CU(croots.alloc(sizeof(double) * 3 * cells * n_chunks, st));
    if (sw) {
        CU(pconst.alloc(sizeof(double) * sw->L.values.size(), st));
        CU(cudaMemcpyAsync(pconst.p, sw->L.values.data(), sizeof(double) * sw->L.values.size(),
                           cudaMemcpyHostToDevice, st));
        info.h2d += sizeof(double) * sw->L.values.size();
        CU(ptev.alloc(sizeof(ssa_u64) * (size_t)sw->P, st));
        CU(cudaMemsetAsync(ptev.p, 0, sizeof(ssa_u64) * (size_t)sw->P, st));
        if ((int)sw->cost.size() == sw->P) {
            // longest-processing-time order within each chunk: the costliest points' trajectories
            // are handed out first, so the end of the launch is not one long trajectory started late
            const ssa_u64 ppc = C / sw->N;   // points per chunk
            std::vector<int> ord((size_t)sw->P);
            for (ssa_u64 p0 = 0; p0 < (ssa_u64)sw->P; p0 += ppc) {
                const ssa_u64 p1 = std::min<ssa_u64>((ssa_u64)sw->P, p0 + ppc);
                std::vector<int> loc;
                for (ssa_u64 q = p0; q < p1; ++q) loc.push_back((int)(q - p0));
                std::stable_sort(loc.begin(), loc.end(), [&](int a, int b) {
                    return sw->cost[(size_t)(p0 + a)] > sw->cost[(size_t)(p0 + b)];
                });
                for (size_t q = 0; q < loc.size(); ++q) ord[(size_t)(p0 + q)] = loc[q];
            }
            CU(ptord.alloc(sizeof(int) * ord.size(), st));
            CU(cudaMemcpyAsync(ptord.p, ord.data(), sizeof(int) * ord.size(), cudaMemcpyHostToDevice, st));
            CU(cudaStreamSynchronize(st));   // ord is a local
            info.h2d += sizeof(int) * ord.size();
        }
    }
    // tail compaction (K1 plain / dump / profiling variants, not for small spread ensembles): the
    // suspended-trajectory buffer, its ready flags and the control words
    const int tail_lanes = (o && o->tail_lanes) ? o->tail_lanes : -1;   // default off
    const bool mig = path == SSA_PATH_THREAD && !sw && !rec && !spread && tail_lanes > 0;
    DevBuf migb, migr, migc;
    const ssa_u64 mig_rec = (ssa_u64)m->S + 6, mig_cap = 4 * (ssa_u64)grid * (ssa_u64)block;
    ssa_u64 mig_host[4] = {0, 0, 0, 0};
    if (mig) {
        CU(migb.alloc(sizeof(double) * mig_rec * mig_cap, st));
        CU(migr.alloc(sizeof(unsigned) * mig_cap, st));
        CU(migc.alloc(sizeof(ssa_u64) * 4, st));
    }
    // time-sliced trajectories (K1 plain / dump / profiling variants): each trajectory runs as
    // SSA_TSLICES phases handed out phase by phase, so a launch ends with short last phases instead
    // of whole trajectories on an emptying GPU (bitwise neutral).  Used when a launch
    // has more trajectories than resident lanes; SSA_K1_SEG overrides the phase count (1 = off).
    int tslices = SSA_TSLICES;
    if (const char* sv = getenv("SSA_K1_SEG")) tslices = std::max(1, std::min(64, atoi(sv)));
    if (path != SSA_PATH_THREAD || sw || rec || spread || mig || (ssa_u64)C <= (ssa_u64)grid * (ssa_u64)block)
        tslices = 1;
    DevBuf segb, segr;
    if (tslices > 1) {
        CU(segb.alloc(sizeof(double) * ((size_t)m->S + 6) * (size_t)C, st));
        CU(segr.alloc(sizeof(unsigned) * (size_t)C, st));
    }
    CU(statsb.alloc(sizeof(ssa_dev_stats), st));
    CU(work.alloc(sizeof(ssa_u64) * n_chunks, st));
    CU(cudaMemsetAsync(statsb.p, 0, sizeof(ssa_dev_stats), st));
    CU(cudaMemsetAsync((char*)statsb.p + offsetof(ssa_dev_stats, first_err_id), 0xFF, sizeof(ssa_u64), st));
    CU(cudaMemsetAsync(work.p, 0, sizeof(ssa_u64) * n_chunks, st));
    if (prof) CU(cudaMemsetAsync(prof, 0, sizeof(double) * ((size_t)m->R + 1), st));

    // dump
    ssa_u64 n_dump = dump ? dump->n : 0;
    int* p_states = nullptr;
    ssa_u64* p_e = nullptr;
    double* p_t = nullptr;
    ssa_dev_summary* p_sum = nullptr;
    if (n_dump) {
        if (!dump->ids) return fail(SSA_ERR_INVALID_ARG, "dump ids null");
        for (ssa_u64 i = 0; i < n_dump; ++i) {
            if (i && dump->ids[i] <= dump->ids[i - 1]) return fail(SSA_ERR_INVALID_ARG, "dump ids must be sorted and unique");
            if (dump->ids[i] < id_begin || dump->ids[i] >= id_end)
                return fail(SSA_ERR_INVALID_ARG, "dump id %llu outside [%llu, %llu)", (unsigned long long)dump->ids[i],
                            (unsigned long long)id_begin, (unsigned long long)id_end);
        }
        CU(dids.alloc(sizeof(ssa_u64) * n_dump, st));
        CU(cudaMemcpyAsync(dids.p, dump->ids, sizeof(ssa_u64) * n_dump, cudaMemcpyHostToDevice, st));
        info.h2d += sizeof(ssa_u64) * n_dump;
        if (dump_on_device) {
            p_states = dump->states; p_e = (ssa_u64*)dump->events_at; p_t = dump->time_at; p_sum = (ssa_dev_summary*)dump->summary;
        }
        if (!p_states) { CU(dstates.alloc(sizeof(int) * n_dump * cells, st)); p_states = dstates.as<int>(); }
        if (!p_e) { CU(de.alloc(sizeof(ssa_u64) * n_dump * G, st)); p_e = de.as<ssa_u64>(); }
        if (!p_t) { CU(dt_.alloc(sizeof(double) * n_dump * G, st)); p_t = dt_.as<double>(); }
        if (!p_sum) { CU(dsum.alloc(sizeof(ssa_dev_summary) * n_dump, st)); p_sum = dsum.as<ssa_dev_summary>(); }
    }

    Events<5> eg;
    CU(eg.create());
    cudaEvent_t ev0 = eg.e[0], ev1 = eg.e[1], evs0 = eg.e[2], evs1 = eg.e[3], evr1 = eg.e[4];
    CU(cudaEventRecord(ev0, st));
    float ssa_ms_total = 0.f, reduce_ms_total = 0.f;

    const ssa_u32 key0 = (ssa_u32)seed, key1 = (ssa_u32)(seed >> 32);
    for (ssa_u64 ch = 0; ch < n_chunks; ++ch) {
        const ssa_u64 cb = id_begin + ch * C;
        const ssa_u64 cn = std::min<ssa_u64>(C, id_end - cb);
        CU(cudaEventRecord(evs0, st));
        if (path == SSA_PATH_THREAD) {
            ssa_k1_params p{};
            p.id_begin = cb; p.n_ids = cn; p.staging = staging.as<int>(); p.stride = stride; p.dt = dt; p.K = K;
            p.key0 = key0; p.key1 = key1; p.work = work.as<ssa_u64>() + ch;
            for (int r = 0; r < 10; ++r) {  // Philox key schedule (mod 2^32)
                p.ks[2 * r] = key0 + (ssa_u32)r * 0x9E3779B9u;
                p.ks[2 * r + 1] = key1 + (ssa_u32)r * 0xBB67AE85u;
            }
            p.dump_ids = dids.as<ssa_u64>(); p.n_dump = n_dump; p.dump_states = p_states; p.dump_e = p_e;
            p.dump_t = p_t; p.dump_sum = p_sum; p.stats = statsb.as<ssa_dev_stats>();
            if (rec) {
                p.rec_count = rec->count; p.rec_cap = rec->cap; p.rec_key = rec->key; p.rec_stride = rec->stride;
                p.rec_t = rec->t; p.rec_j = rec->j; p.rec_pre = rec->pre;
            }
            size_t smem = 0;
            if (sw) {
                p.n_per_point = sw->N;
                p.n_pts = (int)(cn / sw->N);
                p.n_pool = sw->L.n;
                p.pconst = pconst.as<double>() + (cb / sw->N) * (ssa_u64)sw->L.n;
                smem = sizeof(double) * (size_t)p.n_pts * (size_t)p.n_pool;
                p.pt_events = ptev.as<ssa_u64>() + cb / sw->N;
                p.pt_order = ptord.p ? (const int*)ptord.p + cb / sw->N : nullptr;
            }
            p.spread = spread ? 1 : 0;
            p.prof = prof;
            if (mig) {
                ssa_u64 ctl[4] = {0, 0, cn, 0};   // pushed, taken, trajectories to finish, warps running
                CU(cudaMemcpyAsync(migc.p, ctl, sizeof ctl, cudaMemcpyHostToDevice, st));
                CU(cudaMemsetAsync(migr.p, 0, sizeof(unsigned) * mig_cap, st));
                CU(cudaStreamSynchronize(st));   // ctl is a local
                p.mig_thresh = tail_lanes;
                p.mig_buf = migb.as<double>();
                p.mig_ready = migr.as<unsigned>();
                p.mig_cap = mig_cap;
                p.mig_ctl = migc.as<ssa_u64>();
            }
            if (tslices > 1 && cn > (ssa_u64)grid * (ssa_u64)block) {
                CU(cudaMemsetAsync(segr.p, 0, sizeof(unsigned) * (size_t)cn, st));
                p.seg = tslices;
                p.seg_buf = segb.as<double>();
                p.seg_ready = segr.as<unsigned>();
            }
            void* args[] = {&p};
            CU(cudaLaunchKernel((const void*)k1->fn, dim3(grid), dim3(spread ? 32 : block), args, smem, st));
            info.launches += 1;
            info.lanes = std::max<uint64_t>(info.lanes, (uint64_t)grid * (spread ? 1 : block));
            if (mig) {
                CU(cudaMemcpyAsync(mig_host, migc.p, sizeof mig_host, cudaMemcpyDeviceToHost, st));
                CU(cudaStreamSynchronize(st));
                if (getenv("SSA_DEBUG_TAIL"))
                    fprintf(stderr, "[ssa tail] chunk %llu: %llu suspended, %llu resumed, %llu unfinished\n",
                            (unsigned long long)ch, (unsigned long long)mig_host[0], (unsigned long long)mig_host[1],
                            (unsigned long long)mig_host[2]);
                if (mig_host[0] != mig_host[1] || mig_host[2] != 0 || mig_host[3] != 0)
                    return fail(SSA_ERR_CUDA, "tail compaction: %llu suspended, %llu resumed, %llu unfinished",
                                (unsigned long long)mig_host[0], (unsigned long long)mig_host[1],
                                (unsigned long long)mig_host[2]);
            }
        } else {
            ssa_k2_params p{};
            p.n_ent = k2->n_ent; p.n_dep = k2->n_dep;
            p.pk = k2->pk; p.gw = k2->gw; p.rate = k2->rate; p.modc = k2->modc; p.x0 = k2->x0; p.nu_off = k2->nu_off; p.nu_ent = k2->nu_ent;
            p.dep_off = k2->dep_off; p.dep_ent = k2->dep_ent;
            p.rxd_offset = k2k->rxd_offset;
            p.rec = k2->rec; p.dent = k2->dent; p.rfe = k2->rfe;
            p.rec_offset = k2k->rec_offset; p.dent_offset = k2k->dent_offset;
            p.id_begin = cb; p.n_ids = cn; p.staging = staging.as<int>(); p.stride = stride; p.dt = dt; p.K = K;
            p.key0 = key0; p.key1 = key1; p.work = work.as<ssa_u64>() + ch;
            p.dump_ids = dids.as<ssa_u64>(); p.n_dump = n_dump; p.dump_states = p_states; p.dump_e = p_e;
            p.dump_t = p_t; p.dump_sum = p_sum; p.stats = statsb.as<ssa_dev_stats>();
            void* args[] = {&p};
            CU(cudaLaunchKernel((const void*)k2k->fn, dim3(grid), dim3(block), args, k2k->smem, st));
            info.launches += 1;
        }
        CU(cudaGetLastError());
        CU(cudaEventRecord(evs1, st));
        // a9: reduce each segment (the chunk, or each sweep point in it) to its
        // root: the chunk root, the range root when there is one chunk, or the
        // point's root
        const ssa_u64 n_seg = sw ? cn / sw->N : 1;
        for (ssa_u64 q = 0; q < n_seg; ++q) {
            const ssa_u64 sn = sw ? sw->N : cn;
            const int* src = staging.as<int>() + q * seg * stride;
            ssa_tree_out seg_out;
            if (sw) {
                const RangeOut& pr = sw->roots[(size_t)(cb / sw->N + q)];
                seg_out = ssa_tree_out{pr.n, pr.mean, pr.m2, 1, 0, 0};
            } else if (n_chunks > 1) {
                double* b = croots.as<double>();
                seg_out = ssa_tree_out{b, b + cells * n_chunks, b + 2 * cells * n_chunks, n_chunks, 0, ch};
            } else {
                seg_out = ssa_tree_out{root.n, root.mean, root.m2, 1, 0, 0};
            }
            if (n_tiles > 1) {
                double* b = tiles.as<double>();
                ssa_tree_out to{b, b + cells * n_tiles, b + 2 * cells * n_tiles, n_tiles, 1, 0};
                CU(ssa_tree_leaf_launch(src, stride, sn, cells, to, st, &info.launches));
                // only the tiles holding this segment's ids were written (a ragged chunk
                // has fewer than n_tiles): the merge treats positions >= count as empty
                // leaves, the identity, so the tree keeps its shape and its bits
                const ssa_u64 written = (sn + SSA_TREE_SPAN - 1) / SSA_TREE_SPAN;
                TRY(reduce_partials(ssa_tree_in{to.n, to.mean, to.m2, n_tiles, 1}, written, cells, seg_out, st,
                                    &info.launches));
            } else {
                CU(ssa_tree_leaf_launch(src, stride, sn, cells, seg_out, st, &info.launches));
            }
        }
        CU(cudaEventRecord(evr1, st));
        CU(cudaEventSynchronize(evr1));
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, evs0, evs1));
        ssa_ms_total += ms;
        CU(cudaEventElapsedTime(&ms, evs1, evr1));
        reduce_ms_total += ms;
        info.reduce_bytes += cn * cells * sizeof(int);
    }
    // a10 (per GPU): chunk roots -> range root
    if (n_chunks > 1 && !sw) {
        double* b = croots.as<double>();
        TRY(reduce_partials(ssa_tree_in{b, b + cells * n_chunks, b + 2 * cells * n_chunks, n_chunks, 1}, n_chunks, cells,
                            ssa_tree_out{root.n, root.mean, root.m2, 1, 0, 0}, st, &info.launches));
    }
    CU(cudaEventRecord(ev1, st));
    CU(cudaMemcpyAsync(&info.stats, statsb.p, sizeof(ssa_dev_stats), cudaMemcpyDeviceToHost, st));
    info.d2h += sizeof(ssa_dev_stats);
    Events<2> evd;   // the dump copy's events
    if (n_dump) {
        info.dump_bytes = (dump->states ? sizeof(int) * n_dump * cells : 0) + (dump->events_at ? 8 * n_dump * G : 0) +
                          (dump->time_at ? 8 * n_dump * G : 0) + (dump->summary ? sizeof(ssa_dev_summary) * n_dump : 0);
    }
    if (n_dump && !dump_on_device) {
        info.d2h += info.dump_bytes;
        CU(evd.create());
        CU(cudaEventRecord(evd.e[0], st));
        if (dump->states) CU(cudaMemcpyAsync(dump->states, p_states, sizeof(int) * n_dump * cells, cudaMemcpyDeviceToHost, st));
        if (dump->events_at) CU(cudaMemcpyAsync(dump->events_at, p_e, sizeof(ssa_u64) * n_dump * G, cudaMemcpyDeviceToHost, st));
        if (dump->time_at) CU(cudaMemcpyAsync(dump->time_at, p_t, sizeof(double) * n_dump * G, cudaMemcpyDeviceToHost, st));
        if (dump->summary) CU(cudaMemcpyAsync(dump->summary, p_sum, sizeof(ssa_dev_summary) * n_dump, cudaMemcpyDeviceToHost, st));
        CU(cudaEventRecord(evd.e[1], st));
    }
    CU(cudaStreamSynchronize(st));
    float ms = 0.f;
    if (evd.e[0]) {
        CU(cudaEventElapsedTime(&ms, evd.e[0], evd.e[1]));
        info.dump_ms = ms;
    }
    CU(cudaEventElapsedTime(&ms, ev0, ev1));
    info.device_ms = ms;
    info.ssa_ms = ssa_ms_total;
    info.reduce_ms = reduce_ms_total;
    if (sw) {
        sw->events.assign((size_t)sw->P, 0);
        CU(cudaMemcpy(sw->events.data(), ptev.p, sizeof(ssa_u64) * (size_t)sw->P, cudaMemcpyDeviceToHost));
    }
    if (prof) {
        // choose the hot set from the sampled propensity shares (their mean estimates each
        // reaction's share of the events): the top reaction if it carries >= 1/2 of them,
        // the second too if the two carry >= 80% (more hot reactions measured slower,
        // DESIGN.md §6); at least 32 samples
        std::vector<double> h((size_t)m->R + 1);
        CU(cudaMemcpy(h.data(), prof, sizeof(double) * h.size(), cudaMemcpyDeviceToHost));
        const double samples = h[(size_t)m->R];
        h.pop_back();
        double tot = 0.0;
        for (double v : h) tot += v;
        if (samples >= 32.0 && tot > 0.0) {
            std::vector<int> idx((size_t)m->R);
            for (int j = 0; j < m->R; ++j) idx[(size_t)j] = j;
            std::sort(idx.begin(), idx.end(), [&](int a, int b) { return h[(size_t)a] > h[(size_t)b]; });
            std::vector<int> hot;
            const double s1 = m->R > 0 ? h[(size_t)idx[0]] / tot : 0.0;
            const double s2 = m->R > 1 ? h[(size_t)idx[1]] / tot : 0.0;
            if (s1 >= 0.5) hot.push_back(idx[0]);
            if (s1 >= 0.5 && s1 + s2 >= 0.8 && s2 > 0.05) hot.push_back(idx[1]);
            std::lock_guard<std::mutex> lk(m->mu);
            m->hot = hot;
            m->hot_known = true;
        }
    }
    return SSA_OK;
}

static ssa_status fill_result(const RunInfo& info, ssa_result* r)
{
    if (info.stats.pad[0])
        return fail(SSA_ERR_CUDA, "device bounds checks failed %llu times (SSA_DEBUG_CHECKS)",
                    (unsigned long long)info.stats.pad[0]);
    r->events = info.stats.events;
    r->near_ties = info.stats.near_ties;
    r->n_errors = info.stats.n_errors;
    r->first_error_id = 0;
    r->first_error_reaction = -1;
    r->path_used = info.path;
    r->device_ms = info.device_ms;
    r->ssa_ms = info.ssa_ms;
    r->reduce_ms = info.reduce_ms;
    r->reduce_bytes = info.reduce_bytes;
    r->dump_ms = info.dump_ms;
    r->dump_bytes = info.dump_bytes;
    r->jit_ms = info.jit_ms;
    r->h2d_bytes = info.h2d;
    r->d2h_bytes = info.d2h;
    r->kernel_launches = info.launches;
    if (info.stats.n_errors) {
        const ssa_u64 packed = info.stats.first_err_id;
        const ssa_u64 id = packed >> 24, code = (packed >> 20) & 0xF;
        const int rx = (int)(packed & 0xFFFFF) - 1;
        r->first_error_id = id;
        r->first_error_reaction = rx;
        if (code == SSA_DEV_ERR_NUMERIC)
            return fail(SSA_ERR_NUMERIC, "trajectory %llu: non-finite propensity (reaction %d)", (unsigned long long)id, rx);
        return fail(SSA_ERR_OVERFLOW, "trajectory %llu: species count exceeded INT32_MAX", (unsigned long long)id);
    }
    return SSA_OK;
}

static ssa_status check_common(const ssa_model* m, double t_end, double dt, ssa_result* r)
{
    if (!m) return fail(SSA_ERR_INVALID_ARG, "model is null");
    if (!r) return fail(SSA_ERR_INVALID_ARG, "result is null");
    if (!(t_end > 0.0) || !std::isfinite(t_end)) return fail(SSA_ERR_INVALID_ARG, "t_end must be finite and > 0");
    if (!(dt > 0.0) || !std::isfinite(dt)) return fail(SSA_ERR_INVALID_ARG, "sample_dt must be finite and > 0");
    if (ssa_grid_size(t_end, dt) == 0 || ssa_grid_size(t_end, dt) > (1ull << 26))
        return fail(SSA_ERR_INVALID_ARG, "grid too large");
    return SSA_OK;
}

// poisoned: the run had trajectories that ended in an error (their grid rows past
// the error are not samples of the method), so mean, var and M2 are NaN; count
// is still written
static ssa_status finalize_to(const double* rn, const double* rmean, const double* rm2, ssa_u64 cells, uint32_t reducers,
                              ssa_result* r, bool on_device, cudaStream_t st, bool poisoned = false)
{
    double* om = (reducers & SSA_REDUCE_MEAN) ? r->mean : nullptr;
    double* ov = (reducers & SSA_REDUCE_VAR) ? r->var : nullptr;
    double* o2 = r->m2;
    double* oc = r->count;
    r->kernel_launches += 1;
    if (on_device) {
        CU(ssa_finalize_launch(rn, rmean, rm2, cells, om, ov, o2, oc, st));
        if (poisoned)   // all-ones bytes are a quiet NaN
            for (double* q : {om, ov, o2})
                if (q) CU(cudaMemsetAsync(q, 0xFF, sizeof(double) * cells, st));
        CU(cudaStreamSynchronize(st));
        return SSA_OK;
    }
    r->d2h_bytes += sizeof(double) * cells * ((om ? 1 : 0) + (ov ? 1 : 0) + (o2 ? 1 : 0) + (oc ? 1 : 0));
    DevBuf out;
    CU(out.alloc(sizeof(double) * 4 * cells, st));
    double* d = out.as<double>();
    CU(ssa_finalize_launch(rn, rmean, rm2, cells, d, d + cells, d + 2 * cells, d + 3 * cells, st));
    if (om) CU(cudaMemcpyAsync(om, d, sizeof(double) * cells, cudaMemcpyDeviceToHost, st));
    if (ov) CU(cudaMemcpyAsync(ov, d + cells, sizeof(double) * cells, cudaMemcpyDeviceToHost, st));
    if (o2) CU(cudaMemcpyAsync(o2, d + 2 * cells, sizeof(double) * cells, cudaMemcpyDeviceToHost, st));
    if (oc) CU(cudaMemcpyAsync(oc, d + 3 * cells, sizeof(double) * cells, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (poisoned)
        for (double* q : {om, ov, o2})
            if (q) std::fill(q, q + cells, std::numeric_limits<double>::quiet_NaN());
    return SSA_OK;
}

extern "C" ssa_status ssa_run(const ssa_model* m, uint64_t n_trajectories, double t_end, double sample_dt,
                              uint64_t seed, uint32_t reducers, const ssa_run_options* o, ssa_result* r)
{
    TRY(check_common(m, t_end, sample_dt, r));
    if (n_trajectories == 0) return fail(SSA_ERR_INVALID_ARG, "n_trajectories must be >= 1");
    if (n_trajectories > (1ull << 40)) return fail(SSA_ERR_INVALID_ARG, "n_trajectories > 2^40");
    Ctx c;
    TRY(setup_ctx(o, c));
    const ssa_u64 cells = ssa_grid_size(t_end, sample_dt) * (ssa_u64)m->S;
    DevBuf rootb;
    CU(rootb.alloc(sizeof(double) * 3 * cells, c.st));
    double* rb = rootb.as<double>();
    RunInfo info;
    const bool on_dev = o && o->outputs_on_device;
    TRY(run_range(m, 0, n_trajectories, t_end, sample_dt, seed, o, c, RangeOut{rb, rb + cells, rb + 2 * cells}, info,
                  o ? o->dump : nullptr, on_dev));
    ssa_status st = fill_result(info, r);
    TRY(finalize_to(rb, rb + cells, rb + 2 * cells, cells, reducers ? reducers : (SSA_REDUCE_MEAN | SSA_REDUCE_VAR), r,
                    on_dev, c.st, info.stats.n_errors > 0));
    return st;
}

extern "C" ssa_status ssa_run_shard(const ssa_model* m, uint64_t id_begin, uint64_t id_end, double t_end,
                                    double sample_dt, uint64_t seed, double* d_root, const ssa_run_options* o,
                                    ssa_result* r)
{
    TRY(check_common(m, t_end, sample_dt, r));
    if (!d_root) return fail(SSA_ERR_INVALID_ARG, "d_root is null");
    if (id_end <= id_begin) return fail(SSA_ERR_INVALID_ARG, "empty shard");
    if (id_end > (1ull << 40)) return fail(SSA_ERR_INVALID_ARG, "ids beyond 2^40");
    const ssa_u64 span = next_pow2(id_end - id_begin);
    if (id_begin % span) return fail(SSA_ERR_INVALID_ARG, "shard [%llu, %llu) is not an aligned subtree", (unsigned long long)id_begin, (unsigned long long)id_end);
    Ctx c;
    TRY(setup_ctx(o, c));
    const ssa_u64 cells = ssa_grid_size(t_end, sample_dt) * (ssa_u64)m->S;
    RunInfo info;
    TRY(run_range(m, id_begin, id_end, t_end, sample_dt, seed, o, c, RangeOut{d_root, d_root + cells, d_root + 2 * cells},
                  info, o ? o->dump : nullptr, o && o->outputs_on_device));
    if (info.stats.n_errors > 0) {
        // a shard with erroring trajectories has no defined moments: NaN mean and M2
        // (n kept), so every merge that includes this root is NaN as well
        CU(cudaMemsetAsync(d_root + cells, 0xFF, sizeof(double) * 2 * cells, c.st));
        CU(cudaStreamSynchronize(c.st));
    }
    return fill_result(info, r);
}

extern "C" ssa_status ssa_run_sweep(const ssa_model* m, int32_t n_points, const double* rates, const double* mod_coefs,
                                    uint64_t n_per_point, double t_end, double sample_dt, uint64_t seed,
                                    uint32_t reducers, const ssa_run_options* o, ssa_result* r)
{
    TRY(check_common(m, t_end, sample_dt, r));
    if (n_points < 1 || n_points > 65536) return fail(SSA_ERR_INVALID_ARG, "n_points must be in [1, 65536]");
    if (!rates) return fail(SSA_ERR_INVALID_ARG, "rates is null");
    if (n_per_point == 0) return fail(SSA_ERR_INVALID_ARG, "n_per_point must be >= 1");
    if ((ssa_u64)n_points * n_per_point > (1ull << 40)) return fail(SSA_ERR_INVALID_ARG, "n_points * n_per_point > 2^40");
    if (o && (o->path == SSA_PATH_WARP || o->path == SSA_PATH_HALFWARP))
        return fail(SSA_ERR_UNSUPPORTED, "parameter sweeps run on the thread path");
    const size_t R = (size_t)m->R;
    for (size_t i = 0; i < (size_t)n_points * R; ++i) {
        if (!std::isfinite(rates[i]) || rates[i] < 0.0)
            return fail(SSA_ERR_MODEL, "sweep point %zu, reaction %zu: rate must be finite and >= 0", i / R, i % R);
        if (mod_coefs && !std::isfinite(mod_coefs[i]))
            return fail(SSA_ERR_MODEL, "sweep point %zu, reaction %zu: non-finite modifier coefficient", i / R, i % R);
    }
    Ctx c;
    TRY(setup_ctx(o, c));
    const ssa_u64 cells = ssa_grid_size(t_end, sample_dt) * (ssa_u64)m->S;
    SweepSpec sw;
    sw.P = n_points;
    sw.N = n_per_point;
    sw.L = make_pool(*m, n_points, rates, mod_coefs);
    std::string skey;   // this sweep's identity for the point-cost cache
    {
        auto put = [&](const void* q, size_t n) { skey.append((const char*)q, n); };
        put(&n_points, sizeof n_points);
        put(&n_per_point, sizeof n_per_point);
        put(&t_end, sizeof t_end);
        put(&sample_dt, sizeof sample_dt);
        put(rates, sizeof(double) * (size_t)n_points * R);
        if (mod_coefs) put(mod_coefs, sizeof(double) * (size_t)n_points * R);
        std::lock_guard<std::mutex> lk(m->mu);
        auto it = m->sweep_cost.find(skey);
        if (it != m->sweep_cost.end()) sw.cost = it->second;
    }
    DevBuf rootb;
    CU(rootb.alloc(sizeof(double) * 3 * cells * (size_t)n_points, c.st));
    double* rb = rootb.as<double>();
    for (int p = 0; p < n_points; ++p) {
        double* b = rb + (size_t)p * 3 * cells;
        sw.roots.push_back(RangeOut{b, b + cells, b + 2 * cells});
    }
    RunInfo info;
    const bool on_dev = o && o->outputs_on_device;
    ssa_run_options ro = o ? *o : ssa_run_options{};
    ro.path = SSA_PATH_THREAD;   // AUTO included: sweeps run on the thread path at any size
    TRY(run_range(m, 0, (ssa_u64)n_points * n_per_point, t_end, sample_dt, seed, &ro, c, sw.roots[0], info,
                  o ? o->dump : nullptr, on_dev, &sw));
    if ((int)sw.events.size() == n_points) {
        std::vector<double> cost((size_t)n_points);
        for (int q = 0; q < n_points; ++q) cost[(size_t)q] = (double)sw.events[(size_t)q] / (double)n_per_point;
        std::lock_guard<std::mutex> lk(m->mu);
        if (m->sweep_cost.size() >= 64) m->sweep_cost.clear();   // bound the cache
        m->sweep_cost[skey] = cost;
    }
    ssa_status st = fill_result(info, r);
    // finalize every point into its [G*S] slab of the caller's arrays
    for (int p = 0; p < n_points; ++p) {
        ssa_result rp = *r;
        const size_t off = (size_t)p * cells;
        rp.mean = r->mean ? r->mean + off : nullptr;
        rp.var = r->var ? r->var + off : nullptr;
        rp.m2 = r->m2 ? r->m2 + off : nullptr;
        rp.count = r->count ? r->count + off : nullptr;
        rp.kernel_launches = 0;
        rp.d2h_bytes = 0;
        const RangeOut& pr = sw.roots[p];
        TRY(finalize_to(pr.n, pr.mean, pr.m2, cells, reducers ? reducers : (SSA_REDUCE_MEAN | SSA_REDUCE_VAR), &rp,
                        on_dev, c.st, info.stats.n_errors > 0));
        r->kernel_launches += rp.kernel_launches;
        r->d2h_bytes += rp.d2h_bytes;
    }
    return st;
}

extern "C" ssa_status ssa_run_union(const ssa_model* m, uint64_t n_trajectories, double t_end, uint64_t seed,
                                    uint32_t thin_kx, uint64_t capacity, double* times, double* mean, double* var,
                                    double* count, uint64_t* n_points, const ssa_run_options* o, ssa_result* r)
{
    TRY(check_common(m, t_end, t_end, r));
    if (!n_points) return fail(SSA_ERR_INVALID_ARG, "n_points is null");
    *n_points = 0;
    if (n_trajectories == 0 || n_trajectories > (1ull << 24)) return fail(SSA_ERR_INVALID_ARG, "n_trajectories not in [1, 2^24]");
    if (thin_kx == 0) return fail(SSA_ERR_INVALID_ARG, "thin_kx must be >= 1");
    if (o && (o->path == SSA_PATH_WARP || o->path == SSA_PATH_HALFWARP))
        return fail(SSA_ERR_UNSUPPORTED, "event recording runs on the thread path");
    if (o && o->dump) return fail(SSA_ERR_INVALID_ARG, "ssa_run_union takes no dump");
    Ctx c;
    TRY(setup_ctx(o, c));
    cudaStream_t st = c.st;
    const ssa_u64 n = n_trajectories, S = (ssa_u64)m->S;
    const ssa_u64 cells = 2 * S;           // the grid {0, t_end}: a by-product of the runs
    ssa_run_options ro = o ? *o : ssa_run_options{};
    ro.path = SSA_PATH_THREAD;
    ro.dump = nullptr;
    ro.outputs_on_device = 0;
    DevBuf rootb;
    CU(rootb.alloc(sizeof(double) * 3 * cells, st));
    double* rb = rootb.as<double>();
    // one recording run (events appended in any order: they are sorted by time
    // next); if the record buffer was too small, run again with the exact size
    int U = 1;
    for (int j = 0; j < m->R; ++j) U = std::max(U, (int)m->rx[j].nu.size());
    const size_t row = 12 + 4 * (size_t)U;
    size_t free_b = 0, total_b = 0;
    CU(cudaMemGetInfo(&free_b, &total_b));
    ssa_u64 cap = std::min<ssa_u64>((ssa_u64)(free_b / 8) / row, 1ull << 27);   // first guess: <= 1/8 of free HBM
    if (const char* g = getenv("SSA_UNION_CAP0")) cap = strtoull(g, nullptr, 10);   // test hook: force the re-run
    RunInfo info, info1;
    DevBuf dcount, rt, rj, rpre;
    CU(dcount.alloc(8, st));
    ssa_u64 E = 0, rows = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        rt.reset(); rj.reset(); rpre.reset();
        CU(rt.alloc(8 * std::max<ssa_u64>(cap, 1), st));
        CU(rj.alloc(4 * std::max<ssa_u64>(cap, 1), st));
        CU(rpre.alloc(4 * (size_t)U * std::max<ssa_u64>(cap, 1), st));
        CU(cudaMemsetAsync(dcount.p, 0, 8, st));
        RecordSpec rec{1, 0, nullptr, dcount.as<ssa_u64>(), cap, rt.as<double>(), rj.as<int>(), rpre.as<int>()};
        RunInfo& ri = attempt == 0 ? info : info1;
        ri = RunInfo();
        TRY(run_range(m, 0, n, t_end, t_end, seed, &ro, c, RangeOut{rb, rb + cells, rb + 2 * cells}, ri, nullptr,
                      false, nullptr, &rec));
        TRY(fill_result(ri, r));
        CU(cudaMemcpy(&rows, dcount.p, 8, cudaMemcpyDeviceToHost));
        if (rows <= cap) {
            if (attempt == 1) info = info1;
            break;
        }
        // rare: size the second run.  Which trajectories a lane gets depends on the
        // schedule, so its reserved rows can differ from this run's; each lane leaves
        // at most one partly used block, so rows + lanes * block bounds any run.
        cap = rows + ri.lanes * 256ull;
    }
    if (rows > cap)
        return fail(SSA_ERR_OOM, "event record overflow (%llu rows reserved, capacity %llu)", (unsigned long long)rows,
                    (unsigned long long)cap);
    E = info.stats.events;   // valid rows: the first E after sorting by time (unused rows are +inf)
    // model tables for the reduction: changed species and net changes, ensemble sums of x0, x0^2
    const int R1 = std::max(m->R, 1);
    std::vector<int> nsp((size_t)R1 * U, -1), nd((size_t)R1 * U, 0);
    for (int j = 0; j < m->R; ++j)
        for (size_t q = 0; q < m->rx[j].nu.size(); ++q) {
            nsp[(size_t)j * U + q] = m->rx[j].nu[q].first;
            nd[(size_t)j * U + q] = (int)m->rx[j].nu[q].second;
        }
    std::vector<long long> s0(S), s0sq(S);
    for (ssa_u64 q = 0; q < S; ++q) {
        s0[q] = (long long)n * m->x0[q];
        s0sq[q] = (long long)n * m->x0[q] * m->x0[q];
    }
    DevBuf dnsp, dnd, ds0, ds0sq, dout;
    CU(dnsp.alloc(4 * nsp.size(), st));
    CU(dnd.alloc(4 * nd.size(), st));
    CU(ds0.alloc(8 * S, st));
    CU(ds0sq.alloc(8 * S, st));
    CU(cudaMemcpyAsync(dnsp.p, nsp.data(), 4 * nsp.size(), cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(dnd.p, nd.data(), 4 * nd.size(), cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(ds0.p, s0.data(), 8 * S, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(ds0sq.p, s0sq.data(), 8 * S, cudaMemcpyHostToDevice, st));
    const bool on_dev = o && o->outputs_on_device;
    ssa_union_args a{};
    a.E = E; a.rows = rows; a.rec_t = rt.as<double>(); a.rec_j = rj.as<int>(); a.rec_pre = rpre.as<int>(); a.U = U;
    a.S = (int)S; a.nu_sp = dnsp.as<int>(); a.nu_d = dnd.as<int>(); a.s0 = ds0.as<long long>();
    a.s0sq = ds0sq.as<long long>(); a.k = n; a.t_end = t_end; a.kx = thin_kx; a.capacity = capacity;
    if (on_dev) {
        a.times = times; a.mean = mean; a.var = var; a.count = count;
    } else if (capacity) {
        CU(dout.alloc(sizeof(double) * capacity * (2 + 2 * S), st));
        double* b = dout.as<double>();
        a.times = b; a.count = b + capacity; a.mean = b + 2 * capacity; a.var = b + (2 + S) * capacity;
    }
    Events<2> ev;
    CU(ev.create());
    cudaEvent_t e0 = ev.e[0], e1 = ev.e[1];
    CU(cudaEventRecord(e0, st));
    ssa_u64 np = 0;
    int launches = 0;
    CU(ssa_union_reduce(a, st, &np, &launches));
    CU(cudaEventRecord(e1, st));
    CU(cudaEventSynchronize(e1));
    float ums = 0.f;
    cudaEventElapsedTime(&ums, e0, e1);
    *n_points = np;
    r->events = info.stats.events;
    r->near_ties = info.stats.near_ties;
    r->device_ms = info.device_ms + ums;
    r->ssa_ms = info.ssa_ms;
    r->reduce_ms = ums;
    r->reduce_bytes = E * (8 + 4 + 4 * (ssa_u64)U);
    r->dump_ms = 0.0;
    r->dump_bytes = 0;
    r->jit_ms = info.jit_ms;
    r->kernel_launches = info.launches + launches;
    r->h2d_bytes = info.h2d + 8 * (nsp.size() + 2 * S);
    if (np > capacity)
        return fail(SSA_ERR_INVALID_ARG, "capacity %llu < %llu output points (n_points holds the size needed)",
                    (unsigned long long)capacity, (unsigned long long)np);
    if (!on_dev) {
        if (times) CU(cudaMemcpyAsync(times, a.times, 8 * np, cudaMemcpyDeviceToHost, st));
        if (count) CU(cudaMemcpyAsync(count, a.count, 8 * np, cudaMemcpyDeviceToHost, st));
        if (mean) CU(cudaMemcpyAsync(mean, a.mean, 8 * np * S, cudaMemcpyDeviceToHost, st));
        if (var) CU(cudaMemcpyAsync(var, a.var, 8 * np * S, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        r->d2h_bytes = 8 * np * (2 + 2 * S);
    }
    return SSA_OK;
}

extern "C" ssa_status ssa_run_trajectories(const ssa_model* m, uint64_t n_trajectories, double t_end, uint64_t seed,
                                           uint64_t stride, uint64_t capacity, uint32_t* traj, uint64_t* event,
                                           double* time, int32_t* states, uint64_t* n_points,
                                           const ssa_run_options* o, ssa_result* r)
{
    TRY(check_common(m, t_end, t_end, r));
    if (!n_points) return fail(SSA_ERR_INVALID_ARG, "n_points is null");
    *n_points = 0;
    if (n_trajectories == 0 || n_trajectories > (1ull << 23)) return fail(SSA_ERR_INVALID_ARG, "n_trajectories not in [1, 2^23]");
    if (stride == 0) return fail(SSA_ERR_INVALID_ARG, "stride must be >= 1");
    if (o && (o->path == SSA_PATH_WARP || o->path == SSA_PATH_HALFWARP))
        return fail(SSA_ERR_UNSUPPORTED, "trajectory output runs on the thread path");
    if (o && o->dump) return fail(SSA_ERR_INVALID_ARG, "ssa_run_trajectories takes no dump");
    Ctx c;
    TRY(setup_ctx(o, c));
    cudaStream_t st = c.st;
    const ssa_u64 n = n_trajectories, S = (ssa_u64)m->S, cells = 2 * S;
    ssa_run_options ro = o ? *o : ssa_run_options{};
    ro.path = SSA_PATH_THREAD;
    ro.dump = nullptr;
    ro.outputs_on_device = 0;
    DevBuf rootb;
    CU(rootb.alloc(sizeof(double) * 3 * cells, st));
    double* rb = rootb.as<double>();
    const size_t row = 16 + 4 * S;
    size_t free_b = 0, total_b = 0;
    CU(cudaMemGetInfo(&free_b, &total_b));
    ssa_u64 cap = std::min<ssa_u64>((ssa_u64)(free_b / 8) / row, 1ull << 26);
    if (const char* g = getenv("SSA_UNION_CAP0")) cap = strtoull(g, nullptr, 10);   // test hook: force the re-run
    RunInfo info, info1;
    DevBuf dcount, rk, rt, rs;
    CU(dcount.alloc(8, st));
    ssa_u64 rows = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
        rk.reset(); rt.reset(); rs.reset();
        CU(rk.alloc(8 * std::max<ssa_u64>(cap, 1), st));
        CU(rt.alloc(8 * std::max<ssa_u64>(cap, 1), st));
        CU(rs.alloc(4 * S * std::max<ssa_u64>(cap, 1), st));
        CU(cudaMemsetAsync(dcount.p, 0, 8, st));
        RecordSpec rec{2, stride, rk.as<ssa_u64>(), dcount.as<ssa_u64>(), cap, rt.as<double>(), nullptr, rs.as<int>()};
        RunInfo& ri = attempt == 0 ? info : info1;
        ri = RunInfo();
        TRY(run_range(m, 0, n, t_end, t_end, seed, &ro, c, RangeOut{rb, rb + cells, rb + 2 * cells}, ri, nullptr,
                      false, nullptr, &rec));
        TRY(fill_result(ri, r));
        CU(cudaMemcpy(&rows, dcount.p, 8, cudaMemcpyDeviceToHost));
        if (rows <= cap) {
            if (attempt == 1) info = info1;
            break;
        }
        cap = rows + ri.lanes * 32ull;   // as ssa_run_union: any schedule fits (blocks of 32 points)
    }
    if (rows > cap)
        return fail(SSA_ERR_OOM, "point record overflow (%llu rows reserved, capacity %llu)", (unsigned long long)rows,
                    (unsigned long long)cap);
    const bool on_dev = o && o->outputs_on_device;
    DevBuf dout;
    unsigned* ot = nullptr;
    ssa_u64* oe = nullptr;
    double* otm = nullptr;
    int* os = nullptr;
    if (on_dev) {
        ot = traj; oe = (ssa_u64*)event; otm = time; os = states;
    } else if (capacity) {
        CU(dout.alloc((size_t)capacity * (4 + 8 + 8 + 4 * S), st));
        char* b = (char*)dout.p;
        oe = (ssa_u64*)b; otm = (double*)(b + 8 * capacity); ot = (unsigned*)(b + 16 * capacity);
        os = (int*)(b + 20 * capacity);
    }
    Events<3> ev;
    CU(ev.create());
    cudaEvent_t e0 = ev.e[0], e1 = ev.e[1], e2 = ev.e[2];
    CU(cudaEventRecord(e0, st));
    ssa_u64 np = 0;
    int launches = 0;
    CU(ssa_points_gather(rk.as<ssa_u64>(), rt.as<double>(), rs.as<int>(), rows, (int)S, capacity, ot, oe, otm, os,
                         &np, st, &launches));
    CU(cudaEventRecord(e1, st));
    *n_points = np;
    const bool fits = np <= capacity;
    if (fits && !on_dev) {   // the output phase: device -> host
        if (time) CU(cudaMemcpyAsync(time, otm, 8 * np, cudaMemcpyDeviceToHost, st));
        if (event) CU(cudaMemcpyAsync(event, oe, 8 * np, cudaMemcpyDeviceToHost, st));
        if (traj) CU(cudaMemcpyAsync(traj, ot, 4 * np, cudaMemcpyDeviceToHost, st));
        if (states) CU(cudaMemcpyAsync(states, os, 4 * S * np, cudaMemcpyDeviceToHost, st));
        r->d2h_bytes += np * (20 + 4 * S);
    }
    CU(cudaEventRecord(e2, st));
    CU(cudaEventSynchronize(e2));
    float gms = 0.f, cms = 0.f;
    cudaEventElapsedTime(&gms, e0, e1);
    cudaEventElapsedTime(&cms, e1, e2);
    r->device_ms = info.device_ms + gms + cms;
    r->ssa_ms = info.ssa_ms;
    r->reduce_ms = gms;                        // sort + gather of the points
    r->reduce_bytes = rows * (16 + 4 * S);     // recorded point bytes
    r->dump_ms = 0.0;
    r->dump_bytes = 0;
    r->jit_ms = info.jit_ms;
    r->kernel_launches = info.launches + launches;
    if (!fits)
        return fail(SSA_ERR_INVALID_ARG, "capacity %llu < %llu output points (n_points holds the size needed)",
                    (unsigned long long)capacity, (unsigned long long)np);
    return SSA_OK;
}

extern "C" ssa_status ssa_merge_roots(const double* d_roots, int32_t n_roots, uint64_t cells,
                                      const ssa_run_options* o, ssa_result* r)
{
    if (!d_roots || n_roots < 1 || cells == 0 || !r) return fail(SSA_ERR_INVALID_ARG, "bad merge arguments");
    Ctx c;
    TRY(setup_ctx(o, c));
    // a library stream is not ordered after the caller's all-gather: wait for the device first
    if (c.own_stream) CU(cudaDeviceSynchronize());
    DevBuf rootb;
    CU(rootb.alloc(sizeof(double) * 3 * cells, c.st));
    double* rb = rootb.as<double>();
    r->events = r->near_ties = r->n_errors = r->first_error_id = 0;
    r->first_error_reaction = -1;
    r->path_used = 0;
    r->device_ms = r->ssa_ms = r->jit_ms = r->reduce_ms = r->dump_ms = 0.0;
    r->reduce_bytes = r->dump_bytes = 0;
    r->h2d_bytes = r->d2h_bytes = 0;
    r->kernel_launches = 0;
    // element (cell, rank) at d_roots[rank * 3 * cells + {0,1,2} * cells + cell]
    TRY(reduce_partials(ssa_tree_in{d_roots, d_roots + cells, d_roots + 2 * cells, 1, 3 * cells}, (ssa_u64)n_roots,
                        cells, ssa_tree_out{rb, rb + cells, rb + 2 * cells, 1, 0, 0}, c.st, &r->kernel_launches));
    return finalize_to(rb, rb + cells, rb + 2 * cells, cells, SSA_REDUCE_MEAN | SSA_REDUCE_VAR, r,
                       o && o->outputs_on_device, c.st);
}

extern "C" ssa_status ssa_model_prepare(const ssa_model* m, int32_t device, int32_t path)
{
    if (!m) return fail(SSA_ERR_INVALID_ARG, "model is null");
    ssa_run_options o{};
    o.device = device;
    Ctx c;
    TRY(setup_ctx(&o, c));
    if (path == SSA_PATH_AUTO) path = auto_path(*m);
    std::lock_guard<std::mutex> lk(m->mu);
    if (path == SSA_PATH_THREAD) {
        K1Entry* e = nullptr;
        return ensure_k1(*m, c.device, 128, default_minb(*m, 128), false, nullptr, &e, nullptr);
    }
    K2Dev* k = nullptr;
    K2Kernel* kk = nullptr;
    return ensure_k2(*m, c.device, SSA_K2_BLOCK, path == SSA_PATH_HALFWARP ? 3 : 4, false, &k, &kk, nullptr,
                     path == SSA_PATH_HALFWARP);
}

// ------------------------------------------------------------------ misc
extern "C" const char* ssa_status_string(ssa_status s)
{
    switch (s) {
    case SSA_OK: return "ok";
    case SSA_ERR_INVALID_ARG: return "invalid argument";
    case SSA_ERR_MODEL: return "invalid model";
    case SSA_ERR_NUMERIC: return "non-finite propensity";
    case SSA_ERR_OVERFLOW: return "species count overflow";
    case SSA_ERR_OOM: return "out of device memory";
    case SSA_ERR_CUDA: return "CUDA error";
    case SSA_ERR_JIT: return "NVRTC compilation failed";
    case SSA_ERR_UNSUPPORTED: return "unsupported";
    }
    return "unknown status";
}

extern "C" const char* ssa_last_error(void) { return g_err.c_str(); }
extern "C" int32_t ssa_abi_version(void) { return 1; }

// Test/diagnostic hooks (not part of the stable ABI): the generated K1
// source for a model, and compiling it without a device (NVRTC only).
// The model's measured K1 hot set: the number of hot reactions written to out
// (at most cap), or -1 if no profiling run has completed yet.
extern "C" int32_t ssa_debug_model_hot(const ssa_model* m, int32_t* out, int32_t cap)
{
    if (!m) return -1;
    std::lock_guard<std::mutex> lk(m->mu);
    if (!m->hot_known) return -1;
    const int32_t n = (int32_t)m->hot.size();
    for (int32_t i = 0; i < n && i < cap; ++i) out[i] = m->hot[(size_t)i];
    return n;
}

extern "C" const char* ssa_debug_k1_source(const ssa_model* m, int32_t block, int32_t minb, int32_t dump, int64_t seed)
{
    static thread_local std::string s;
    if (!m) return "";
    // flags: bit 0 dump, bits 1-2 record mode, bit 3 the sweep variant (the model's own rates as one point)
    PoolLayout L;
    if (dump & 8) L = make_pool(*m, 1, nullptr, nullptr);
    s = k1_full_source(*m, block, minb, (dump & 1) != 0, (dump & 8) ? &L : nullptr, seed, (dump >> 1) & 3);
    return s.c_str();
}

extern "C" ssa_status ssa_debug_k1_compile(const ssa_model* m, int32_t block, int32_t minb, int32_t dump, char* log,
                                           uint64_t log_cap, uint64_t* cubin_bytes)
{
    if (!m) return fail(SSA_ERR_INVALID_ARG, "model is null");
    std::vector<char> cubin;
    std::string lg;
    ssa_status st = nvrtc_compile(k1_full_source(*m, block, minb, dump != 0, nullptr), cubin, lg);
    if (log && log_cap) {
        std::string all = (st == SSA_OK) ? lg : g_err;
        strncpy(log, all.c_str(), (size_t)log_cap - 1);
        log[log_cap - 1] = 0;
    }
    if (cubin_bytes) *cubin_bytes = cubin.size();
    return st;
}

extern "C" const char* ssa_debug_k2_source(const ssa_model* m, int32_t block, int32_t dump)
{
    static thread_local std::string s;
    if (!m) return "";
    // dump: bit 0 = the dump variant, bit 1 = two trajectories per warp (HALFWARP)
    const bool half = (dump & 2) != 0;
    s = k2_full_source(*m, std::max(1, (m->R + (half ? 15 : 31)) / (half ? 16 : 32)), block, 1, (dump & 1) != 0, half);
    return s.c_str();
}

extern "C" ssa_status ssa_debug_k2_compile(const ssa_model* m, int32_t block, int32_t dump, char* log, uint64_t log_cap,
                                           uint64_t* cubin_bytes)
{
    if (!m) return fail(SSA_ERR_INVALID_ARG, "model is null");
    std::vector<char> cubin;
    std::string lg;
    // dump: bit 0 = the dump variant, bit 1 = HALFWARP, bits 4-7 = the residency target (0: 1)
    const bool half = (dump & 2) != 0;
    const int minb = std::max(1, (dump >> 4) & 15);
    ssa_status st = nvrtc_compile(
        k2_full_source(*m, std::max(1, (m->R + (half ? 15 : 31)) / (half ? 16 : 32)), block, minb, (dump & 1) != 0, half),
        cubin, lg);
    if (log && log_cap) {
        std::string all = (st == SSA_OK) ? lg : g_err;
        strncpy(log, all.c_str(), (size_t)log_cap - 1);
        log[log_cap - 1] = 0;
    }
    if (cubin_bytes) *cubin_bytes = cubin.size();
    return st;
}

