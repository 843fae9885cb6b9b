// k2_warp.cuh -- K2: one trajectory per warp, model-specialised (sm_100a).
//
// The warp path of north_star (a) for networks with hundreds of reactions.
// Compiled by NVRTC at run time after ssa_device.cuh and a generated section
// (runtime.cu: gen_k2_model) that defines SSA_S, SSA_R, SSA_P = ceil(R/32),
// SSA_K2_BLOCK, SSA_K2_MINB (residency target), SSA_K2_DUMP, SSA_HAS_M3 (a
// reactant with coefficient 3), SSA_HAS_GATES (gated propensities, NEXT 3),
// SSA_NU_MAX and SSA_DEP_MAX (longest net-change
// and dependency lists).  The model
// tables (packed reactant words, rates, modifier coefficients, x0, net
// changes, and per-reaction dependency lists) come from the run's device
// image (ssa_k2_params) and are staged in shared memory once per block.
//
// Layout and order (DESIGN.md §2 "warp32", R13): lane l owns the P
// contiguous reactions j = l*P + q; their propensities live in shared memory
// a[q][lane] (conflict-free) so that any lane can recompute any reaction.
// Per event:
//   a2  Philox amortised: every 32 events lane l draws the block of event e+l
//       and broadcasts E, u2 with __shfl_sync (same values: counter-based).
//   a4  L_l = sequential sum of the lane's P propensities, inclusive
//       Hillis-Steele scan over lanes (offsets 1..16), a0 = v_31.
//   a7  every lane speculatively runs its part of the definition -- p =
//       v_{l-1}, p += a_j over its reactions, first q with p > r -- without
//       divergence; lane* = ffs(ballot(v_l > r)) picks the answer.  The
//       rounding fallback (no p > r inside lane*) is a warp-uniform rare path.
//   a8  lane t < |nu_j| applies the t-th net change of j in shared memory.
//   a3  lane t recomputes the t-th reaction of dep(j) -- the reactions whose
//       propensity reads a species that j changes (a precomputed list) --
//       bit-identical to a full recompute since a_j is a function of x.

// ssa_k2_params is defined in ssa_device.cuh (shared with the host runtime).

struct k2_rx {
    ssa_u64 pk;      // n_reac | 3 x (14-bit species, 2-bit coef) | 14-bit modifier species
    double rate;
    double modc;
    ssa_u64 gw;      // gates: count (3 bits) | 4 x (14-bit species, 1-bit kind: 0 [x>0], 1 [x==0])
};

// NEXT 3: a closed gate makes the propensity exactly 0 (R33)
static __device__ __forceinline__ double k2_gated(double a, ssa_u64 gw, const double* __restrict__ x)
{
#if SSA_HAS_GATES
    const int ng = (int)(gw & 7ull);
    bool open = true;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        const ssa_u64 w = gw >> (3 + 15 * g);
        const double xg = x[(int)(w & 0x3FFF)];
        const bool ok = ((w >> 14) & 1ull) ? (xg == 0.0) : (xg > 0.0);
        open = open && (g >= ng || ok);
    }
    return open ? a : 0.0;
#else
    (void)gw; (void)x;
    return a;
#endif
}

// C(x, m) for m in {1, 2, 3}, exact for counts < 2^26.
static __device__ __forceinline__ double k2_factor(double x, int m)
{
    if (m == 1) return x;
    const double x1 = __dmul_rn(x, __dadd_rn(x, -1.0));
    if (m == 2) return __dmul_rn(x1, 0.5);
    return __ddiv_rn(__dmul_rn(x1, __dadd_rn(x, -2.0)), 6.0);
}

#if !SSA_HAS_M3
// Decoded reaction descriptor (built in shared memory from the packed tables
// at block start): at most two reactant terms (no coefficient 3 in this
// model), absent terms/modifier encoded so that they contribute exact
// neutral operands.
struct k2_rxd {
    double rate;     // k
    double modc;     // d, 0.0 when the reaction has no modifier
    int sab;         // reactant species a | b << 16 (absent: 0)
    int sms;         // modifier species (none: 0) | propensity slot (q*32 + l) << 16
    int mab;         // coefficient of a | of b << 8 (0 = absent factor)
    int pad;
    ssa_u64 gw;      // gate word (as k2_rx)
};

// select without a branch (selp on the 64-bit value; ptxas would otherwise
// turn the ternaries of the factor into divergent branches)
static __device__ __forceinline__ double k2_sel(bool p, double a, double b)
{
    double r;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %3, 0;\n\tselp.f64 %0, %1, %2, q;\n\t}"
        : "=d"(r) : "d"(a), "d"(b), "r"((int)p));
    return r;
}

static __device__ __forceinline__ double k2_factor_bf(double x, int m)
{
    const double x2 = __dmul_rn(__dmul_rn(x, __dadd_rn(x, -1.0)), 0.5);   // C(x,2)
    return k2_sel(m == 2, x2, k2_sel(m == 1, x, 1.0));
}

// Branch-free form (the 32 lanes evaluate different reactions, so branches
// would diverge): absent reactant terms contribute the exact factor 1.0 and
// an absent modifier the exact term +0 (0 * x), so every case performs the
// definition's operations: h = f1 * f2, k^ = max(0, k + d x_m), a = k^ * h --
// up to the sign of a zero propensity (a -0 rate), which changes no sum,
// comparison or selection.
static __device__ __forceinline__ double k2_propensity_d(const k2_rxd& d, const double* __restrict__ x)
{
    const double f1 = k2_factor_bf(x[d.sab & 0xFFFF], d.mab & 0xFF);
    const double f2 = k2_factor_bf(x[(unsigned)d.sab >> 16], d.mab >> 8);
    const double h = __dmul_rn(f1, f2);
#if SSA_HAS_MODS
    double k = __dadd_rn(d.rate, __dmul_rn(d.modc, x[d.sms & 0xFFFF]));
    k = (k < 0.0) ? 0.0 : k;
#else
    const double k = d.rate;   // no modifier in the model: k + 0*x = k exactly
#endif
    return k2_gated(__dmul_rn(k, h), d.gw, x);
}
#endif

// General form (any model, e.g. with coefficient-3 reactants).
static __device__ __forceinline__ double k2_propensity(const k2_rx& q, const double* __restrict__ x)
{
    const ssa_u64 pk = q.pk;
    const int n = (int)(pk & 3ull);
    double h = 1.0;
    if (n >= 1) h = k2_factor(x[(int)((pk >> 2) & 0x3FFF)], (int)((pk >> 16) & 3));
    if (n >= 2) h = __dmul_rn(h, k2_factor(x[(int)((pk >> 18) & 0x3FFF)], (int)((pk >> 32) & 3)));
    if (n >= 3) h = __dmul_rn(h, k2_factor(x[(int)((pk >> 34) & 0x3FFF)], (int)((pk >> 48) & 3)));
    double k = q.rate;
    const int ms = (int)(pk >> 50);
    if (ms != 0x3FFF) {
        k = __dadd_rn(k, __dmul_rn(q.modc, x[ms]));
        k = (k < 0.0) ? 0.0 : k;
    }
    return k2_gated((n == 0) ? k : __dmul_rn(k, h), q.gw, x);
}

#define SSA_K2_WARPS (SSA_K2_BLOCK / 32)

#if !SSA_K2_HALF
extern "C" __global__ void __launch_bounds__(SSA_K2_BLOCK, SSA_K2_MINB) ssa_k2(const ssa_k2_params P)
{
    extern __shared__ __align__(16) unsigned char k2_smem_raw[];
    // lane index and the warp's state address computed once and kept opaque (as
    // in the half-warp kernel: no S2R re-derivation inside the event loop)
    int lane_ = threadIdx.x & 31;
    asm volatile("" : "+r"(lane_));
    const int lane = lane_;
    const int warp = threadIdx.x >> 5;
    const unsigned FULL = 0xffffffffu;
    // shared: rx[R] | x0[S] | per warp (x[S] | a[P][32]) | nu_off[R+1] | nu_ent | dep_off[R+1] | dep_ent
    // the packed table rx is needed only by the general evaluator (coefficient-3 models)
    k2_rx* rx = (k2_rx*)k2_smem_raw;
    double* x0 = (double*)(rx + (SSA_HAS_M3 ? SSA_R : 0));
    double* x = x0 + SSA_S + (size_t)warp * (SSA_S + 32 * SSA_P);
    {
        unsigned xs = (unsigned)__cvta_generic_to_shared(x);
        asm volatile("" : "+r"(xs));
        x = (double*)__cvta_shared_to_generic(xs);
    }
    double* a = x + SSA_S;                                     // a[q*32 + l]: reaction l*P + q
    int* nu_off = (int*)(x0 + SSA_S + (size_t)SSA_K2_WARPS * (SSA_S + 32 * SSA_P));
    int* nu_ent = nu_off + (SSA_R + 1);
    int* dep_off = nu_ent + P.n_ent;
    int* dep_ent = dep_off + (SSA_R + 1);
#if !SSA_HAS_M3
    k2_rxd* rxd = (k2_rxd*)(k2_smem_raw + P.rxd_offset);   // 16-byte aligned, after dep_ent
#endif
#if SSA_HAS_M3
    for (int i = threadIdx.x; i < SSA_R; i += SSA_K2_BLOCK) {
        k2_rx q;
        q.pk = P.pk[i]; q.rate = P.rate[i]; q.modc = P.modc[i]; q.gw = P.gw[i];
        rx[i] = q;
    }
#else
    (void)rx;
#endif
    for (int i = threadIdx.x; i < SSA_S; i += SSA_K2_BLOCK) x0[i] = P.x0[i];
    for (int i = threadIdx.x; i <= SSA_R; i += SSA_K2_BLOCK) { nu_off[i] = P.nu_off[i]; dep_off[i] = P.dep_off[i]; }
    for (int i = threadIdx.x; i < P.n_ent; i += SSA_K2_BLOCK) nu_ent[i] = P.nu_ent[i];
    for (int i = threadIdx.x; i < P.n_dep; i += SSA_K2_BLOCK) dep_ent[i] = P.dep_ent[i];
#if !SSA_HAS_M3
    for (int i = threadIdx.x; i < SSA_R; i += SSA_K2_BLOCK) {
        const ssa_u64 pk = P.pk[i];
        const int n = (int)(pk & 3ull);
        const int ms = (int)(pk >> 50);
        k2_rxd d;
        d.rate = P.rate[i];
        d.modc = (ms != 0x3FFF) ? P.modc[i] : 0.0;
        const int sa = n >= 1 ? (int)((pk >> 2) & 0x3FFF) : 0, sb = n >= 2 ? (int)((pk >> 18) & 0x3FFF) : 0;
        const int ma = n >= 1 ? (int)((pk >> 16) & 3) : 0, mb = n >= 2 ? (int)((pk >> 32) & 3) : 0;
        const int slot = (i % SSA_P) * 32 + i / SSA_P;
        d.sab = sa | (sb << 16);
        d.sms = (ms != 0x3FFF ? ms : 0) | (slot << 16);
        d.mab = ma | (mb << 8);
        d.pad = 0;
        d.gw = P.gw[i];
        rxd[i] = d;
    }
#endif
    __syncthreads();

    const double INF = __longlong_as_double(0x7FF0000000000000ll);
    const double dt = P.dt;
    const long long K = P.K;
    const ssa_u64 G = (ssa_u64)K + 1;
    ssa_u64 my_events = 0, my_ties = 0;

    for (;;) {
        // a1: the warp takes the next trajectory id
        ssa_u64 rel = 0;
        if (lane == 0) rel = atomicAdd(P.work, 1ull);
        rel = __shfl_sync(FULL, rel, 0);
        if (rel >= P.n_ids) break;
        const ssa_u64 id = P.id_begin + rel;
#if SSA_K2_DUMP
        const long long slot = P.n_dump ? ssa_dump_slot(P.dump_ids, P.n_dump, id) : -1ll;
#endif
        for (int s = lane; s < SSA_S; s += 32) x[s] = x0[s];
        __syncwarp();
        // a3 at the initial state: every propensity of this lane's block
#pragma unroll
        for (int q = 0; q < SSA_P; ++q) {
            const int j = lane * SSA_P + q;
#if SSA_HAS_M3
            a[q * 32 + lane] = (j < SSA_R) ? k2_propensity(rx[j], x) : 0.0;
#else
            a[q * 32 + lane] = (j < SSA_R) ? k2_propensity_d(rxd[j], x) : 0.0;
#endif
        }
        __syncwarp();

        double t = 0.0, s_next = 0.0;
        ssa_u64 e = 0, ties = 0;
#if SSA_K2_DUMP
        ssa_u64 hash = SSA_FNV_OFFSET;
#endif
        long long k = 0;
        int status = 0, absorbed = 0, err_r = -1;
        const ssa_u32 idlo = (ssa_u32)id, idhi = (ssa_u32)(id >> 32);
        double Ec = 0.0, U2c = 0.0;

        for (;;) {
            // a2, amortised: lane l draws event e0 + l for the next 32 events
            if ((e & 31ull) == 0) {
                const ssa_u64 ee = e + (ssa_u64)lane;
                const ssa_philox_out o = ssa_philox4x32_10((ssa_u32)ee, (ssa_u32)(ee >> 32), idlo, idhi,
                                                           P.key0, P.key1);
                Ec = -ssa_plog(ssa_u53(o.o1, o.o0), c_plog);
                U2c = ssa_u53(o.o3, o.o2);
            }
            // a4: the lane's propensities (kept for the selection), lane sum, warp scan
            double aq[SSA_P];
            double L = 0.0;
#pragma unroll
            for (int q = 0; q < SSA_P; ++q) {
                aq[q] = a[q * 32 + lane];
                L = __dadd_rn(L, aq[q]);       // from 0.0, as the definition (zero signs included)
            }
            double v = L;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                v = ssa_scan_step(v, o, 0);          // width 32
            }
            const double a0 = __shfl_sync(FULL, v, 31);
            // a5
            const int src = (int)(e & 31ull);
            const double E = __shfl_sync(FULL, Ec, src);
            const double u2 = __shfl_sync(FULL, U2c, src);
            const unsigned a0hi = (unsigned)__double2hiint(a0);
            const bool fast = a0hi - (123u << 20) < ((1923u - 123u) << 20);   // a0 in [2^-900, 2^901)
            double tn = __dadd_rn(t, ssa_ddiv_inrange(E, a0));
            if (!fast || tn > s_next) {           // warp-uniform rare path
                if (!fast) {
                    if (a0 > 0.0 && a0 < INF) {
                        tn = __dadd_rn(t, __ddiv_rn(E, a0));
                    } else if (a0 == 0.0) {
                        tn = INF;
                        absorbed = 1;
                    } else {
                        status = 1;
                        int bad = SSA_R;   // first reaction with a non-finite propensity
#pragma unroll
                        for (int q = SSA_P - 1; q >= 0; --q)
                            if (lane * SSA_P + q < SSA_R && !(fabs(aq[q]) < INF)) bad = lane * SSA_P + q;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) bad = min(bad, __shfl_xor_sync(FULL, bad, o));
                        err_r = bad < SSA_R ? bad : -1;
                        break;
                    }
                }
                // a6: grid alignment (warp-uniform)
                if (tn > s_next) {
                    do {
                        const double tol = __dmul_rn(1e-9, s_next);
                        const bool near = (tn < INF && fabs(__dadd_rn(tn, -s_next)) <= tol) ||
                                          (e > 0 && fabs(__dadd_rn(t, -s_next)) <= tol);
                        ties += near ? 1 : 0;
                        int ovf = 0;
                        for (int s = lane; s < SSA_S; s += 32) {
                            const double xv = x[s];
                            ovf |= (xv > 2147483647.0) ? 1 : 0;
                            P.staging[rel * P.stride + (ssa_u64)k * SSA_S + s] = (int)xv;   // trajectory-major row
#if SSA_K2_DUMP
                            if (slot >= 0) P.dump_states[((ssa_u64)slot * G + (ssa_u64)k) * SSA_S + s] = (int)xv;
#endif
                        }
                        if (__any_sync(FULL, ovf)) status = 2;
#if SSA_K2_DUMP
                        if (slot >= 0 && lane == 0) {
                            P.dump_e[(ssa_u64)slot * G + (ssa_u64)k] = e;
                            P.dump_t[(ssa_u64)slot * G + (ssa_u64)k] = (e > 0) ? t : 0.0;
                        }
#endif
                        ++k;
                        s_next = (k <= K) ? __dmul_rn((double)k, dt) : INF;
                    } while (tn > s_next);
                    if (k > K) break;
                }
            }
            // a7, speculatively in every lane: p = v_{l-1}, p += a_j in order,
            // first q with p > r; lane* = first lane with v_l > r
            const double r = __dmul_rn(u2, a0);
            const double vprev = __shfl_up_sync(FULL, v, 1);
            double p = (lane > 0) ? vprev : 0.0;
            // p is nondecreasing over the lane's reactions: the first q with
            // p > r is P - #{q : p_q > r} (none: -1)
            int over = 0;
#pragma unroll
            for (int q = 0; q < SSA_P; ++q) {
                p = __dadd_rn(p, aq[q]);
                asm("{\n\t.reg .pred p;\n\tsetp.gt.f64 p, %1, %2;\n\t@p add.s32 %0, %0, 1;\n\t}"
                    : "+r"(over) : "d"(p), "d"(r));
            }
            const int jl = over ? SSA_P - over : -1;
            const int ls = __ffs(__ballot_sync(FULL, v > r)) - 1;
            int jq = __shfl_sync(FULL, jl, ls);
            int j;
            if (jq >= 0) {
                j = ls * SSA_P + jq;
            } else {
                // rounding fallback (rare): the largest j <= lane*'s last index with a_j > 0
                int lp = -1;
#pragma unroll
                for (int q = 0; q < SSA_P; ++q)
                    if (aq[q] > 0.0) lp = lane * SSA_P + q;
                const unsigned m2 = __ballot_sync(FULL, lp >= 0 && lane <= ls);
                j = __shfl_sync(FULL, lp, 31 - __clz(m2));
            }
            // a8: state update, lane t takes the t-th net change of j
            const int nb = nu_off[j], ne = nu_off[j + 1];
#if SSA_NU_MAX <= 32
            if (nb + lane < ne) {
                const int q = nb + lane;
#else
            for (int q = nb + lane; q < ne; q += 32) {
#endif
                const int ent = nu_ent[q];
                const int sp = ent & 0xFFFF;
                x[sp] = __dadd_rn(x[sp], (double)(ent >> 16));   // arithmetic shift: signed delta
            }
            __syncwarp();
            // a3: lane t recomputes the t-th reaction of dep(j)
            const int db = dep_off[j], de = dep_off[j + 1];
#if SSA_DEP_MAX <= 32
            if (db + lane < de) {
                const int q = db + lane;
#else
            for (int q = db + lane; q < de; q += 32) {
#endif
                const int jj = dep_ent[q];
#if !SSA_HAS_M3
                const k2_rxd d = rxd[jj];
                a[(unsigned)d.sms >> 16] = k2_propensity_d(d, x);
#else
                const int l = jj / SSA_P, qq = jj - l * SSA_P;
                a[qq * 32 + l] = k2_propensity(rx[jj], x);
#endif
            }
            __syncwarp();
            t = tn;
            ++e;
#if SSA_K2_DUMP
            hash = (hash ^ (ssa_u64)j) * SSA_FNV_PRIME;
#endif
        }
        __syncwarp();
        if (lane == 0) {
            my_events += e;
            my_ties += ties;
#if SSA_K2_DUMP
            if (slot >= 0) {
                ssa_dev_summary sm;
                sm.events = e; sm.hash = hash; sm.t_last = t; sm.near_ties = ties;
                sm.absorbed = absorbed; sm.status = status == 1 ? 3 : (status == 2 ? 4 : 0);
                sm.err_reaction = err_r; sm.pad = 0;
                P.dump_sum[slot] = sm;
            }
#endif
            if (status) {
                const ssa_u64 code = status == 1 ? SSA_DEV_ERR_NUMERIC : SSA_DEV_ERR_OVERFLOW;
                atomicAdd(&P.stats->n_errors, 1ull);
                atomicOr(&P.stats->err_code, code);
                const ssa_u64 packed = (id << 24) | (code << 20) | ((ssa_u64)(err_r + 1) & 0xFFFFFull);
                atomicMin(&P.stats->first_err_id, packed);
            }
        }
    }
    if (lane == 0) {
        atomicAdd(&P.stats->events, my_events);
        if (my_ties) atomicAdd(&P.stats->near_ties, my_ties);
    }
}
#endif  // !SSA_K2_HALF
