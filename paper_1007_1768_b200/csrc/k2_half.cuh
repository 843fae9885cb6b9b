// k2_half.cuh -- K2 with two trajectories per warp: a half warp (L = 16 lanes)
// per trajectory (sm_100a, NVRTC).  Appended after k2_warp.cuh (whose
// helpers -- k2_rx, k2_rxd, the propensity evaluators -- it uses) when the
// generated section defines SSA_K2_HALF = 1.
//
// Order "warp16s" (R13, R34; oracle mode 3): lane l of the half owns
// the P = ceil(R/16) contiguous reactions l*P + q; lane sums from 0.0 in q
// order, then an inclusive Hillis-Steele scan over the 16 lanes (offsets 1, 2,
// 4, 8; the shuffles are segmented with width 16), a0 = v_15, lane* = min{l :
// v_l > r}.  The step inside lane* is a second 16-position Hillis-Steele scan
// over lane*'s propensities, one per lane of the half (lane q reads lane*'s
// q-th reaction), p_q = v_{lane*-1} + s_q, j* = lane*'s first q with p_q > r --
// a ballot instead of every lane re-summing its P propensities sequentially.
// Per warp the scans, the broadcasts, the division and the update/recompute
// passes serve two events.
//
// Shared memory per half (16-byte aligned window): the propensities a[l*18 + q]
// (reaction l*P + q; row stride 18 doubles: the lane sums read their row two
// doubles at a time with 2 wavefronts per half, the lane* scan reads one row
// with 1) and then x[S].  Per block: the model's per-reaction record {nu begin,
// nu end, dep begin, dep end} (one 16-byte load once j* is known) and the
// dependency entries pre-resolved to (reactant species and coefficients,
// propensity slot, reaction), so the recompute of dep(j*) reads x and the rate
// directly.  The shared-memory addresses are computed once and kept opaque:
// otherwise the compiler re-derives the shared window base (S2R of the CTA id
// + LEA) inside the event loop.
//
// Random numbers: lane l of a half draws (E, u2) of event base + l into the half's
// 16-entry buffer in shared memory; every lane reads event e's pair with one
// broadcast load.  Both halves refill at the same iteration (when either has used
// its 16): they then stay in step, so the Philox + plog pass -- a divergent
// branch when only one half takes it -- runs once per 16 iterations, not twice.
// A half's early refill re-draws the same counter-based values.
//
// Both halves execute the common path in lockstep (the shuffles are
// full-warp); rare paths (grid crossing, end of a trajectory, refill, the
// rounding fallback) run per half with half-warp masks.  A half with no work
// left keeps executing the common path on a frozen, absorbed state and
// records nothing.

#if SSA_K2_HALF
#define SSA_HL 16
#define SSA_AR 18                            // row stride of a[] (doubles)
#define SSA_XW ((SSA_S + 2) & ~1)            // x[S] and the constant x_S = 1.0, rounded up to even
#define SSA_AWIN (SSA_HL * SSA_AR + SSA_XW + 32)   // per-half window (doubles, even): a | x | (E, u2)[16]

#if SSA_K2_FE
// Fast evaluator (runtime.cu k2_fe_ok): a = k * ((x_a * (x_b - d)) * s) with (d, s) = (0, 1) or,
// for a reactant of coefficient 2 (b = a), (1, 1/2); a missing factor reads x_S = 1.0.  The
// operations are those of k2_propensity_d for the same reaction: f1 * f2 with f = x or C(x, 2) =
// (x (x - 1)) * 0.5 and the absent factor 1.0, then k * h -- so the bits are the same.
// w: sa | sb << 16 | d << 41 (| slot, reaction in a dependency entry)
static __device__ __forceinline__ double k2h_fe(ssa_u64 w, double rate, const double* __restrict__ x)
{
    const unsigned lo = (unsigned)w, hi = (unsigned)(w >> 32);
    const double xa = x[lo & 0xFFFFu], xb = x[lo >> 16];
    const unsigned f = (hi >> 9) & 1u;
    const double nd = __hiloint2double(f ? (int)0xBFF00000 : (int)0x80000000, 0);   // -1.0 or -0.0
    const double sc = __hiloint2double((int)(0x3FF00000u - (f << 20)), 0);           // 0.5 or 1.0
    return __dmul_rn(rate, __dmul_rn(__dmul_rn(xa, __dadd_rn(xb, nd)), sc));
}
#elif !SSA_HAS_M3
// dependency entry: sa | sb << 14 | ma << 28 | mb << 30 | slot << 32 | reaction << 48
static __device__ __forceinline__ double k2h_propensity(ssa_u64 de, const k2_rxd* __restrict__ rxd,
                                                        const double* __restrict__ x)
{
    const unsigned lo = (unsigned)de;
    const int rxi = (int)(de >> 48);
    const double f1 = k2_factor_bf(x[lo & 0x3FFFu], (int)((lo >> 28) & 3u));
    const double f2 = k2_factor_bf(x[(lo >> 14) & 0x3FFFu], (int)(lo >> 30));
    const double h = __dmul_rn(f1, f2);
#if SSA_HAS_MODS
    const k2_rxd& d = rxd[rxi];
    double k = __dadd_rn(d.rate, __dmul_rn(d.modc, x[d.sms & 0xFFFF]));
    k = (k < 0.0) ? 0.0 : k;
    return k2_gated(__dmul_rn(k, h), d.gw, x);
#else
    return k2_gated(__dmul_rn(rxd[rxi].rate, h), rxd[rxi].gw, x);
#endif
}
#endif

// one inclusive-scan step over the half with a precomputed mask (hi word 0x3ff00000 where the
// source lane exists, 0 where it does not): v <- fma(y, m, v), fma(y, 1, v) = fl(y + v)
static __device__ __forceinline__ double ssa_scan_step_m(double v, int o, unsigned mh)
{
    asm("{\n\t.reg .b32 lo, hi, z;\n\t.reg .f64 y, m;\n\t"
        "mov.b64 {lo, hi}, %0;\n\t"
        "shfl.sync.up.b32 lo, lo, %1, 0x1000, -1;\n\t"
        "shfl.sync.up.b32 hi, hi, %1, 0x1000, -1;\n\t"
        "mov.b64 y, {lo, hi};\n\t"
        "mov.b32 z, 0;\n\t"
        "mov.b64 m, {z, %2};\n\t"
        "fma.rn.f64 %0, y, m, %0;\n\t}"
        : "+d"(v) : "r"(o), "r"(mh));
    return v;
}

template <class T> static __device__ __forceinline__ T* k2h_opaque(T* p)
{
    unsigned s = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("" : "+r"(s));
    return (T*)__cvta_shared_to_generic(s);
}

extern "C" __global__ void __launch_bounds__(SSA_K2_BLOCK, SSA_K2_MINB) ssa_k2(const ssa_k2_params P)
{
    extern __shared__ __align__(16) unsigned char k2_smem_raw[];
    int lane_ = threadIdx.x & 31;
    asm volatile("" : "+r"(lane_));
    const int lane = lane_;
    const int warp = threadIdx.x >> 5;
    const int h = lane >> 4;                 // which half (trajectory slot) of the warp
    const int hl = lane & 15;                // lane within the half
    const unsigned FULL = 0xffffffffu;
    const unsigned HALF = 0xFFFFu << (16 * h);
    // shared: rx[R] | x0[S] | (16-aligned) per warp, per half (a[16*18] | x[S]) | rec[R] | nu_ent | dent | rxd
    // the packed table rx is needed only by the general evaluator (coefficient-3 models)
    k2_rx* rx = (k2_rx*)k2_smem_raw;
    double* x0 = (double*)(rx + (SSA_HAS_M3 ? SSA_R : 0));
    double* win0 = (double*)(((unsigned long long)(x0 + SSA_S) + 15ull) & ~15ull);
    double* a = k2h_opaque(win0 + ((size_t)warp * 2 + h) * SSA_AWIN);   // a[l*18 + q]: reaction l*P + q
    double* x = k2h_opaque(win0 + ((size_t)warp * 2 + h) * SSA_AWIN + SSA_HL * SSA_AR);
    double2* eub = k2h_opaque((double2*)(win0 + ((size_t)warp * 2 + h) * SSA_AWIN + SSA_HL * SSA_AR + SSA_XW));
    const int4* rec = k2h_opaque((const int4*)(k2_smem_raw + P.rec_offset));   // {nu b, nu e, dep b, dep e}
    const int* nu_ent = k2h_opaque((const int*)(k2_smem_raw + P.rec_offset + 16 * SSA_R));
    const ssa_u64* dent = k2h_opaque((const ssa_u64*)(k2_smem_raw + P.dent_offset));
#if !SSA_HAS_M3
    const k2_rxd* rxd = k2h_opaque((const k2_rxd*)(k2_smem_raw + P.rxd_offset));
#endif
#if SSA_K2_FE
    const double* rt = k2h_opaque((const double*)(k2_smem_raw + P.rxd_offset));     // rate[R]
    const ssa_u64* __restrict__ rfe = P.rfe;                                          // (start only)
#endif
    {
        int4* rec_w = (int4*)(k2_smem_raw + P.rec_offset);
        int* nu_w = (int*)(k2_smem_raw + P.rec_offset + 16 * SSA_R);
        ssa_u64* dent_w = (ssa_u64*)(k2_smem_raw + P.dent_offset);
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
        for (int i = threadIdx.x; i < SSA_R; i += SSA_K2_BLOCK) rec_w[i] = P.rec[i];
        for (int i = threadIdx.x; i < P.n_ent; i += SSA_K2_BLOCK) nu_w[i] = P.nu_ent[i];
        for (int i = threadIdx.x; i < P.n_dep; i += SSA_K2_BLOCK) dent_w[i] = P.dent[i];
#if SSA_K2_FE
        for (int i = threadIdx.x; i < SSA_R; i += SSA_K2_BLOCK) {
            ((double*)(k2_smem_raw + P.rxd_offset))[i] = P.rate[i];
        }
#elif !SSA_HAS_M3
        k2_rxd* rxd_w = (k2_rxd*)(k2_smem_raw + P.rxd_offset);
        for (int i = threadIdx.x; i < SSA_R; i += SSA_K2_BLOCK) {
            const ssa_u64 pk = P.pk[i];
            const int n = (int)(pk & 3ull);
            const int ms = (int)(pk >> 50);
            k2_rxd d;
            d.rate = P.rate[i];
            d.modc = (ms != 0x3FFF) ? P.modc[i] : 0.0;
            const int sa = n >= 1 ? (int)((pk >> 2) & 0x3FFF) : 0, sb = n >= 2 ? (int)((pk >> 18) & 0x3FFF) : 0;
            const int ma = n >= 1 ? (int)((pk >> 16) & 3) : 0, mb = n >= 2 ? (int)((pk >> 32) & 3) : 0;
            d.sab = sa | (sb << 16);
            d.sms = (ms != 0x3FFF ? ms : 0);
            d.mab = ma | (mb << 8);
            d.pad = 0;
            d.gw = P.gw[i];
            rxd_w[i] = d;
        }
#endif
        // the padding entries of every propensity row stay 0
        for (int i = threadIdx.x; i < SSA_K2_WARPS * 2 * SSA_HL * SSA_AR; i += SSA_K2_BLOCK) {
            const int w = i / (SSA_HL * SSA_AR), o = i - w * (SSA_HL * SSA_AR);
            win0[(size_t)w * SSA_AWIN + o] = 0.0;
        }
    }
    __syncthreads();

    const double INF = __longlong_as_double(0x7FF0000000000000ll);
    const double dt = P.dt;
    const long long K = P.K;
    const ssa_u64 G = (ssa_u64)K + 1;
    ssa_u64 my_events = 0, my_ties = 0;
    // scan masks: the source lane hl - o exists
    const unsigned mk1 = hl >= 1 ? 0x3ff00000u : 0u, mk2 = hl >= 2 ? 0x3ff00000u : 0u;
    const unsigned mk4 = hl >= 4 ? 0x3ff00000u : 0u, mk8 = hl >= 8 ? 0x3ff00000u : 0u;
    const bool in_row = hl < SSA_P;          // this lane holds a position of lane*'s row

    // per-half trajectory state (uniform within the half)
    bool live = false;
    ssa_u64 rel = 0, id = 0, e = 0, ties = 0, ebase = 0;
    double t = 0.0, s_next = 0.0;
    long long k = 0;
    int status = 0, absorbed = 0, err_r = -1;
#if SSA_K2_DUMP
    long long slot = -1;
    ssa_u64 hash = SSA_FNV_OFFSET;
#endif
    bool need_rng = true;                    // this half's buffer is used up (or a new trajectory)

    // a1 for this half: take the next id and initialise (half-warp collective)
    auto start = [&]() {
        ssa_u64 r0 = 0;
        if (hl == 0) r0 = atomicAdd(P.work, 1ull);
        rel = __shfl_sync(HALF, r0, 0, SSA_HL);
        live = rel < P.n_ids;
        id = P.id_begin + rel;
#if SSA_K2_DUMP
        slot = (live && P.n_dump) ? ssa_dump_slot(P.dump_ids, P.n_dump, id) : -1ll;
        hash = SSA_FNV_OFFSET;
#endif
        for (int s = hl; s < SSA_S; s += SSA_HL) x[s] = x0[s];
        if (hl == 0) x[SSA_S] = 1.0;                 // the fast evaluator's missing factor
        __syncwarp(HALF);
#pragma unroll
        for (int q = 0; q < SSA_P; ++q) {
            const int j = hl * SSA_P + q;
#if SSA_HAS_M3
            const double aj = (live && j < SSA_R) ? k2_propensity(rx[j], x) : 0.0;
#elif SSA_K2_FE
            const double aj = (live && j < SSA_R) ? k2h_fe(rfe[j], rt[j], x) : 0.0;
#else
            const double aj = (live && j < SSA_R) ? k2_propensity_d(rxd[j], x) : 0.0;
#endif
            a[hl * SSA_AR + q] = aj;
        }
        __syncwarp(HALF);
        t = 0.0; s_next = 0.0; e = 0; ties = 0; k = 0;
        status = 0; absorbed = 0; err_r = -1;
        need_rng = true;
    };
    start();

    while (__any_sync(FULL, live)) {
        // a2: both halves refill their 16-event buffers together when either needs it
        if (__any_sync(FULL, need_rng && live)) {
            ebase = e;
            const ssa_u64 ee = e + (ssa_u64)hl;
            const ssa_philox_out o = ssa_philox4x32_10((ssa_u32)ee, (ssa_u32)(ee >> 32), (ssa_u32)id,
                                                       (ssa_u32)(id >> 32), P.key0, P.key1);
            eub[hl] = make_double2(-ssa_plog(ssa_u53(o.o1, o.o0), c_plog), ssa_u53(o.o3, o.o2));
            need_rng = false;
            __syncwarp();
        }
        // a4: lane sum (sequential, two propensities per load), scan over the half (width 16).
        // (A pairwise-tree lane sum -- a 4-deep chain instead of 16 -- measured 2% slower; so did
        // rows kept in registers with the changed entries reloaded, and row sums re-done only by
        // the lanes whose rows changed: DESIGN.md §6.)
        double L = 0.0;
#pragma unroll
        for (int q = 0; q + 1 < SSA_P; q += 2) {
            const double2 v2 = *reinterpret_cast<const double2*>(a + hl * SSA_AR + q);
            L = __dadd_rn(__dadd_rn(L, v2.x), v2.y);
        }
        if (SSA_P & 1) L = __dadd_rn(L, a[hl * SSA_AR + SSA_P - 1]);
        double v = ssa_scan_step_m(L, 1, mk1);
        v = ssa_scan_step_m(v, 2, mk2);
        v = ssa_scan_step_m(v, 4, mk4);
        v = ssa_scan_step_m(v, 8, mk8);
        const double a0 = __shfl_sync(FULL, v, SSA_HL - 1, SSA_HL);
        // a5
        // (E, u2) of event e: one broadcast load (a half with no work left may hold a stale
        // ebase: the mask keeps its -- unused -- index inside the buffer)
        const double2 eu = eub[(int)(e - ebase) & 15];
        const double E = eu.x, u2 = eu.y;
        const unsigned a0hi = (unsigned)__double2hiint(a0);
        const bool fast = a0hi - (123u << 20) < ((1923u - 123u) << 20);   // a0 in [2^-900, 2^901)
        double tn = __dadd_rn(t, ssa_ddiv_inrange(E, a0));
        // a7: lane* = min{l : v_l > r}; then lane q of the half takes lane*'s q-th
        // propensity, a second scan gives s_q, p_q = v_{lane*-1} + s_q, q* = min{q : p_q > r}
        const double r = __dmul_rn(u2, a0);
        const unsigned bal = (__ballot_sync(FULL, v > r) >> (16 * h)) & 0xFFFFu;
        const int ls = __ffs(bal | 0x10000u) - 1;          // 16 when none (non-finite a0: rare path)
        const int lsc = ls & 15;
        const double base = __shfl_sync(FULL, v, lsc > 0 ? lsc - 1 : 0, SSA_HL);
        double y = (in_row && lsc * SSA_P + hl < SSA_R) ? a[lsc * SSA_AR + hl] : 0.0;
        y = ssa_scan_step_m(y, 1, mk1);
        y = ssa_scan_step_m(y, 2, mk2);
        y = ssa_scan_step_m(y, 4, mk4);
        y = ssa_scan_step_m(y, 8, mk8);
        const double p = (lsc > 0) ? __dadd_rn(base, y) : y;
        const unsigned bq = (__ballot_sync(FULL, in_row && p > r) >> (16 * h)) & 0xFFFFu;
        int j = lsc * SSA_P + (__ffs(bq) - 1);

        bool apply = live;
        if (live && (!fast || tn > s_next || bq == 0)) {     // rare path of this half
            bool fin = false;
            if (!fast) {
                if (a0 > 0.0 && a0 < INF) {
                    tn = __dadd_rn(t, __ddiv_rn(E, a0));
                } else if (a0 == 0.0) {
                    tn = INF;
                    absorbed = 1;
                } else {
                    status = 1;
                    int bad = SSA_R;
#pragma unroll
                    for (int q = SSA_P - 1; q >= 0; --q)
                        if (hl * SSA_P + q < SSA_R && !(fabs(a[hl * SSA_AR + q]) < INF)) bad = hl * SSA_P + q;
#pragma unroll
                    for (int o = 8; o > 0; o >>= 1) bad = min(bad, __shfl_xor_sync(HALF, bad, o, SSA_HL));
                    err_r = bad < SSA_R ? bad : -1;
                    fin = true;
                }
            }
            if (!fin && tn > s_next) {
                do {
                    const double tol = __dmul_rn(1e-9, s_next);
                    const bool near = (tn < INF && fabs(__dadd_rn(tn, -s_next)) <= tol) ||
                                      (e > 0 && fabs(__dadd_rn(t, -s_next)) <= tol);
                    ties += near ? 1 : 0;
                    int ovf = 0;
                    for (int s = hl; s < SSA_S; s += SSA_HL) {
                        const double xv = x[s];
                        ovf |= (xv > 2147483647.0) ? 1 : 0;
                        SSA_CHECK(k <= K && rel < P.n_ids, P.stats);
                        P.staging[rel * P.stride + (ssa_u64)k * SSA_S + s] = (int)xv;   // trajectory-major row
#if SSA_K2_DUMP
                        if (slot >= 0) P.dump_states[((ssa_u64)slot * G + (ssa_u64)k) * SSA_S + s] = (int)xv;
#endif
                    }
                    if (__any_sync(HALF, ovf)) status = 2;
#if SSA_K2_DUMP
                    if (slot >= 0 && hl == 0) {
                        P.dump_e[(ssa_u64)slot * G + (ssa_u64)k] = e;
                        P.dump_t[(ssa_u64)slot * G + (ssa_u64)k] = (e > 0) ? t : 0.0;
                    }
#endif
                    ++k;
                    s_next = (k <= K) ? __dmul_rn((double)k, dt) : INF;
                } while (tn > s_next);
                fin = (k > K);
            }
            if (fin) {
                // trajectory done: records, then refill this half
                if (hl == 0) {
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
                start();
                apply = false;
            } else if (bq == 0) {
                // rounding fallback: the largest j <= lane*'s last index with a_j > 0
                int lp = -1;
#pragma unroll
                for (int q = 0; q < SSA_P; ++q)
                    if (hl * SSA_P + q < SSA_R && a[hl * SSA_AR + q] > 0.0) lp = hl * SSA_P + q;
                const unsigned m2 = (__ballot_sync(HALF, lp >= 0 && hl <= lsc) >> (16 * h)) & 0xFFFFu;
                j = __shfl_sync(HALF, lp, 31 - __clz(m2), SSA_HL);
            }
        }
        if (!apply) j = 0;
        // Both halves run the update and the recompute loops (a half that does not
        // apply an event has empty ranges), so the two syncs are full-warp ones.
        {
            // a8: state update (lane t of the half takes the t-th net change)
            SSA_CHECK(j >= 0 && j < (SSA_R > 0 ? SSA_R : 1), P.stats);
            const int4 rj = rec[j];
            SSA_CHECK(!apply || (0 <= rj.x && rj.x <= rj.y && rj.y <= P.n_ent && 0 <= rj.z && rj.z <= rj.w &&
                                 rj.w <= P.n_dep), P.stats);
            const int nb = apply ? rj.x : 0, ne = apply ? rj.y : 0;
            const int db = apply ? rj.z : 0, de = apply ? rj.w : 0;
            // (one pass of 16 lanes covers the longest net-change list and, for most models,
            // the longest dependency list: single passes without loop control then)
#pragma unroll 2
            for (int q0 = 0; q0 < SSA_NU_MAX; q0 += SSA_HL) {
                const int q = nb + q0 + hl;
                if (q < ne) {
                    const int ent = nu_ent[q];
                    const int sp = ent & 0xFFFF;
                    SSA_CHECK(sp < SSA_S, P.stats);
                    x[sp] = __dadd_rn(x[sp], (double)(ent >> 16));
                }
            }
            __syncwarp();
            // a3: the half recomputes dep(j), one entry per lane
#pragma unroll 2
            for (int q0 = 0; q0 < SSA_DEP_MAX; q0 += SSA_HL) {
                const int q = db + q0 + hl;
                if (q >= de) continue;
                const ssa_u64 d = dent[q];
                const unsigned dhi = (unsigned)(d >> 32);
                SSA_CHECK((int)(dhi & 0x1FFu) < SSA_HL * SSA_AR && (int)(dhi & 0x1FFu) % SSA_AR < SSA_P &&
                          (int)(dhi >> 16) < SSA_R, P.stats);
#if SSA_K2_FE
                SSA_CHECK((int)(d & 0xFFFF) <= SSA_S && (int)((d >> 16) & 0xFFFF) <= SSA_S, P.stats);
                a[dhi & 0x1FFu] = k2h_fe(d, rt[dhi >> 16], x);
#elif !SSA_HAS_M3
                SSA_CHECK((int)(d & 0x3FFF) < SSA_S && (int)((d >> 14) & 0x3FFF) < SSA_S, P.stats);
                a[dhi & 0x1FFu] = k2h_propensity(d, rxd, x);
#else
                a[dhi & 0x1FFu] = k2_propensity(rx[(int)(dhi >> 16)], x);
#endif
            }
            __syncwarp();
            if (apply) {
                t = tn;
                ++e;
                need_rng = need_rng || (e - ebase >= 16);
#if SSA_K2_DUMP
                hash = (hash ^ (ssa_u64)j) * SSA_FNV_PRIME;
#endif
            }
        }
    }
    // per-warp counter totals (lanes 0 and 16 hold their halves' sums)
    my_events += __shfl_down_sync(FULL, my_events, 16);
    my_ties += __shfl_down_sync(FULL, my_ties, 16);
    if (lane == 0) {
        atomicAdd(&P.stats->events, my_events);
        if (my_ties) atomicAdd(&P.stats->near_ties, my_ties);
    }
}
#endif
