// k1_thread.cuh -- K1: one trajectory per thread, model-specialised (sm_100a).
//
// This text is compiled by NVRTC at run time, after ssa_device.cuh and a
// generated model section (runtime.cu: gen_k1_model) that defines
//   SSA_S, SSA_R, SSA_K1_BLOCK, SSA_K1_MINB
//   __constant__ double c_k[] (distinct rate / modifier constants), c_x0[]
//   ssa_khat(x, kh)       the modified rates k^ = max(0, k + d x_m), cached per trajectory
//   ssa_prefix(x, kh, c)  a3 + a4: c_j = c_{j-1} + a_j, sequential order (R13)
//   ssa_apply(j, x)       a8: x += nu_j (one indirect branch through a table)
//   ssa_first_bad(x)      first reaction with a non-finite propensity
// so that species counts (fp64, exact integers) and the propensity prefix
// live in registers, with the model's constants in constant memory.  The
// event loop is SURVEY.md §8(a) a1-a8; the definitions are those of
// DESIGN.md §2 and PAPER.md:60 ("a single transition amongst the possible
// ones is selected, and the state updated accordingly").
//
// Scheduling (north_star (c)): persistent threads; a lane that finishes a
// trajectory takes the next id from an atomic counter, so lanes are refilled
// as trajectories end.  Output is keyed by id, so results do not depend on
// the schedule.
//
// SSA_K1_DUMP = 0 (runs without dumped ids) drops the raw-trajectory dump
// and the firing hash, which only the dump exposes.
//
// Control flow: one loop iteration = one candidate event.  The common case
// (a0 in the fast-division range, no grid point crossed) runs straight
// through to the update with a single, rarely taken branch; everything else
// -- a grid crossing (a6), absorbing state, non-finite propensity, end of the
// trajectory and the refill (a1) -- lives on that rare path.

// ssa_k1_params is defined in ssa_device.cuh (shared with the host runtime).

// a7: j* = LO + #{ j in [LO, R-2] : c_j <= r }, valid when c_j <= r for all
// j < LO (c is nondecreasing and r < a0 = c_{R-1}); compare + predicated
// increment, in four independent partial sums to shorten the dependency chain.
template <int LO>
static __device__ __forceinline__ int ssa_count_from(const double (&c)[SSA_R > 0 ? SSA_R : 1], double r)
{
    int jp[4] = {0, 0, 0, 0};
#pragma unroll
    for (int q = LO; q < SSA_R - 1; ++q) {
        if (SSA_K1_SEL == 3)
            // speed A/B only: high words alone (a tie of high words miscounts; no fallback)
            asm("{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %1, %2;\n\t@p add.s32 %0, %0, 1;\n\t}"
                : "+r"(jp[q & 3]) : "r"(__double2hiint(c[q])), "r"(__double2hiint(r)));
        else if (SSA_K1_SEL == 1 || (SSA_K1_SEL == 2 && (q & 1)))
            // c_j, r >= +0 and not NaN: their bit patterns order as int64 (ALU pipe)
            asm("{\n\t.reg .pred p;\n\tsetp.le.s64 p, %1, %2;\n\t@p add.s32 %0, %0, 1;\n\t}"
                : "+r"(jp[q & 3]) : "l"(__double_as_longlong(c[q])), "l"(__double_as_longlong(r)));
        else
            asm("{\n\t.reg .pred p;\n\tsetp.le.f64 p, %1, %2;\n\t@p add.s32 %0, %0, 1;\n\t}"
                : "+r"(jp[q & 3]) : "d"(c[q]), "d"(r));
    }
    return LO + ((jp[0] + jp[1]) + (jp[2] + jp[3]));
}

#if SSA_K1_SELX
// a7 on the ALU pipe: j0 = #{ j in [0, R-2] : hi(c_j) < hi(r) }.  For c_j, r >= 0 finite the
// high words order as int32, so hi(c_j) < hi(r) implies c_j < r and hi(c_j) > hi(r) implies
// c_j > r: j0 <= j*, and j0 == j* unless hi(c_j0) == hi(r) (c is nondecreasing, so only the
// first entry not counted can tie).  ssa_apply_sel (runtime.cu) checks that tie in the update's
// own jump-table case and recounts in fp64 when it occurs (~1e-6 of events): the same j* as
// ssa_count_from, bit for bit.
static __device__ __forceinline__ int ssa_count_hi(const double (&c)[SSA_R > 0 ? SSA_R : 1], double r)
{
    int jp[4] = {0, 0, 0, 0};
    const int hr = __double2hiint(r);
#pragma unroll
    for (int q = 0; q < SSA_R - 1; ++q)
        asm("{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %1, %2;\n\t@p add.s32 %0, %0, 1;\n\t}"
            : "+r"(jp[q & 3]) : "r"(__double2hiint(c[q])), "r"(hr));
    return (jp[0] + jp[1]) + (jp[2] + jp[3]);
}
#endif

extern "C" __global__ void __launch_bounds__(SSA_K1_BLOCK, SSA_K1_MINB) ssa_k1(const ssa_k1_params P)
{
    const double INF = __longlong_as_double(0x7FF0000000000000ll);
    const double dt = P.dt;
    const long long K = P.K;
    const ssa_u64 G = (ssa_u64)K + 1;
    ssa_u64 my_events = 0, my_ties = 0;

#if SSA_K1_SWEEP
    // parameter sweep: the chunk's per-point constants in shared memory; kp
    // points at the row of the current trajectory's sweep point
    extern __shared__ double s_k[];
    for (int q = threadIdx.x; q < P.n_pts * P.n_pool; q += blockDim.x) s_k[q] = P.pconst[q];
    __syncthreads();
    const double* kp = s_k;
#endif
#if SSA_K1_MIG
    // tail compaction (P.mig_thresh > 0): live lanes per warp
    __shared__ int s_wlive[SSA_K1_BLOCK / 32];
    const int wid = threadIdx.x >> 5, wl = threadIdx.x & 31;
    const double s_last = __dmul_rn((double)K, dt);   // s_K: a crossing past it ends the trajectory
    bool may_suspend = true;                          // a resumed lane first crosses its pending grid point
    const bool mig = P.mig_thresh > 0 && !P.spread;
    volatile ssa_u64* const mctl = P.mig_ctl;
#endif
#if SSA_K1_SEG
    // time-sliced trajectories (P.seg > 1): job q of [0, seg * n_ids) is phase q / n_ids of
    // trajectory q % n_ids; phase p runs from the grid crossing where phase p - 1 stopped to the
    // one at index kb(p) = (p + 1) G / seg (the last phase to the end).  Jobs are handed out in
    // order, so the launch ends with the last phases -- 1/seg of a trajectory each -- instead of
    // whole trajectories running on an emptying GPU.  seg_ready[rel] = the next phase to run
    // (seg: finished); the state crosses phases through seg_buf as (x[S], t, e, k, hash, ties).
#if SSA_K1_MIG
    const int seg = (P.seg > 1 && !P.spread && !mig) ? P.seg : 1;
#else
    const int seg = (P.seg > 1 && !P.spread) ? P.seg : 1;
#endif
    int seg_p = 0;
    long long seg_kb = K + 2;
    auto seg_kb_of = [&](int p) -> long long {
        return p + 1 < seg ? (long long)(((ssa_u64)(p + 1) * G) / (ssa_u64)seg) : K + 2;
    };
#endif
    // plog's table in shared memory (lanes index it independently)
    __shared__ __align__(16) double s_plog_[128][4];
    for (int q = threadIdx.x; q < 128 * 4; q += blockDim.x) (&s_plog_[0][0])[q] = (&ssa_plog_tab[0][0])[q];
    __syncthreads();
    // the table's address computed once and kept opaque: otherwise the loop re-derives the
    // shared window base (S2R of the CTA id) every event
    const double (*s_plog)[4];
    {
        unsigned sa = (unsigned)__cvta_generic_to_shared(&s_plog_[0][0]);
        asm volatile("" : "+r"(sa));
        s_plog = (const double (*)[4])__cvta_shared_to_generic(sa);
    }
    // small ensembles (spread launch): one working lane per warp and one warp
    // per block, so each trajectory has an SM sub-partition to itself
    if (P.spread && (threadIdx.x & 31) != 0) return;
    double x[SSA_S];
    double kh[SSA_NKH > 0 ? SSA_NKH : 1];   // cached modified rates k^ (ssa_khat)
    // the propensity prefix (a4); with SSA_CSKIP its first SSA_CSKIP entries are
    // carried across iterations and recomputed only when a lane changed a species
    // they read (cold-prefix reuse, runtime.cu gen_k1_model)
    double c[SSA_R > 0 ? SSA_R : 1];
#if SSA_CSKIP
    bool lo_dirty = true;
#endif
    double t = 0.0, s_next = 0.0;
    ssa_u64 e = 0, hash = 0, ties = 0, rel = 0, id = 0, vid = 0;
    long long k = 0, slot = -1;
    int status = 0, absorbed = 0, err_r = -1;

#if SSA_K1_SWEEP
    ssa_u64 my_ptl = 0;                 // this lane's sweep point (chunk-local)
#endif
#if SSA_K1_SEG
    // time slices: trajectory rel's state between phases, S + 6 doubles at seg_buf[rel]
    auto seg_save = [&]() {
        double* st = P.seg_buf + rel * (ssa_u64)(SSA_S + 6);
#pragma unroll
        for (int s = 0; s < SSA_S; ++s) __stcg(st + s, x[s]);
        __stcg(st + SSA_S, t);
        __stcg(st + SSA_S + 1, __longlong_as_double((long long)e));
        __stcg(st + SSA_S + 2, __longlong_as_double(k));
        __stcg(st + SSA_S + 3, __longlong_as_double((long long)ties));
        __stcg(st + SSA_S + 4, __longlong_as_double((long long)hash));
    };
    auto seg_restore = [&](ssa_u64 r) {
        const double* st = P.seg_buf + r * (ssa_u64)(SSA_S + 6);
#pragma unroll
        for (int s = 0; s < SSA_S; ++s) x[s] = __ldcg(st + s);     // L2: written by another SM
        t = __ldcg(st + SSA_S);
        e = (ssa_u64)__double_as_longlong(__ldcg(st + SSA_S + 1));
        k = __double_as_longlong(__ldcg(st + SSA_S + 2));
        ties = (ssa_u64)__double_as_longlong(__ldcg(st + SSA_S + 3));
        hash = (ssa_u64)__double_as_longlong(__ldcg(st + SSA_S + 4));
        rel = r;
        vid = P.id_begin + rel;
        id = vid;
#if SSA_K1_DUMP
        slot = P.n_dump ? ssa_dump_slot(P.dump_ids, P.n_dump, vid) : -1ll;
#endif
        ssa_khat(x, kh SSA_KP_ARG);
        s_next = (k <= K) ? __dmul_rn((double)k, dt) : INF;
        status = 0; absorbed = 0; err_r = -1;
#if SSA_CSKIP
        lo_dirty = true;
#endif
    };
    // phase 0 of a job: take it; later phases: wait for and reload the state (true: resumed)
    auto seg_take = [&](int ph, bool& resumed) -> bool {
        resumed = false;
        if (ph == 0) { seg_p = 0; seg_kb = seg_kb_of(0); return true; }
        unsigned r;
        while ((r = ((volatile unsigned*)P.seg_ready)[rel]) < (unsigned)ph) __nanosleep(64);
        if (r > (unsigned)ph) return false;      // finished, or stopped at a later boundary
        __threadfence();
        seg_restore(rel);
        seg_p = ph;
        seg_kb = seg_kb_of(ph);
        resumed = true;
        return true;
    };
#endif
    // a1: take the next trajectory id (atomic counter) and initialise it
    auto start = [&]() -> bool {
#if SSA_K1_SWEEP
        {
            // sweep points are interleaved in the order lanes take work (w mod
            // points), so trajectories of short and long points mix over the
            // whole launch; the staging column stays point-major (dense per point)
            const ssa_u64 w = atomicAdd(P.work, 1ull);
            if (w >= P.n_ids) return false;
            ssa_u64 ptl;
            if (P.pt_order) {
                // points in the given order (costliest first, measured by an earlier run)
                const ssa_u64 o = w / P.n_per_point;
                ptl = (ssa_u64)P.pt_order[o];
                id = w - o * P.n_per_point;
            } else {
                ptl = w % (ssa_u64)P.n_pts;
                id = w / (ssa_u64)P.n_pts;      // trajectory id within its sweep point (RNG key)
            }
            my_ptl = ptl;
            rel = ptl * P.n_per_point + id;
            kp = s_k + ptl * (ssa_u64)P.n_pool;
        }
#else
#if SSA_K1_SEG
        if (seg > 1) {
            for (;;) {
                const ssa_u64 q = atomicAdd(P.work, 1ull);
                if (q >= (ssa_u64)seg * P.n_ids) return false;
                const int ph = (int)(q / P.n_ids);
                rel = q - (ssa_u64)ph * P.n_ids;
                // (phase ph - 1 of this trajectory was handed out n_ids jobs ago)
                bool resumed;
                if (!seg_take(ph, resumed)) continue;
                if (resumed) return true;
                break;                                 // a fresh trajectory (below)
            }
        } else
#endif
        {
            rel = atomicAdd(P.work, 1ull);
            if (rel >= P.n_ids) return false;
        }
#endif
        vid = P.id_begin + rel;
#if !SSA_K1_SWEEP
        id = vid;
#endif
#if SSA_K1_DUMP
        slot = P.n_dump ? ssa_dump_slot(P.dump_ids, P.n_dump, vid) : -1ll;
#endif
#pragma unroll
        for (int s = 0; s < SSA_S; ++s) x[s] = c_x0[s];
        ssa_khat(x, kh SSA_KP_ARG);
        t = 0.0; s_next = 0.0; e = 0; k = 0; hash = SSA_FNV_OFFSET; ties = 0;
        status = 0; absorbed = 0; err_r = -1;
#if SSA_CSKIP
        lo_dirty = true;
#endif
        return true;
    };

#if SSA_K1_RECORD
#define SSA_REC_BLOCK (SSA_K1_RECORD == 1 ? 256 : 32)
    ssa_u64 rec_cur = 0, rec_end = 0;   // this lane's reserved record rows [rec_cur, rec_end)
    // one row from the lane's block (a new block every SSA_REC_BLOCK rows; rows >= cap are dropped)
    auto rec_row = [&]() -> ssa_u64 {
        if (rec_cur == rec_end) {
            rec_cur = atomicAdd(P.rec_count, (ssa_u64)SSA_REC_BLOCK);
            rec_end = rec_cur + SSA_REC_BLOCK;
        }
        return rec_cur++;
    };
#endif
#if SSA_K1_RECORD == 2
    // stride-sampled output (SPEC.md:162 Stride(s)): (0, x0), every s-th event, the horizon
    ssa_u64 rec_left = 0;               // events until the next stride point
    double rec_last_t = 0.0;            // time of the last point emitted
    auto rec_point = [&](ssa_u64 seq, double tp) {
        const ssa_u64 pos = rec_row();
        if (pos < P.rec_cap) {
            P.rec_key[pos] = (rel << 41) | seq;
            P.rec_t[pos] = tp;
#pragma unroll
            for (int s = 0; s < SSA_S; ++s) P.rec_pre[pos * SSA_S + s] = (int)x[s];
        }
        rec_last_t = tp;
    };
#endif
#if SSA_K1_MIG
    // suspended trajectory slot q: (x[S], t, e, k, rel, hash, ties) as S + 6 doubles
    auto mig_restore = [&](ssa_u64 q) {
        SSA_CHECK(q < P.mig_cap, P.stats);
        while (((volatile unsigned*)P.mig_ready)[q] == 0u) __nanosleep(32);   // the pusher has reserved it
        __threadfence();
        const double* st = P.mig_buf + q * (ssa_u64)(SSA_S + 6);
#pragma unroll
        for (int s = 0; s < SSA_S; ++s) x[s] = __ldcg(st + s);     // L2: written by another SM
        t = __ldcg(st + SSA_S);
        e = (ssa_u64)__double_as_longlong(__ldcg(st + SSA_S + 1));
        k = __double_as_longlong(__ldcg(st + SSA_S + 2));
        rel = (ssa_u64)__double_as_longlong(__ldcg(st + SSA_S + 3));
        hash = (ssa_u64)__double_as_longlong(__ldcg(st + SSA_S + 4));
        ties = (ssa_u64)__double_as_longlong(__ldcg(st + SSA_S + 5));
        vid = P.id_begin + rel;
        id = vid;
#if SSA_K1_DUMP
        slot = P.n_dump ? ssa_dump_slot(P.dump_ids, P.n_dump, vid) : -1ll;
#endif
        ssa_khat(x, kh SSA_KP_ARG);
        s_next = (k <= K) ? __dmul_rn((double)k, dt) : INF;
        status = 0; absorbed = 0; err_r = -1;
        may_suspend = false;
#if SSA_CSKIP
        lo_dirty = true;
#endif
    };
    // push this lane's trajectory (false: the buffer is full)
    auto mig_push = [&]() -> bool {
        ssa_u64 pt = mctl[0];
        for (;;) {
            if (pt >= P.mig_cap) return false;
            const ssa_u64 o = atomicCAS((ssa_u64*)&P.mig_ctl[0], pt, pt + 1);
            if (o == pt) break;
            pt = o;
        }
        double* st = P.mig_buf + pt * (ssa_u64)(SSA_S + 6);
#pragma unroll
        for (int s = 0; s < SSA_S; ++s) __stcg(st + s, x[s]);
        __stcg(st + SSA_S, t);
        __stcg(st + SSA_S + 1, __longlong_as_double((long long)e));
        __stcg(st + SSA_S + 2, __longlong_as_double(k));
        __stcg(st + SSA_S + 3, __longlong_as_double((long long)rel));
        __stcg(st + SSA_S + 4, __longlong_as_double((long long)hash));
        __stcg(st + SSA_S + 5, __longlong_as_double((long long)ties));
        __threadfence();
        atomicExch(&P.mig_ready[pt], 1u);
        return true;
    };
    // take one suspended trajectory (false: none)
    auto mig_pop1 = [&]() -> bool {
        ssa_u64 pb = mctl[1];
        for (;;) {
            if (pb >= mctl[0]) return false;
            const ssa_u64 o = atomicCAS((ssa_u64*)&P.mig_ctl[1], pb, pb + 1);
            if (o == pb) break;
            pb = o;
        }
        mig_restore(pb);
        return true;
    };
#endif
    bool live = start();
#if SSA_K1_RECORD == 2
    if (live) { rec_left = P.rec_stride; rec_point(0, 0.0); }
#endif
#if SSA_K1_MIG
    bool running = false;      // this warp is counted in mig_ctl[3] (warp-uniform)
    if (mig) {
        const unsigned b = __ballot_sync(0xffffffffu, live);
        if (wl == 0) {
            s_wlive[wid] = __popc(b);
            if (b) atomicAdd((ssa_u64*)&P.mig_ctl[3], 1ull);
        }
        running = b != 0;
        __syncwarp();
    }
    for (;;) {
#endif
    while (live) {
        // a2: one Philox block per candidate event, counter (e, id)
#if SSA_KS_IMM
        // key schedule compiled in: the round keys are instruction immediates
        const ssa_philox_out o = ssa_philox_seeded((ssa_u32)e, (ssa_u32)(e >> 32), (ssa_u32)id, (ssa_u32)(id >> 32));
#else
        const ssa_philox_out o = ssa_philox4x32_10_ks((ssa_u32)e, (ssa_u32)(e >> 32), (ssa_u32)id,
                                                      (ssa_u32)(id >> 32), P.ks);
#endif
        // a3 + a4 (the propensity prefix chain) and a5's logarithm are
        // independent dependency chains in one basic block, so the scheduler
        // interleaves them.
#if SSA_CSKIP
        // c_0..c_{CSKIP-1}: recomputed by the whole warp (a uniform branch) when any
        // lane's last event changed a species they read, else reused as they are
        if (__any_sync(__activemask(), lo_dirty)) ssa_prefix_lo(x, kh, c SSA_KP_ARG);
        const double a0 = ssa_prefix_hi(x, kh, c SSA_KP_ARG);
#else
        const double a0 = ssa_prefix(x, kh, c SSA_KP_ARG);
#endif
#if SSA_K1_PROF
        // dispatch profile (a model's first thread-path run): at every 4096th event of a
        // trajectory, the propensity shares a_j / a0 of the current state -- their mean
        // estimates each reaction's share of the events; prof[R] counts the samples
        if (P.prof && (e & 4095ull) == 4095ull && a0 > 0.0 && a0 < INF) {
            double prev = 0.0;
            for (int q = 0; q < SSA_R; ++q) {
                atomicAdd(&P.prof[q], (c[q] - prev) / a0);
                prev = c[q];
            }
            atomicAdd(&P.prof[SSA_R], 1.0);
        }
#endif
        // keep the prefix in registers: without this barrier the compiler
        // recomputes the whole propensity chain for the selection (a7)
#pragma unroll
        for (int q = 0; q < SSA_R - 1; ++q) asm volatile("" : "+d"(c[q]));
#if SSA_PLOG_DIV
        const double E = -ssa_plog_div(ssa_u53(o.o1, o.o0), c_plog_div);   // speed A/B only
#elif SSA_PLOG_GLOBAL
        const double E = -ssa_plog(ssa_u53(o.o1, o.o0), c_plog);
#else
        const double E = -ssa_plog<true>(ssa_u53(o.o1, o.o0), c_plog, s_plog);
#endif
        // a7, speculatively (used only if the event is applied): r = u2 a0,
        // j* = #{ j : c_j <= r } (c nondecreasing, r < a0), counted in four
        // independent partial sums to shorten the dependency chain.
        const double r = __dmul_rn(ssa_u53(o.o3, o.o2), a0);
#if SSA_K1_SELX
        int j = ssa_count_hi(c, r);   // j0 <= j*: made exact by ssa_apply_sel
#else
        const int j = ssa_count_from<0>(c, r);
#endif
        SSA_CHECK(j >= 0 && j < (SSA_R > 0 ? SSA_R : 1), P.stats);
        // a5: tau = E / a0 by the fast in-range IEEE division (speculative:
        // replaced on the rare path when a0 is outside [2^-900, 2^901))
        const unsigned a0hi = (unsigned)__double2hiint(a0);
        const bool fast = a0hi - (123u << 20) < ((1923u - 123u) << 20);
        double tn = __dadd_rn(t, ssa_ddiv_inrange(E, a0));
        if (!fast || tn > s_next) {
            // ---------------- rare path: a5 edge cases, a6, end + refill
#if SSA_K1_MIG
            // tail compaction: no ids left, this warp is sparse and another warp runs --
            // suspend before this grid crossing (the candidate is a function of (x, t, e),
            // so the resumed lane recomputes it bit for bit) and leave the warp
            if (mig && may_suspend && status == 0 && fast && tn <= s_last &&
                *(volatile int*)&s_wlive[wid] <= P.mig_thresh && *(volatile ssa_u64*)P.work >= P.n_ids &&
                mctl[3] > 1 && mig_push()) {
                atomicSub(&s_wlive[wid], 1);
                live = false;
                continue;
            }
#endif
#if SSA_K1_SEG
            // time slice: at the first crossing at or past this phase's boundary, hand the
            // trajectory to its next phase's job (the candidate is a function of (x, t, e): the
            // resumed lane recomputes it bit for bit and processes this crossing)
            if (seg > 1 && k >= seg_kb && status == 0 && fast) {
                seg_save();
                __threadfence();
                atomicExch(&P.seg_ready[rel], (unsigned)(seg_p + 1));
                live = start();
                continue;
            }
#endif
            bool fin = false;
            if (!fast) {
                if (a0 > 0.0 && a0 < INF) {
                    tn = __dadd_rn(t, __ddiv_rn(E, a0));
                } else if (a0 == 0.0) {
                    tn = INF;            // absorbing: hold x to the end of the grid
                    absorbed = 1;
                } else {
                    tn = INF;            // non-finite propensity: error (id, reaction)
                    status = 1;
                    err_r = ssa_first_bad(x SSA_KP_ARG);
                    fin = true;
                }
            }
            // a6: grid alignment (selective memory on the grid): x is the
            // state just before the first event past s_k
            if (!fin && tn > s_next) {
                do {
                    const double tol = __dmul_rn(1e-9, s_next);
                    const bool near = (tn < INF && fabs(__dadd_rn(tn, -s_next)) <= tol) ||
                                      (e > 0 && fabs(__dadd_rn(t, -s_next)) <= tol);
                    ties += near ? 1 : 0;
                    SSA_CHECK(k <= K && rel < P.n_ids && (ssa_u64)(k + 1) * SSA_S <= P.stride, P.stats);
                    int* dst = P.staging + rel * P.stride + (ssa_u64)k * SSA_S;   // trajectory-major row
#pragma unroll
                    for (int s = 0; s < SSA_S; ++s) {
                        if (x[s] > 2147483647.0) status = 2;
                        dst[s] = (int)x[s];
                    }
#if SSA_K1_DUMP
                    if (slot >= 0) {
                        SSA_CHECK((ssa_u64)slot < P.n_dump, P.stats);
                        const ssa_u64 base = (ssa_u64)slot * G + (ssa_u64)k;
#pragma unroll
                        for (int s = 0; s < SSA_S; ++s) P.dump_states[base * SSA_S + s] = (int)x[s];
                        P.dump_e[base] = e;
                        P.dump_t[base] = (e > 0) ? t : 0.0;
                    }
#endif
                    ++k;
                    s_next = (k <= K) ? __dmul_rn((double)k, dt) : INF;
                } while (tn > s_next);
                fin = (k > K);
#if SSA_K1_MIG
                may_suspend = true;
#endif
            }
            if (fin) {
                // trajectory done: per-trajectory records, then refill (a1)
#if SSA_K1_SEG
                if (seg > 1) atomicExch(&P.seg_ready[rel], (unsigned)seg);   // later phases: nothing to do
#endif
                my_events += e;
                my_ties += ties;
#if SSA_K1_SWEEP
                if (P.pt_events) atomicAdd(&P.pt_events[my_ptl], e);
#endif
#if SSA_K1_DUMP
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
                    // smallest id wins; pack (id, code, reaction) so one atomicMin keeps them together
                    const ssa_u64 packed = (vid << 24) | (code << 20) | ((ssa_u64)(err_r + 1) & 0xFFFFFull);
                    atomicMin(&P.stats->first_err_id, packed);
                }
#if SSA_K1_RECORD == 2
                // the horizon point (held state at s_K), unless the last point is already there
                {
                    const double hz = __dmul_rn((double)K, dt);
                    if (rec_last_t < hz) rec_point(2 * e + 1, hz);
                }
#endif
#if SSA_K1_MIG
                if (mig) atomicAdd((ssa_u64*)&P.mig_ctl[2], ~0ull);   // one trajectory fewer to finish
#endif
                live = start();
#if SSA_K1_MIG
                // no ids left: a lane of a dense warp takes a suspended trajectory
                if (!live && mig && *(volatile int*)&s_wlive[wid] > P.mig_thresh) live = mig_pop1();
                if (!live && mig) atomicSub(&s_wlive[wid], 1);
#endif
#if SSA_K1_RECORD == 2
                if (live) { rec_left = P.rec_stride; rec_point(0, 0.0); }
#endif
                continue;
            }
        }
        // a8: apply the selected reaction
#if SSA_K1_RECORD == 1
        {   // full event stream (union-time selective memory): time, reaction,
            // pre-event counts, in this lane's current block of reserved rows;
            // the counts are stored by the update's own jump-table case
            const ssa_u64 pos = rec_row();
            int* out = nullptr;
            if (pos < P.rec_cap) {
                P.rec_t[pos] = tn;
                P.rec_j[pos] = j;
                out = P.rec_pre + pos * SSA_REC_U;
            }
            ssa_apply_rec(j, x, out);
        }
#elif SSA_K1_SELX
        j = ssa_apply_sel(j, x, c, r);   // j* exact from here on
#else
        ssa_apply(j, x);
#endif
        if (ssa_khat_dirty(j)) ssa_khat(x, kh SSA_KP_ARG);   // a modifier species changed
#if SSA_CSKIP
        lo_dirty = !ssa_lo_clean(j);
#endif
        t = tn;
        ++e;
#if SSA_K1_DUMP
        hash = (hash ^ (ssa_u64)j) * SSA_FNV_PRIME;   // firing hash: observable only through the dump
#endif
#if SSA_K1_RECORD == 2
        if (--rec_left == 0) {
            rec_point(2 * e, t);
            rec_left = P.rec_stride;
        }
#endif
    }
#if SSA_K1_MIG
        // every lane of this warp is idle: take up to 32 suspended trajectories at once
        // (a full warp's worth, or what is left once no warp runs), or stop when every
        // trajectory of the launch has finished
        if (!mig) break;
        __syncwarp();
        if (running && wl == 0) atomicAdd((ssa_u64*)&P.mig_ctl[3], ~0ull);
        running = false;
        long long got = 0;
        ssa_u64 base = 0;
        ssa_u64 seen = ~0ull, since = 0;   // safety: stop after 30 s without any progress of the launch
        ssa_u64 pending = 0;               // since when suspended trajectories have been waiting (ns)
        for (;;) {
            if (wl == 0) {
                got = 0;
                const ssa_u64 pt = mctl[0], pb = mctl[1];
                const ssa_u64 avail = pt > pb ? pt - pb : 0;
                ssa_u64 now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                if (avail == 0) pending = 0;
                else if (pending == 0) pending = now;
                // a full warp's worth, or whatever is left once no warp runs or it has waited 100 us
                if (avail >= 32 || (avail > 0 && (mctl[3] == 0 || now - pending > 100000ull))) {
                    const ssa_u64 n = avail < 32 ? avail : 32;
                    if (atomicCAS((ssa_u64*)&P.mig_ctl[1], pb, pb + n) == pb) {
                        base = pb;
                        got = (long long)n;
                        atomicAdd((ssa_u64*)&P.mig_ctl[3], 1ull);
                        s_wlive[wid] = (int)n;
                    }
                } else if (mctl[2] == 0) {
                    got = -1;                   // every trajectory has finished
                } else {
                    const ssa_u64 prog = mctl[2] * 0x9E3779B97F4A7C15ull + pt * 31 + pb;
                    if (prog != seen) { seen = prog; since = now; }
                    else if (now - since > 30000000000ull) got = -1;   // the host reports what is left
                }
            }
            got = __shfl_sync(0xffffffffu, got, 0);
            if (got != 0) break;
            __nanosleep(2000);
        }
        if (got < 0) break;
        base = __shfl_sync(0xffffffffu, base, 0);
        running = true;
        __syncwarp();
        live = (long long)wl < got;
        if (live) mig_restore(base + (ssa_u64)wl);
    }
#endif
#if SSA_K1_RECORD
    // unused reserved rows sort last: time +inf
    for (; rec_cur < rec_end; ++rec_cur)
        if (rec_cur < P.rec_cap) {
            P.rec_t[rec_cur] = INF;
#if SSA_K1_RECORD == 1
            P.rec_j[rec_cur] = 0;
#else
            P.rec_key[rec_cur] = ~0ull;
#endif
        }
#endif
    if (P.spread) {   // one lane per warp: no warp reduction
        atomicAdd(&P.stats->events, my_events);
        if (my_ties) atomicAdd(&P.stats->near_ties, my_ties);
        return;
    }
    // warp-level reduction of the counters, then one atomic per warp
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        my_events += __shfl_down_sync(0xffffffffu, my_events, off);
        my_ties += __shfl_down_sync(0xffffffffu, my_ties, off);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&P.stats->events, my_events);
        if (my_ties) atomicAdd(&P.stats->near_ties, my_ties);
    }
}
