// union.cu -- union-time selective memory on sm_100a.
//
// The paper's selective memory aligns the streams of k simulations by
// simulation time before reducing them (§3.2.1, Fig. 3 left:
// Avg-Y "derived via oversampling and time-aligned reduction"), then reduces
// k_x successive aligned points along time (Fig. 3 right: Avg-XY).  SPEC.md
// (:244-262) writes it as Y-points at every distinct union time u -- each
// stream's zero-order-hold value at u, folded into (n, sum, sumsq) -- grouped
// k_x at a time (group time = mean of the Y-times).  Here, for one ensemble
// whose full event streams were recorded by K1 (record variant):
//   1. sort all events by time (CUB radix sort of the fp64 bit patterns --
//      times are positive, so they order as unsigned integers);
//   2. the last event of every run of equal times is a Y-point (equal union
//      times collapse into one slice); an exclusive scan of those run ends
//      gives every event its Y-point y(e) (Y-points are 0, the D run ends, and
//      the horizon);
//   3. the X-groups are cut into tiles of <= 256, one thread per group (a
//      group's events are contiguous after the sort; the thread owns the
//      group's row of per-species accumulators in shared memory -- no
//      atomics); pass T sums each tile's exact changes of sum x and sum x^2
//      (d1 = nu, d2 = 2 x nu + nu^2 from the recorded pre-event count; only
//      the <= U species each reaction changes -- sparse, no dense
//      per-species columns) and a small scan over the tiles gives each
//      tile's starting sums;
//   4. pass F re-reads the tile's events once more: per group the plain and
//      the Y-weighted changes and the left-to-right sum of its Y-times, a
//      per-species prefix over the tile's groups, then for group g
//        sum_{y in g} S(y) = m_g P(g) + sum_{e in g} (y1(g) - y(e)) d(e)
//      exactly in integers, mean = S1/n and population variance
//      (n S2 - S1^2)/n^2 correctly rounded.
// After the sort every pass streams the sorted events once (the gathers of the
// recorded rows follow the k trajectories' own time-ordered blocks).
#include <cub/cub.cuh>
#include <algorithm>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "ssa_kernels.h"

namespace {

__global__ void k_keys(const double* __restrict__ t, ssa_u64 E, ssa_u64* __restrict__ keys,
                       unsigned* __restrict__ idx)
{
    for (ssa_u64 m = blockIdx.x * (ssa_u64)blockDim.x + threadIdx.x; m < E; m += (ssa_u64)gridDim.x * blockDim.x) {
        keys[m] = (ssa_u64)__double_as_longlong(t[m]);
        idx[m] = (unsigned)m;
    }
}

// N / D rounded once to the nearest double (ties to even), for 0 <= N, 0 < D < 2^126:
// the quotient's first 55 significant bits by integer (long) division, the rest folded
// into a sticky bit -- the value a correctly rounded exact division (the oracle's
// Fraction -> float) gives, so means and variances are bitwise the oracle's.
__device__ int bitlen128(unsigned __int128 v)
{
    const unsigned long long hi = (unsigned long long)(v >> 64), lo = (unsigned long long)v;
    return hi ? 128 - __clzll((long long)hi) : (lo ? 64 - __clzll((long long)lo) : 0);
}

__device__ double ratio_rn(unsigned __int128 N, unsigned __int128 D)
{
    if (N == 0) return 0.0;
    unsigned __int128 q = N / D, r = N % D;
    int ex = 0;
    bool sticky;
    const int qb = bitlen128(q);
    if (qb > 55) {
        const int sh = qb - 55;
        sticky = r != 0 || (q & ((((unsigned __int128)1) << sh) - 1)) != 0;
        q >>= sh;
        ex = sh;
    } else {
        while (bitlen128(q) < 55) {      // next quotient bits of the fraction r / D
            r <<= 1;
            const bool b = r >= D;
            if (b) r -= D;
            q = (q << 1) | (b ? 1u : 0u);
            --ex;
        }
        sticky = r != 0;
    }
    unsigned long long m = (unsigned long long)(q >> 2);
    const bool guard = ((unsigned)q >> 1) & 1u, rest = (((unsigned)q & 1u) != 0) || sticky;
    if (guard && (rest || (m & 1ull))) ++m;
    if (m == (1ull << 53)) { m >>= 1; ++ex; }
    return ldexp((double)m, ex + 2);
}

// N / D correctly rounded: one IEEE division when both are exact doubles (the
// quotient of two exact operands rounded once is the correctly rounded ratio),
// else the integer long division above.
__device__ double div_rn(unsigned __int128 N, unsigned __int128 D)
{
    const unsigned __int128 lim = ((unsigned __int128)1) << 53;
    if (N < lim && D < lim) {
        const unsigned long long d = (unsigned long long)D;
        if ((d & (d - 1)) == 0)                                 // n = k k_x is often 2^p: an exact scaling
            return (double)(unsigned long long)N * __longlong_as_double((long long)(1023 - (63 - __clzll(d))) << 52);
        return __ddiv_rn((double)(unsigned long long)N, (double)d);
    }
    return ratio_rn(N, D);
}

// the union-time Y-point of sorted event m: 1 + (equal-time runs ending before m)
__device__ __forceinline__ ssa_u64 y_of(const unsigned* __restrict__ yi, ssa_u64 m) { return 1ull + yi[m]; }

// first event of every X-group (groups without events start at E; group 0
// starts at 0 -- Y-point 0 is the initial slice, with no event)
__global__ void k_group_starts_init(ssa_u64 E, ssa_u64 NX, ssa_u64* __restrict__ gs)
{
    for (ssa_u64 g = blockIdx.x * (ssa_u64)blockDim.x + threadIdx.x; g <= NX; g += (ssa_u64)gridDim.x * blockDim.x)
        gs[g] = g == 0 ? 0 : E;
}

__global__ void k_group_starts_scatter(const unsigned* __restrict__ yi, ssa_u64 E, ssa_u64 kx,
                                       ssa_u64* __restrict__ gs)
{
    for (ssa_u64 m = blockIdx.x * (ssa_u64)blockDim.x + threadIdx.x; m < E; m += (ssa_u64)gridDim.x * blockDim.x) {
        const ssa_u64 y = y_of(yi, m);
        if ((m == 0 || yi[m - 1] != yi[m]) && y % kx == 0) gs[y / kx] = m;
    }
}

// One pass over the sorted events, in tiles.  A warp owns a segment of GW
// consecutive X-groups (lane l owns group l; a group's events are contiguous
// after the sort); a block of WPB warps is a tile, taken in order from a ticket
// counter.  Each warp stages its segment's events through shared memory BT at
// a time -- coalesced, independent loads by all 32 lanes -- and the owners
// walk their own group's events in order out of shared memory into the
// group's row of per-species accumulators: no atomics, no cross-lane
// dependence.  The tiles' starting sums come from a decoupled look-back over
// the preceding tiles' published totals.
struct Geo {
    ssa_u64 E, NY, NX;
    unsigned GW;                       // groups per warp (<= 32)
    int WPB;                           // warps per block
    int BT;                            // events staged per warp per batch
    int horizon;                       // Y-point D+1 at t_end exists
};

__host__ __device__ inline size_t stage_bytes(int BT, int U) { return (size_t)BT * (16 + 4 * (size_t)U); }
__host__ __device__ inline int row_stride(int S) { return 4 * S + 1; }      // odd: owners' rows spread over banks

struct Stage {
    double* t;                         // event time
    unsigned* ev;                      // recorded row
    int* j;                            // reaction | 1 << 31 at a Y-point (the last event of its time)
    int* pre;                          // [BT][U] pre-event counts
};

__device__ __forceinline__ Stage stage_at(char* base, int BT, int U, int w)
{
    char* p = base + (size_t)w * stage_bytes(BT, U);
    Stage st;
    st.t = (double*)p;
    st.ev = (unsigned*)(st.t + BT);
    st.j = (int*)(st.ev + BT);
    st.pre = st.j + BT;
    return st;
}

// Two phases, each a run of independent global loads: the sorted arrays, then
// the recorded rows they name.  The SM issues in order and a store waits for
// the load it stores, so each lane first issues the loads of SB events into
// registers and only then stores them (load, store, load, store ... would pay
// one full memory latency per load).  __ldg: global-space loads, free to move
// past the shared-memory stores.
#define SB 4
__device__ __forceinline__ void stage_load(const ssa_union_args& a, const Geo& G, Stage st, ssa_u64 cb, int n,
                                           const unsigned* __restrict__ perm, const unsigned* __restrict__ yi,
                                           const ssa_u64* __restrict__ sk, int lane)
{
    const int U = a.U;
    const int* __restrict__ rj = a.rec_j;
    const int* __restrict__ rp = a.rec_pre;
    for (int i0 = lane; i0 < n; i0 += 32 * SB) {
        unsigned yv[SB], yn[SB], pm[SB];
        ssa_u64 kt[SB];
#pragma unroll
        for (int k = 0; k < SB; ++k) {
            const int i = i0 + 32 * k;
            const ssa_u64 mm = cb + (i < n ? i : 0);
            yv[k] = __ldg(yi + mm);
            yn[k] = mm + 1 < G.E ? __ldg(yi + mm + 1) : ~0u;
            kt[k] = __ldg(sk + mm);
            pm[k] = __ldg(perm + mm);
        }
#pragma unroll
        for (int k = 0; k < SB; ++k) {
            const int i = i0 + 32 * k;
            if (i < n) {
                st.t[i] = __longlong_as_double((long long)kt[k]);
                st.ev[i] = pm[k] | (yn[k] != yv[k] ? 0x80000000u : 0u);
            }
        }
    }
    __syncwarp();
    for (int i0 = lane; i0 < n; i0 += 32 * SB) {
        unsigned ev[SB], fl[SB];
        int jj[SB], pv[SB][4];
#pragma unroll
        for (int k = 0; k < SB; ++k) {
            const int i = i0 + 32 * k;
            const unsigned e = i < n ? st.ev[i] : st.ev[i0];
            ev[k] = e & 0x7fffffffu;
            fl[k] = e & 0x80000000u;
        }
#pragma unroll
        for (int k = 0; k < SB; ++k) {
            jj[k] = __ldg(rj + ev[k]);
#pragma unroll
            for (int q = 0; q < 4; ++q) pv[k][q] = q < U ? __ldg(rp + (ssa_u64)ev[k] * U + q) : 0;
        }
#pragma unroll
        for (int k = 0; k < SB; ++k) {
            const int i = i0 + 32 * k;
            if (i < n) {
                st.j[i] = jj[k] | (int)fl[k];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (q < U) st.pre[i * U + q] = pv[k][q];
                for (int q = 4; q < U; ++q) st.pre[i * U + q] = __ldg(rp + (ssa_u64)ev[k] * U + q);
            }
        }
    }
}
#undef SB

// Per tile -- each group's own changes (A: plain, B: weighted by the Y-points
// of the group at or after the event) and its Y-time sum, the tile's starting
// sums (look-back), the per-species exclusive prefix over the tile's groups,
// then the groups' exact sums, means and variances.  Sum over the Y-points y of
// group g of the ensemble sum
//   = m_g * P(g) + sum over events e in g of (y1(g) - y(e)) * delta(e),
// P(g) the sum just before the group's first Y-point, m_g its Y-points.
__global__ void __launch_bounds__(128) k_union_pass(ssa_union_args a, Geo G, const unsigned* __restrict__ perm,
                                                    const unsigned* __restrict__ yi, const ssa_u64* __restrict__ sk,
                                                    const ssa_u64* __restrict__ gs, long long* agg, long long* incl,
                                                    unsigned* flag, unsigned* ticket)
{
    extern __shared__ long long sh[];                // rows [WPB*GW][RS] (A1 A2 B1 B2), seg [WPB][2S], tpre [2S], staging
    __shared__ unsigned s_tile;
    const int S = a.S, S2 = 2 * S, RS = row_stride(S), U = a.U, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const unsigned t = s_tile;
    const ssa_u64 TG = (ssa_u64)G.WPB * G.GW, g0 = t * TG;
    const unsigned ng = (unsigned)((G.NX - g0 < TG) ? G.NX - g0 : TG);
    const ssa_u64 kx = a.kx;
    long long* seg = sh + TG * RS;
    long long* tpre = seg + G.WPB * S2;
    const Stage st = stage_at((char*)(tpre + S2), G.BT, U, w);
    const unsigned gl = w * G.GW + lane;
    const unsigned nw = (w * G.GW < ng) ? min(G.GW, ng - w * G.GW) : 0;   // groups of this warp
    const bool own = (unsigned)lane < nw;
    long long* r = sh + (ssa_u64)gl * RS;
    ssa_u64 m = 0, m1 = 0, y0 = 0, y1 = 0, yc = 0;
    double tsum = 0.0;
    if (own) {
        for (int c = 0; c < 4 * S; ++c) r[c] = 0;
        const ssa_u64 g = g0 + gl;
        y0 = g * kx;
        y1 = (y0 + kx < G.NY) ? y0 + kx : G.NY;
        yc = y0 ? y0 : 1;                            // Y-point of the group's next event (0 has none)
        if (y0 == 0) tsum = __dadd_rn(tsum, 0.0);
        m = gs[g];
        m1 = gs[g + 1];
    }
    ssa_u64 e0 = 0, e1 = 0;
    if (nw) {
        e0 = gs[g0 + w * G.GW];
        e1 = gs[g0 + w * G.GW + nw];
    }
    for (ssa_u64 cb = e0; cb < e1; cb += G.BT) {
        const int n = (int)((e1 - cb < (ssa_u64)G.BT) ? e1 - cb : G.BT);
        __syncwarp();
        stage_load(a, G, st, cb, n, perm, yi, sk, lane);
        __syncwarp();
        if (own) {
            const ssa_u64 ce = (m1 < cb + n) ? m1 : cb + n;
            for (; m < ce; ++m) {
                const int i = (int)(m - cb), jf = st.j[i], j = jf & 0x7fffffff;
                const long long wt = (long long)(y1 - yc);
                for (int q = 0; q < U; ++q) {
                    const int sp = __ldg(a.nu_sp + j * U + q);
                    if (sp < 0) continue;
                    const long long v = __ldg(a.nu_d + j * U + q), x = st.pre[i * U + q];
                    const long long d2 = 2 * x * v + v * v;
                    r[sp] += v;
                    r[S + sp] += d2;
                    r[2 * S + sp] += wt * v;
                    r[3 * S + sp] += wt * d2;
                }
                if (jf < 0) {                                          // a Y-point: its time, left to right
                    tsum = __dadd_rn(tsum, st.t[i]);
                    ++yc;
                }
            }
        }
    }
    if (own) {
        const ssa_u64 g = g0 + gl;
        if (G.horizon && y1 == G.NY) tsum = __dadd_rn(tsum, a.t_end);
        a.times[g] = __ddiv_rn(tsum, (double)(y1 - y0));
        a.count[g] = (double)((long long)a.k * (long long)(y1 - y0));
    }
    __syncthreads();
    // the warp segments' column totals (a lane per column, down the rows)
    for (int c = lane; c < S2; c += 32) {
        long long v = 0;
        for (unsigned q = 0; q < nw; ++q) v += sh[(ssa_u64)(w * G.GW + q) * RS + c];
        seg[w * S2 + c] = v;
    }
    __syncthreads();
    // decoupled look-back: publish this tile's total, add up the predecessors'
    if (w == 0) {
        for (int c = lane; c < S2; c += 32) {
            long long v = 0;
            for (int k = 0; k < G.WPB; ++k) v += seg[k * S2 + c];
            if (t == 0) {
                const long long s0 = c < S ? a.s0[c] : a.s0sq[c - S];
                tpre[c] = s0;
                __stcg(incl + c, s0 + v);
            } else {
                tpre[c] = 0;
                __stcg(agg + (ssa_u64)t * S2 + c, v);
            }
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicExch(flag + t, t == 0 ? 2u : 1u);
        if (t > 0) {
            for (long long p = (long long)t - 1;; --p) {
                unsigned f;
                do {
                    f = *(volatile unsigned*)(flag + p);
                } while (f == 0);
                __threadfence();
                const long long* src = (f == 2 ? incl : agg) + (ssa_u64)p * S2;
                for (int c = lane; c < S2; c += 32) tpre[c] += __ldcg(src + c);
                if (f == 2) break;
            }
            for (int c = lane; c < S2; c += 32) {
                long long v = 0;
                for (int k = 0; k < G.WPB; ++k) v += seg[k * S2 + c];
                __stcg(incl + (ssa_u64)t * S2 + c, tpre[c] + v);
            }
            __threadfence();
            __syncwarp();
            if (lane == 0) atomicExch(flag + t, 2u);
        }
    }
    __syncthreads();
    // rows' A -> exclusive prefix P (a lane per column, down the warp's rows)
    for (int c = lane; c < S2; c += 32) {
        long long run = tpre[c];
        for (int k = 0; k < w; ++k) run += seg[k * S2 + c];
        for (unsigned q = 0; q < nw; ++q) {
            long long* p = sh + (ssa_u64)(w * G.GW + q) * RS + c;
            const long long v = *p;
            *p = run;
            run += v;
        }
    }
    __syncthreads();
    const unsigned cells = ng * (unsigned)S;
    for (unsigned i = threadIdx.x; i < cells; i += blockDim.x) {
        const unsigned q = i / (unsigned)S, sp = i - q * (unsigned)S;
        const ssa_u64 g = g0 + q;
        const ssa_u64 gy0 = g * kx, gy1 = (gy0 + kx < G.NY) ? gy0 + kx : G.NY;
        const long long mg = (long long)(gy1 - gy0), n = (long long)a.k * mg;
        const long long* rr = sh + (ssa_u64)q * RS;
        const __int128 x1 = (__int128)mg * rr[sp] + rr[2 * S + sp];
        const __int128 x2 = (__int128)mg * rr[S + sp] + rr[3 * S + sp];
        const __int128 num = (__int128)n * x2 - x1 * x1;               // >= 0 (Cauchy-Schwarz)
        a.mean[g * S + sp] = div_rn((unsigned __int128)x1, (unsigned __int128)n);
        a.var[g * S + sp] = div_rn((unsigned __int128)num, (unsigned __int128)n * (unsigned __int128)n);
    }
}

// the two-level sort by time: radix sort of the high 32 bits of the fp64
// pattern (4 digit passes instead of 8), then each run of equal high words
// sorted by the full pattern (CUB segmented sort; the runs are short)
__global__ void k_keys_hi(const double* __restrict__ t, ssa_u64 n, unsigned* __restrict__ hi,
                          unsigned* __restrict__ idx)
{
    for (ssa_u64 m = blockIdx.x * (ssa_u64)blockDim.x + threadIdx.x; m < n; m += (ssa_u64)gridDim.x * blockDim.x) {
        hi[m] = (unsigned)((ssa_u64)__double_as_longlong(__ldg(t + m)) >> 32);
        idx[m] = (unsigned)m;
    }
}

__global__ void k_keys_full(const double* __restrict__ t, const unsigned* __restrict__ hi2,
                            const unsigned* __restrict__ idx2, ssa_u64 n, ssa_u64* __restrict__ keys,
                            unsigned* __restrict__ head)
{
    for (ssa_u64 m = blockIdx.x * (ssa_u64)blockDim.x + threadIdx.x; m < n; m += (ssa_u64)gridDim.x * blockDim.x) {
        keys[m] = (ssa_u64)__double_as_longlong(__ldg(t + __ldg(idx2 + m)));
        head[m] = (m == 0 || __ldg(hi2 + m) != __ldg(hi2 + m - 1)) ? 1u : 0u;
    }
}

unsigned grid_for(ssa_u64 n)
{
    const ssa_u64 b = (n + 255) / 256;
    return (unsigned)(b < 148ull * 64 ? (b ? b : 1) : 148ull * 64);
}

struct Scratch {
    void* p = nullptr;
    cudaStream_t st = nullptr;
    ~Scratch()
    {
        if (p) cudaFreeAsync(p, st);
    }
    cudaError_t alloc(size_t b, cudaStream_t s)
    {
        st = s;
        return cudaMallocAsync(&p, b ? b : 1, s);
    }
};

}  // namespace

#define UCHK(x)                                   \
    do {                                          \
        cudaError_t e_ = (x);                     \
        if (e_ != cudaSuccess) return e_;         \
    } while (0)

__global__ void k_yflags(const ssa_u64* __restrict__ keys, ssa_u64 E, unsigned* __restrict__ f)
{
    for (ssa_u64 m = blockIdx.x * (ssa_u64)blockDim.x + threadIdx.x; m < E; m += (ssa_u64)gridDim.x * blockDim.x)
        f[m] = (m + 1 == E || keys[m] != keys[m + 1]) ? 1u : 0u;
}

// rows sorted by time: keys_out = the sorted fp64 patterns, perm_out = their rows
cudaError_t sort_by_time(const double* t, ssa_u64 NR, ssa_u64* keys_out, unsigned* perm_out, cudaStream_t st,
                         int* launches)
{
    const char* mode = getenv("SSA_UNION_SORT");                  // "64": one 64-bit radix sort (A/B)
    if (mode && !strcmp(mode, "64")) {
        Scratch keys, idx, temp;
        UCHK(keys.alloc(8 * NR, st));
        UCHK(idx.alloc(4 * NR, st));
        k_keys<<<grid_for(NR), 256, 0, st>>>(t, NR, (ssa_u64*)keys.p, (unsigned*)idx.p);
        UCHK(cudaGetLastError());
        size_t tb = 0;
        UCHK(cub::DeviceRadixSort::SortPairs(nullptr, tb, (const ssa_u64*)keys.p, keys_out, (const unsigned*)idx.p,
                                             perm_out, (int64_t)NR, 0, 64, st));
        UCHK(temp.alloc(tb, st));
        UCHK(cub::DeviceRadixSort::SortPairs(temp.p, tb, (const ssa_u64*)keys.p, keys_out, (const unsigned*)idx.p,
                                             perm_out, (int64_t)NR, 0, 64, st));
        *launches += 2;
        return cudaSuccess;
    }
    Scratch hi, hi2, idx, idx2, full, head, segb, nseg, temp, temp2, temp3;
    UCHK(hi.alloc(4 * NR, st));
    UCHK(hi2.alloc(4 * NR, st));
    UCHK(idx.alloc(4 * NR, st));
    UCHK(idx2.alloc(4 * NR, st));
    k_keys_hi<<<grid_for(NR), 256, 0, st>>>(t, NR, (unsigned*)hi.p, (unsigned*)idx.p);
    UCHK(cudaGetLastError());
    size_t tb = 0;
    UCHK(cub::DeviceRadixSort::SortPairs(nullptr, tb, (const unsigned*)hi.p, (unsigned*)hi2.p, (const unsigned*)idx.p,
                                         (unsigned*)idx2.p, (int64_t)NR, 0, 32, st));
    UCHK(temp.alloc(tb, st));
    UCHK(cub::DeviceRadixSort::SortPairs(temp.p, tb, (const unsigned*)hi.p, (unsigned*)hi2.p, (const unsigned*)idx.p,
                                         (unsigned*)idx2.p, (int64_t)NR, 0, 32, st));
    UCHK(full.alloc(8 * NR, st));
    UCHK(head.alloc(4 * NR, st));
    k_keys_full<<<grid_for(NR), 256, 0, st>>>(t, (const unsigned*)hi2.p, (const unsigned*)idx2.p, NR,
                                              (ssa_u64*)full.p, (unsigned*)head.p);
    UCHK(cudaGetLastError());
    // the runs of equal high words: their first rows, and NR closing the last
    UCHK(segb.alloc(4 * (NR + 1), st));
    UCHK(nseg.alloc(8, st));
    size_t fb = 0;
    cub::CountingInputIterator<unsigned> it(0);
    UCHK(cub::DeviceSelect::Flagged(nullptr, fb, it, (const unsigned*)head.p, (unsigned*)segb.p, (ssa_u64*)nseg.p,
                                    (int64_t)NR, st));
    UCHK(temp2.alloc(fb, st));
    UCHK(cub::DeviceSelect::Flagged(temp2.p, fb, it, (const unsigned*)head.p, (unsigned*)segb.p, (ssa_u64*)nseg.p,
                                    (int64_t)NR, st));
    ssa_u64 ns = 0;
    UCHK(cudaMemcpyAsync(&ns, nseg.p, 8, cudaMemcpyDeviceToHost, st));
    UCHK(cudaStreamSynchronize(st));
    const unsigned end = (unsigned)NR;
    UCHK(cudaMemcpyAsync((unsigned*)segb.p + ns, &end, 4, cudaMemcpyHostToDevice, st));
    const unsigned* sb = (const unsigned*)segb.p;
    size_t qb = 0;
    UCHK(cub::DeviceSegmentedSort::SortPairs(nullptr, qb, (const ssa_u64*)full.p, keys_out, (const unsigned*)idx2.p,
                                             perm_out, (int)NR, (int)ns, sb, sb + 1, st));
    UCHK(temp3.alloc(qb, st));
    UCHK(cub::DeviceSegmentedSort::SortPairs(temp3.p, qb, (const ssa_u64*)full.p, keys_out, (const unsigned*)idx2.p,
                                             perm_out, (int)NR, (int)ns, sb, sb + 1, st));
    *launches += 5;
    UCHK(cudaGetLastError());
    return cudaStreamSynchronize(st);                              // the host value `end` is read by the copy
}

cudaError_t ssa_union_reduce(ssa_union_args a, cudaStream_t st, ssa_u64* n_points, int* launches)
{
    const ssa_u64 E = a.E, NR = a.rows;
    Scratch keys2, idx2, yi, gst, tot;
    ssa_u64 D = 0;
    int horizon = 1;
    if (E > 0) {
        if (NR >= (1ull << 31)) return cudaErrorInvalidValue;      // row indices are 31-bit (+ a flag bit)
        UCHK(keys2.alloc(8 * NR, st));
        UCHK(idx2.alloc(4 * NR, st));
        // 1. sort by time (the +inf rows of unused reservations go last; the
        //    first E sorted rows are the events)
        UCHK(sort_by_time(a.rec_t, NR, (ssa_u64*)keys2.p, (unsigned*)idx2.p, st, launches));
        // 2. Y-point index of every event: exclusive count of the runs of equal
        //    times that end before it (in place over the run-end flags)
        UCHK(yi.alloc(4 * E, st));
        k_yflags<<<grid_for(E), 256, 0, st>>>((const ssa_u64*)keys2.p, E, (unsigned*)yi.p);
        ++*launches;
        UCHK(cudaGetLastError());
        size_t sb = 0;
        UCHK(cub::DeviceScan::ExclusiveSum(nullptr, sb, (unsigned*)yi.p, (unsigned*)yi.p, (int64_t)E, st));
        Scratch t2;
        UCHK(t2.alloc(sb, st));
        UCHK(cub::DeviceScan::ExclusiveSum(t2.p, sb, (unsigned*)yi.p, (unsigned*)yi.p, (int64_t)E, st));
        ++*launches;
        unsigned ylast = 0;
        ssa_u64 klast = 0;
        UCHK(cudaMemcpyAsync(&ylast, (const unsigned*)yi.p + (E - 1), 4, cudaMemcpyDeviceToHost, st));
        UCHK(cudaMemcpyAsync(&klast, (const ssa_u64*)keys2.p + (E - 1), 8, cudaMemcpyDeviceToHost, st));
        UCHK(cudaStreamSynchronize(st));
        D = (ssa_u64)ylast + 1;                                    // the last event ends a run
        double tlast = 0.0;
        memcpy(&tlast, &klast, 8);
        horizon = tlast < a.t_end ? 1 : 0;
    }
    // Y-points: 0, the D run ends, and the horizon unless an event sits on it
    const ssa_u64 NY = 1 + D + (ssa_u64)horizon;
    const ssa_u64 NX = (NY + a.kx - 1) / a.kx;
    *n_points = NX;
    if (NX > a.capacity) return cudaSuccess;                      // caller reports the required capacity
    // 3. warps of GW X-groups (one lane per group), tiles of WPB warps; the
    //    groups' accumulator rows and the warps' staging fit the shared memory
    const int S = a.S, U = a.U;
    const size_t grow = 8 * (size_t)row_stride(S), rows_budget = 80 * 1024;
    Geo G{};
    G.E = E; G.NY = NY; G.NX = NX; G.horizon = horizon;
    G.GW = (unsigned)std::min<size_t>(32, rows_budget / grow);
    if (G.GW < 1) return cudaErrorInvalidConfiguration;         // S in the thousands: the rows do not fit
    if (const char* h = getenv("SSA_UNION_GT"))                   // test hook: force small segments
        if (atoi(h) > 0 && (unsigned)atoi(h) < G.GW) G.GW = (unsigned)atoi(h);
    G.WPB = (int)std::max<size_t>(1, std::min<size_t>(4, rows_budget / (G.GW * grow)));
    G.BT = 512;
    if (const char* h = getenv("SSA_UNION_CH"))                   // test hook / tuning: events per batch
        if (atoi(h) > 0) G.BT = atoi(h);
    while (G.BT > 32 && G.WPB * stage_bytes(G.BT, U) > 64 * 1024) G.BT /= 2;
    const ssa_u64 TG = (ssa_u64)G.WPB * G.GW, tiles = (NX + TG - 1) / TG;
    if (tiles >= (1ull << 31)) return cudaErrorInvalidValue;
    const unsigned block = 32u * (unsigned)G.WPB;
    const size_t sm = TG * grow + 8 * (size_t)(G.WPB + 1) * 2 * S + (size_t)G.WPB * stage_bytes(G.BT, U);
    if (sm > 227 * 1024) return cudaErrorInvalidConfiguration;
    UCHK(gst.alloc(8 * (NX + 1), st));
    UCHK(tot.alloc(2 * 16 * tiles * (size_t)S + 4 * (tiles + 1), st));
    long long* agg = (long long*)tot.p;
    long long* incl = agg + tiles * 2 * S;
    unsigned* flags = (unsigned*)(incl + tiles * 2 * S);          // [tiles] + the ticket
    UCHK(cudaMemsetAsync(flags, 0, 4 * (tiles + 1), st));
    k_group_starts_init<<<grid_for(NX + 1), 256, 0, st>>>(E, NX, (ssa_u64*)gst.p);
    ++*launches;
    UCHK(cudaGetLastError());
    if (E > 0) {
        k_group_starts_scatter<<<grid_for(E), 256, 0, st>>>((const unsigned*)yi.p, E, a.kx, (ssa_u64*)gst.p);
        ++*launches;
    }
    UCHK(cudaFuncSetAttribute(k_union_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_union_pass<<<(unsigned)tiles, block, sm, st>>>(a, G, (const unsigned*)idx2.p, (const unsigned*)yi.p,
                                                     (const ssa_u64*)keys2.p, (const ssa_u64*)gst.p, agg, incl,
                                                     flags, flags + tiles);
    ++*launches;
    UCHK(cudaGetLastError());
    return cudaStreamSynchronize(st);
}

// --------------------------------------------------------------------------
// Stride-sampled trajectory output ("a
// 1:10 sampling (outputting 1 simulation point every 10)"): the points K1's
// stride-record variant appended (key = trajectory << 41 | seq, seq = 2k
// after event k, 0 initial, 2E+1 horizon; unused rows key ~0) are sorted by
// key and gathered into per-trajectory, time-ordered output rows.
namespace {

__global__ void k_iota(ssa_u64 n, unsigned* __restrict__ idx)
{
    for (ssa_u64 m = blockIdx.x * (ssa_u64)blockDim.x + threadIdx.x; m < n; m += (ssa_u64)gridDim.x * blockDim.x)
        idx[m] = (unsigned)m;
}

__global__ void k_count_valid(const ssa_u64* __restrict__ keys, ssa_u64 n, ssa_u64* __restrict__ valid)
{
    for (ssa_u64 m = blockIdx.x * (ssa_u64)blockDim.x + threadIdx.x; m < n; m += (ssa_u64)gridDim.x * blockDim.x)
        if (keys[m] != ~0ull && (m + 1 == n || keys[m + 1] == ~0ull)) *valid = m + 1;
}

__global__ void k_gather_points(const ssa_u64* __restrict__ keys, const unsigned* __restrict__ idx, ssa_u64 P, int S,
                                const double* __restrict__ t, const int* __restrict__ st, ssa_u64 traj_base,
                                unsigned* __restrict__ o_traj, ssa_u64* __restrict__ o_event,
                                double* __restrict__ o_time, int* __restrict__ o_state)
{
    for (ssa_u64 m = blockIdx.x * (ssa_u64)blockDim.x + threadIdx.x; m < P; m += (ssa_u64)gridDim.x * blockDim.x) {
        const ssa_u64 k = keys[m], src = idx[m];
        o_traj[m] = (unsigned)(traj_base + (k >> 41));
        o_event[m] = (k & ((1ull << 41) - 1)) >> 1;
        o_time[m] = t[src];
        for (int s = 0; s < S; ++s) o_state[m * S + s] = st[src * S + s];
    }
}

}  // namespace

cudaError_t ssa_points_gather(const ssa_u64* keys_in, const double* t, const int* states, ssa_u64 rows, int S,
                              ssa_u64 capacity, unsigned* o_traj, ssa_u64* o_event, double* o_time, int* o_state,
                              ssa_u64* n_points, cudaStream_t st, int* launches)
{
    *n_points = 0;
    if (rows == 0) return cudaSuccess;
    Scratch keys2, idx, idx2, temp, valid;
    UCHK(keys2.alloc(8 * rows, st));
    UCHK(idx.alloc(4 * rows, st));
    UCHK(idx2.alloc(4 * rows, st));
    UCHK(valid.alloc(8, st));
    UCHK(cudaMemsetAsync(valid.p, 0, 8, st));
    k_iota<<<grid_for(rows), 256, 0, st>>>(rows, (unsigned*)idx.p);
    size_t tb = 0;
    UCHK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys_in, (ssa_u64*)keys2.p, (const unsigned*)idx.p,
                                         (unsigned*)idx2.p, (int64_t)rows, 0, 64, st));
    UCHK(temp.alloc(tb, st));
    UCHK(cub::DeviceRadixSort::SortPairs(temp.p, tb, keys_in, (ssa_u64*)keys2.p, (const unsigned*)idx.p,
                                         (unsigned*)idx2.p, (int64_t)rows, 0, 64, st));
    k_count_valid<<<grid_for(rows), 256, 0, st>>>((const ssa_u64*)keys2.p, rows, (ssa_u64*)valid.p);
    *launches += 3;
    ssa_u64 P = 0;
    UCHK(cudaMemcpyAsync(&P, valid.p, 8, cudaMemcpyDeviceToHost, st));
    UCHK(cudaStreamSynchronize(st));
    *n_points = P;
    if (P > capacity) return cudaSuccess;
    k_gather_points<<<grid_for(P), 256, 0, st>>>((const ssa_u64*)keys2.p, (const unsigned*)idx2.p, P, S, t, states, 0,
                                                 o_traj, o_event, o_time, o_state);
    ++*launches;
    UCHK(cudaGetLastError());
    return cudaStreamSynchronize(st);
}
