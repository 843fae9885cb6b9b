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
//   2. per sorted event, the exact changes of sum x and sum x^2 of the species
//      the reaction touches (d1 = nu, d2 = 2 x nu + nu^2 from the recorded
//      pre-event count), as dense per-species int64 columns;
//   3. inclusive scans of those columns: the ensemble sums just after each
//      event, exact in integers;
//   4. the last event of every run of equal times is a Y-point (equal union
//      times collapse into one slice); Y-points are 0, those events, and the
//      horizon;
//   5. one thread per X-group of k_x Y-points: mean time (left-to-right sum),
//      exact sums, mean = S1/n, population variance = (n S2 - S1^2)/n^2.
// Every pass is a streaming pass over HBM (the path is bandwidth-bound).
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>
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

// dense deltas of sum x (d1) and sum x^2 (d2) per species, in sorted order
__global__ void k_deltas(const unsigned* __restrict__ perm, ssa_u64 E, const int* __restrict__ rec_j,
                         const int* __restrict__ rec_pre, int U, const int* __restrict__ nu_sp,
                         const int* __restrict__ nu_d, long long* __restrict__ d1, long long* __restrict__ d2)
{
    for (ssa_u64 m = blockIdx.x * (ssa_u64)blockDim.x + threadIdx.x; m < E; m += (ssa_u64)gridDim.x * blockDim.x) {
        const ssa_u64 ev = perm[m];
        const int j = rec_j[ev];
        for (int q = 0; q < U; ++q) {
            const int s = nu_sp[j * U + q];
            if (s < 0) continue;
            const long long v = nu_d[j * U + q];
            const long long x = rec_pre[ev * U + q];
            d1[(ssa_u64)s * E + m] = v;
            d2[(ssa_u64)s * E + m] = 2 * x * v + v * v;
        }
    }
}

__global__ void k_flags(const ssa_u64* __restrict__ keys, ssa_u64 E, unsigned char* __restrict__ f)
{
    for (ssa_u64 m = blockIdx.x * (ssa_u64)blockDim.x + threadIdx.x; m < E; m += (ssa_u64)gridDim.x * blockDim.x)
        f[m] = (m + 1 == E || keys[m] != keys[m + 1]) ? 1 : 0;
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

__global__ void k_xgroups(ssa_union_args a, const ssa_u64* __restrict__ keys, const unsigned* __restrict__ ypos,
                          ssa_u64 D, ssa_u64 NY, const long long* __restrict__ p1, const long long* __restrict__ p2)
{
    const ssa_u64 g = blockIdx.x * (ssa_u64)blockDim.x + threadIdx.x;
    const ssa_u64 NX = (NY + a.kx - 1) / a.kx;
    if (g >= NX) return;
    const ssa_u64 y0 = g * a.kx, y1 = (y0 + a.kx < NY) ? y0 + a.kx : NY;
    double tsum = 0.0;
    for (ssa_u64 y = y0; y < y1; ++y) {
        double ty;
        if (y == 0) ty = 0.0;
        else if (y <= D) ty = __longlong_as_double((long long)keys[ypos[y - 1]]);
        else ty = a.t_end;
        tsum = __dadd_rn(tsum, ty);
    }
    const double m = (double)(y1 - y0);
    a.times[g] = __ddiv_rn(tsum, m);
    const long long n = (long long)a.k * (long long)(y1 - y0);
    a.count[g] = (double)n;
    for (int s = 0; s < a.S; ++s) {
        long long x1 = 0;
        __int128 x2 = 0;
        for (ssa_u64 y = y0; y < y1; ++y) {
            long long s1 = a.s0[s];
            long long s2 = a.s0sq[s];
            if (y >= 1 && a.E > 0) {
                const ssa_u64 pos = (y <= D) ? ypos[y - 1] : a.E - 1;    // horizon: after every event
                s1 += p1[(ssa_u64)s * a.E + pos];
                s2 += p2[(ssa_u64)s * a.E + pos];
            }
            x1 += s1;
            x2 += (__int128)s2;
        }
        const __int128 num = (__int128)n * x2 - (__int128)x1 * x1;     // >= 0 (Cauchy-Schwarz)
        a.mean[g * a.S + s] = ratio_rn((unsigned __int128)x1, (unsigned __int128)n);
        a.var[g * a.S + s] = ratio_rn((unsigned __int128)num, (unsigned __int128)n * (unsigned __int128)n);
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

cudaError_t ssa_union_reduce(ssa_union_args a, cudaStream_t st, ssa_u64* n_points, int* launches)
{
    const ssa_u64 E = a.E, NR = a.rows;
    Scratch keys, keys2, idx, idx2, d1, d2, flags, ypos, nsel, temp;
    ssa_u64 D = 0;
    if (E > 0) {
        UCHK(keys.alloc(8 * NR, st));
        UCHK(keys2.alloc(8 * NR, st));
        UCHK(idx.alloc(4 * NR, st));
        UCHK(idx2.alloc(4 * NR, st));
        k_keys<<<grid_for(NR), 256, 0, st>>>(a.rec_t, NR, (ssa_u64*)keys.p, (unsigned*)idx.p);
        ++*launches;
        // 1. sort by time (the +inf rows of unused reservations go last; the
        //    first E sorted rows are the events)
        size_t tb = 0;
        UCHK(cub::DeviceRadixSort::SortPairs(nullptr, tb, (const ssa_u64*)keys.p, (ssa_u64*)keys2.p,
                                             (const unsigned*)idx.p, (unsigned*)idx2.p, (int64_t)NR, 0, 64, st));
        UCHK(temp.alloc(tb, st));
        UCHK(cub::DeviceRadixSort::SortPairs(temp.p, tb, (const ssa_u64*)keys.p, (ssa_u64*)keys2.p,
                                             (const unsigned*)idx.p, (unsigned*)idx2.p, (int64_t)NR, 0, 64, st));
        ++*launches;
        const ssa_u64* sk = (const ssa_u64*)keys2.p;
        const unsigned* perm = (const unsigned*)idx2.p;
        // 2. dense deltas
        UCHK(d1.alloc(8 * E * (size_t)a.S, st));
        UCHK(d2.alloc(8 * E * (size_t)a.S, st));
        UCHK(cudaMemsetAsync(d1.p, 0, 8 * E * (size_t)a.S, st));
        UCHK(cudaMemsetAsync(d2.p, 0, 8 * E * (size_t)a.S, st));
        k_deltas<<<grid_for(E), 256, 0, st>>>(perm, E, a.rec_j, a.rec_pre, a.U, a.nu_sp, a.nu_d, (long long*)d1.p,
                                             (long long*)d2.p);
        ++*launches;
        // 3. per-species inclusive scans (in place)
        for (int s = 0; s < a.S; ++s) {
            long long* c1 = (long long*)d1.p + (size_t)s * E;
            long long* c2 = (long long*)d2.p + (size_t)s * E;
            size_t sb = 0;
            UCHK(cub::DeviceScan::InclusiveSum(nullptr, sb, c1, c1, (int64_t)E, st));
            Scratch t2;
            UCHK(t2.alloc(sb, st));
            UCHK(cub::DeviceScan::InclusiveSum(t2.p, sb, c1, c1, (int64_t)E, st));
            UCHK(cub::DeviceScan::InclusiveSum(t2.p, sb, c2, c2, (int64_t)E, st));
            *launches += 2;
        }
        // 4. Y-points: the last event of every run of equal times
        UCHK(flags.alloc(E, st));
        UCHK(ypos.alloc(4 * E, st));
        UCHK(nsel.alloc(8, st));
        k_flags<<<grid_for(E), 256, 0, st>>>(sk, E, (unsigned char*)flags.p);
        ++*launches;
        size_t fb = 0;
        cub::CountingInputIterator<unsigned> it(0);
        UCHK(cub::DeviceSelect::Flagged(nullptr, fb, it, (const unsigned char*)flags.p, (unsigned*)ypos.p,
                                        (ssa_u64*)nsel.p, (int64_t)E, st));
        Scratch t3;
        UCHK(t3.alloc(fb, st));
        UCHK(cub::DeviceSelect::Flagged(t3.p, fb, it, (const unsigned char*)flags.p, (unsigned*)ypos.p,
                                        (ssa_u64*)nsel.p, (int64_t)E, st));
        ++*launches;
        UCHK(cudaMemcpyAsync(&D, nsel.p, 8, cudaMemcpyDeviceToHost, st));
        double tlast = 0.0;
        ssa_u64 klast = 0;
        UCHK(cudaMemcpyAsync(&klast, sk + (E - 1), 8, cudaMemcpyDeviceToHost, st));
        UCHK(cudaStreamSynchronize(st));
        memcpy(&tlast, &klast, 8);
        const ssa_u64 NY = 1 + D + (tlast < a.t_end ? 1 : 0);
        const ssa_u64 NX = (NY + a.kx - 1) / a.kx;
        *n_points = NX;
        if (NX > a.capacity) return cudaSuccess;                  // caller reports the required capacity
        k_xgroups<<<(unsigned)((NX + 255) / 256), 256, 0, st>>>(a, sk, (const unsigned*)ypos.p, D, NY,
                                                                (const long long*)d1.p, (const long long*)d2.p);
        ++*launches;
        UCHK(cudaGetLastError());
        return cudaStreamSynchronize(st);
    }
    // no event at all: the two slices 0 and t_end hold x0
    const ssa_u64 NY = 2, NX = (NY + a.kx - 1) / a.kx;
    *n_points = NX;
    if (NX > a.capacity) return cudaSuccess;
    k_xgroups<<<1, 256, 0, st>>>(a, nullptr, nullptr, 0, NY, nullptr, nullptr);
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
