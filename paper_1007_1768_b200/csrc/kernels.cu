// kernels.cu -- nvcc-compiled kernels of the ensemble-SSA hot path (sm_100a):
//   K2  ssa_k2<P>      one trajectory per warp (networks with hundreds of
//                      reactions): lane-contiguous propensity blocks, a
//                      Hillis-Steele warp scan, ballot/ffs selection, state in
//                      shared memory, RNG amortised 32 events per lane
//                      (north_star (a)), order R13.
//   K3  ssa_tree_leaf  canonical-tree Welford reduction of a chunk's staged
//                      grid samples (a9, no atomics: north_star (d)).
//   K4  ssa_tree_merge merge of partial roots (tiles -> chunk -> shard -> GPUs)
//       ssa_finalize   mean, population variance = M2/n (a10).
// K1 (thread path) is model-specialised and compiled by NVRTC (jit.cpp).
#include <cuda_runtime.h>
#include <stdint.h>

#include "ssa_device.cuh"
#include "ssa_kernels.h"

__constant__ double k2_plog[14] = SSA_PLOG_COEF_INIT;

// =========================================================================
// K2: warp per trajectory
// =========================================================================
// Propensities live in shared memory, laid out [q][lane] for the lane-
// contiguous blocks j = lane*P + q (conflict-free), and after each event only
// the reactions that read a changed species are recomputed (dependency graph,
// a_j is a pure function of x, so the cached values are
// bit-identical to a full recompute).  The summation order is the warp32
// order of DESIGN.md §2.
//
// Packed reaction word (see ensure_k2 in runtime.cu):
//   bits [0,2) n_reac; term q: species [2+16q, 16+16q), coef [16+16q, 18+16q);
//   bits [50,64) modifier species (0x3FFF = none).
struct k2_rx {
    ssa_u64 pk;
    double rate;
    double modc;
};

// C(x, m) for m in {1, 2}; m == 3 is rare and branches.
static __device__ __forceinline__ double k2_factor(double x, int m)
{
    const double x1 = __dmul_rn(x, __dadd_rn(x, -1.0));
    double f = (m == 1) ? x : __dmul_rn(x1, 0.5);
    if (m == 3) f = __ddiv_rn(__dmul_rn(x1, __dadd_rn(x, -2.0)), 6.0);
    return f;
}

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
    return (n == 0) ? k : __dmul_rn(k, h);
}

size_t ssa_k2_smem_bytes(int S, int R, int P, int n_ent, int n_dep, int block)
{
    const size_t warps = (size_t)(block / 32);
    return sizeof(k2_rx) * (size_t)R + sizeof(double) * (size_t)S                    // tables, x0
           + warps * sizeof(double) * ((size_t)S + 32 * (size_t)P)                    // x, a per warp
           + sizeof(int) * ((size_t)R + 1 + n_ent + (size_t)S + 1 + n_dep);           // nu, dep CSR
}

template <int PMAX>
__global__ void __launch_bounds__(SSA_K2_BLOCK, 4) ssa_k2(const ssa_k2_params P)
{
    extern __shared__ __align__(16) unsigned char k2_smem_raw[];
    const int S = P.S, R = P.R, Pl = P.P;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const unsigned FULL = 0xffffffffu;
    // shared layout: rx[R] | x0[S] | (x[S] | a[32 P]) per warp | nu_off[R+1] | nu_ent | dep_off[S+1] | dep_ent
    k2_rx* rx = (k2_rx*)k2_smem_raw;
    double* x0 = (double*)(rx + R);
    double* wbase = x0 + S;
    double* x = wbase + (size_t)warp * (S + 32 * Pl);
    double* a = x + S;                                   // a[q*32 + l] = propensity of j = l*P + q
    int* nu_off = (int*)(wbase + (size_t)nwarps * (S + 32 * Pl));
    int* nu_ent = nu_off + (R + 1);
    int* dep_off = nu_ent + P.n_ent;
    int* dep_ent = dep_off + (S + 1);
    for (int i = threadIdx.x; i < R; i += blockDim.x) {
        k2_rx q;
        q.pk = P.pk[i]; q.rate = P.rate[i]; q.modc = P.modc[i];
        rx[i] = q;
    }
    for (int i = threadIdx.x; i < S; i += blockDim.x) x0[i] = P.x0[i];
    for (int i = threadIdx.x; i <= R; i += blockDim.x) nu_off[i] = P.nu_off[i];
    for (int i = threadIdx.x; i < P.n_ent; i += blockDim.x) nu_ent[i] = P.nu_ent[i];
    for (int i = threadIdx.x; i <= S; i += blockDim.x) dep_off[i] = P.dep_off[i];
    for (int i = threadIdx.x; i < P.n_dep; i += blockDim.x) dep_ent[i] = P.dep_ent[i];
    __syncthreads();

    const double INF = __longlong_as_double(0x7FF0000000000000ll);
    const double dt = P.dt;
    const long long K = P.K;
    const ssa_u64 G = (ssa_u64)K + 1;
    ssa_u64 my_events = 0, my_ties = 0;

    for (;;) {
        ssa_u64 rel = 0;
        if (lane == 0) rel = atomicAdd(P.work, 1ull);
        rel = __shfl_sync(FULL, rel, 0);
        if (rel >= P.n_ids) break;
        const ssa_u64 id = P.id_begin + rel;
        const long long slot = P.n_dump ? ssa_dump_slot(P.dump_ids, P.n_dump, id) : -1ll;
        for (int s = lane; s < S; s += 32) x[s] = x0[s];
        __syncwarp();
        // a3 at the initial state: every propensity of this lane's block
#pragma unroll
        for (int q = 0; q < PMAX; ++q) {
            if (q < Pl) {
                const int j = lane * Pl + q;
                a[q * 32 + lane] = (j < R) ? k2_propensity(rx[j], x) : 0.0;
            }
        }
        __syncwarp();

        double t = 0.0, s_next = 0.0;
        ssa_u64 e = 0, hash = SSA_FNV_OFFSET, ties = 0;
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
                Ec = -ssa_plog(ssa_u53(o.o1, o.o0), k2_plog);
                U2c = ssa_u53(o.o3, o.o2);
            }
            // a4: lane sum (sequential over the lane's block), then warp scan
            double L = 0.0;
#pragma unroll
            for (int q = 0; q < PMAX; ++q)
                if (q < Pl) L = __dadd_rn(L, a[q * 32 + lane]);
            double v = L;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double y = __shfl_up_sync(FULL, v, o);
                if (lane >= o) v = __dadd_rn(y, v);
            }
            const double a0 = __shfl_sync(FULL, v, 31);
            // a5
            const int src = (int)(e & 31ull);
            const double E = __shfl_sync(FULL, Ec, src);
            const double u2 = __shfl_sync(FULL, U2c, src);
            double tn;
            if (a0 > 0.0 && a0 < INF) {
                tn = __dadd_rn(t, ssa_div_tau(E, a0));
            } else if (a0 == 0.0) {
                tn = INF;
                absorbed = 1;
            } else {
                status = 1;
                int bad = R;   // first reaction with a non-finite propensity
#pragma unroll
                for (int q = PMAX - 1; q >= 0; --q)
                    if (q < Pl && lane * Pl + q < R && !(fabs(a[q * 32 + lane]) < INF)) bad = lane * Pl + q;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) bad = min(bad, __shfl_xor_sync(FULL, bad, o));
                err_r = bad < R ? bad : -1;
                break;
            }
            // a6 (warp-uniform)
            if (tn > s_next) {
                do {
                    const double tol = __dmul_rn(1e-9, s_next);
                    const bool near = (tn < INF && fabs(__dadd_rn(tn, -s_next)) <= tol) ||
                                      (e > 0 && fabs(__dadd_rn(t, -s_next)) <= tol);
                    ties += near ? 1 : 0;
                    int ovf = 0;
                    for (int s = lane; s < S; s += 32) {
                        const double xv = x[s];
                        ovf |= (xv > 2147483647.0) ? 1 : 0;
                        P.staging[((ssa_u64)k * S + s) * P.stride + rel] = (int)xv;
                        if (slot >= 0) P.dump_states[((ssa_u64)slot * G + (ssa_u64)k) * S + s] = (int)xv;
                    }
                    if (__any_sync(FULL, ovf)) status = 2;
                    if (slot >= 0 && lane == 0) {
                        P.dump_e[(ssa_u64)slot * G + (ssa_u64)k] = e;
                        P.dump_t[(ssa_u64)slot * G + (ssa_u64)k] = (e > 0) ? t : 0.0;
                    }
                    ++k;
                    s_next = (k <= K) ? __dmul_rn((double)k, dt) : INF;
                } while (tn > s_next);
                if (k > K) break;
            }
            // a7: lane* = first lane whose inclusive prefix exceeds r
            const double r = __dmul_rn(u2, a0);
            const unsigned mask = __ballot_sync(FULL, v > r);
            const int ls = __ffs(mask) - 1;
            const double vprev = __shfl_up_sync(FULL, v, 1);
            int j = -1;
            if (lane == ls) {
                double p = (lane > 0) ? vprev : 0.0;
                for (int q = 0; q < Pl; ++q) {
                    p = __dadd_rn(p, a[q * 32 + lane]);
                    if (p > r) { j = lane * Pl + q; break; }
                }
                if (j < 0)
                    for (int q = Pl - 1; q >= 0; --q)
                        if (a[q * 32 + lane] > 0.0) { j = lane * Pl + q; break; }
            }
            j = __shfl_sync(FULL, j, ls);
            if (j < 0) {
                // rounding fallback: last positive propensity in an earlier lane
                int lp = -1;
                for (int q = 0; q < Pl; ++q)
                    if (a[q * 32 + lane] > 0.0) lp = lane * Pl + q;
                const unsigned m2 = __ballot_sync(FULL, lp >= 0 && lane < ls);
                j = __shfl_sync(FULL, lp, 31 - __clz(m2));
            }
            // a8: state update
            const int nb = nu_off[j], ne = nu_off[j + 1];
            for (int q = nb + lane; q < ne; q += 32) {
                const int ent = nu_ent[q];
                const int sp = ent & 0xFFFF;
                x[sp] = __dadd_rn(x[sp], (double)(ent >> 16));   // arithmetic shift: signed delta
            }
            __syncwarp();
            // a3 for the reactions that read a changed species (lane t takes
            // the t-th entry of the concatenated dependency lists)
            int T = 0;
            for (int q = nb; q < ne; ++q) {
                const int sp = nu_ent[q] & 0xFFFF;
                T += dep_off[sp + 1] - dep_off[sp];
            }
            for (int base = 0; base < T; base += 32) {
                int rem = base + lane, jj = -1;
                for (int q = nb; q < ne; ++q) {
                    const int sp = nu_ent[q] & 0xFFFF;
                    const int o = dep_off[sp], len = dep_off[sp + 1] - o;
                    if (rem >= 0 && rem < len) jj = dep_ent[o + rem];
                    rem -= len;
                }
                if (jj >= 0) {
                    const int l = jj / Pl, q = jj - l * Pl;
                    a[q * 32 + l] = k2_propensity(rx[jj], x);
                }
            }
            __syncwarp();
            t = tn;
            ++e;
            hash = (hash ^ (ssa_u64)j) * SSA_FNV_PRIME;
        }
        __syncwarp();
        if (lane == 0) {
            my_events += e;
            my_ties += ties;
            if (slot >= 0) {
                ssa_dev_summary sm;
                sm.events = e; sm.hash = hash; sm.t_last = t; sm.near_ties = ties;
                sm.absorbed = absorbed; sm.status = status == 1 ? 3 : (status == 2 ? 4 : 0);
                sm.err_reaction = err_r; sm.pad = 0;
                P.dump_sum[slot] = sm;
            }
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

static const void* k2_fn(int pmax)
{
    switch (pmax) {
    case 1: return (const void*)ssa_k2<1>;
    case 2: return (const void*)ssa_k2<2>;
    case 4: return (const void*)ssa_k2<4>;
    case 8: return (const void*)ssa_k2<8>;
    case 16: return (const void*)ssa_k2<16>;
    default: return nullptr;
    }
}

cudaError_t ssa_k2_launch(const ssa_k2_params& p, int grid, int block, cudaStream_t st)
{
    const size_t smem = ssa_k2_smem_bytes(p.S, p.R, p.P, p.n_ent, p.n_dep, block);
    const void* fn = k2_fn(p.PMAX);
    if (!fn) return cudaErrorInvalidValue;
    cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    void* args[] = {(void*)&p};
    return cudaLaunchKernel(fn, dim3(grid), dim3(block), args, smem, st);
}

int ssa_k2_max_blocks_per_sm(int pmax, int block, size_t smem)
{
    int n = 0;
    const void* fn = k2_fn(pmax);
    if (!fn) return 0;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, block, smem) != cudaSuccess) return 0;
    return n;
}

// =========================================================================
// K3/K4: canonical-tree Welford reduction (no atomics)
// =========================================================================
// One block reduces SSA_TREE_SPAN = 8 * SSA_TREE_BLOCK consecutive leaves of
// one row (a (k, s) cell) into one partial: a thread folds 8 adjacent leaves
// as a perfect tree, warps combine adjacent subtrees with shuffles at offsets
// 1..16, and the 8 warps combine in shared memory -- every level merges two
// adjacent, equal-size, aligned subtrees (lower ids on the left), so the
// composition over passes is the perfect binary tree over the ids (R26).
// Leaves past `count` are empty (n = 0), the identity of the merge.
static __device__ __forceinline__ ssa_welford tree_block(ssa_welford w)
{
    __shared__ ssa_welford sh[SSA_TREE_BLOCK / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        ssa_welford b;
        b.n = __shfl_down_sync(0xffffffffu, w.n, o);
        b.mean = __shfl_down_sync(0xffffffffu, w.mean, o);
        b.m2 = __shfl_down_sync(0xffffffffu, w.m2, o);
        if ((lane & (2 * o - 1)) == 0) w = ssa_welford_merge(w, b);
    }
    if (lane == 0) sh[warp] = w;
    __syncthreads();
    if (threadIdx.x == 0) {
        ssa_welford v[SSA_TREE_BLOCK / 32];
#pragma unroll
        for (int i = 0; i < SSA_TREE_BLOCK / 32; ++i) v[i] = sh[i];
#pragma unroll
        for (int o = 1; o < SSA_TREE_BLOCK / 32; o <<= 1)
#pragma unroll
            for (int i = 0; i + o < SSA_TREE_BLOCK / 32; i += 2 * o) v[i] = ssa_welford_merge(v[i], v[i + o]);
        w = v[0];
    }
    return w;
}

static __device__ __forceinline__ ssa_welford fold8(ssa_welford v[8])
{
    v[0] = ssa_welford_merge(v[0], v[1]);
    v[2] = ssa_welford_merge(v[2], v[3]);
    v[4] = ssa_welford_merge(v[4], v[5]);
    v[6] = ssa_welford_merge(v[6], v[7]);
    v[0] = ssa_welford_merge(v[0], v[2]);
    v[4] = ssa_welford_merge(v[4], v[6]);
    return ssa_welford_merge(v[0], v[4]);
}

// Full tiles (no empty leaf): every merge joins two full subtrees of equal
// size h (a power of two), where the divisions of the Chan merge are exact --
// n_B / n = 1/2 and (n_A n_B) / n = h/2 -- so the merge reduces to
//   d = m_B - m_A;  m = m_A + d * 0.5;  M2 = (M2_A + M2_B) + (d * d) * (h/2)
// with bitwise the same result as ssa_welford_merge (R26), and no division.
// This keeps K3 at HBM speed instead of FP64-division bound.
static __device__ __forceinline__ void wf_merge_full(double& mA, double& m2A, double mB, double m2B, double half_h)
{
    const double d = __dadd_rn(mB, -mA);
    mA = __dadd_rn(mA, __dmul_rn(d, 0.5));
    m2A = __dadd_rn(__dadd_rn(m2A, m2B), __dmul_rn(__dmul_rn(d, d), half_h));
}

static __device__ __forceinline__ void tree_block_full(const int4 q0, const int4 q1, double& mean, double& m2)
{
    __shared__ double shm[SSA_TREE_BLOCK / 32], shq[SSA_TREE_BLOCK / 32];
    // 8 adjacent leaves per thread: levels h = 1, 2, 4
    double m[8] = {(double)q0.x, (double)q0.y, (double)q0.z, (double)q0.w,
                   (double)q1.x, (double)q1.y, (double)q1.z, (double)q1.w};
    double v[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    wf_merge_full(m[0], v[0], m[1], v[1], 0.5);
    wf_merge_full(m[2], v[2], m[3], v[3], 0.5);
    wf_merge_full(m[4], v[4], m[5], v[5], 0.5);
    wf_merge_full(m[6], v[6], m[7], v[7], 0.5);
    wf_merge_full(m[0], v[0], m[2], v[2], 1.0);
    wf_merge_full(m[4], v[4], m[6], v[6], 1.0);
    wf_merge_full(m[0], v[0], m[4], v[4], 2.0);
    double mm = m[0], vv = v[0];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // warp levels: subtrees of 8*o leaves, h/2 = 4*o
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double mb = __shfl_down_sync(0xffffffffu, mm, o);
        const double vb = __shfl_down_sync(0xffffffffu, vv, o);
        if ((lane & (2 * o - 1)) == 0) wf_merge_full(mm, vv, mb, vb, 4.0 * o);
    }
    if (lane == 0) { shm[warp] = mm; shq[warp] = vv; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a[SSA_TREE_BLOCK / 32], b[SSA_TREE_BLOCK / 32];
#pragma unroll
        for (int i = 0; i < SSA_TREE_BLOCK / 32; ++i) { a[i] = shm[i]; b[i] = shq[i]; }
        // block levels: subtrees of 256*o leaves, h/2 = 128*o
#pragma unroll
        for (int o = 1; o < SSA_TREE_BLOCK / 32; o <<= 1)
#pragma unroll
            for (int i = 0; i + o < SSA_TREE_BLOCK / 32; i += 2 * o) wf_merge_full(a[i], b[i], a[i + o], b[i + o], 128.0 * o);
        mean = a[0];
        m2 = b[0];
    }
}

// Full tiles only (launched over the first count / SPAN tiles of each row):
// every thread issues the loads of its 8 leaves in TWO adjacent tiles before
// reducing either, so each thread keeps 64 B in flight (the kernel is HBM
// bound); no general-path code, so it stays small in registers.
__global__ void __launch_bounds__(SSA_TREE_BLOCK, 4) ssa_tree_leaf_full(const int* __restrict__ staging,
                                                                       ssa_u64 stride, ssa_u64 n_full,
                                                                       ssa_u64 rows, ssa_tree_out out)
{
    const ssa_u64 row = (ssa_u64)blockIdx.y + 65535ull * blockIdx.z;
    if (row >= rows) return;
    const ssa_u64 t0 = 2ull * blockIdx.x;                 // first tile of this block
    const int* src = staging + row * stride + (ssa_u64)threadIdx.x * 8;
    const bool two = t0 + 1 < n_full;
    const int4 a0 = __ldcs(reinterpret_cast<const int4*>(src + t0 * SSA_TREE_SPAN));
    const int4 a1 = __ldcs(reinterpret_cast<const int4*>(src + t0 * SSA_TREE_SPAN + 4));
    int4 b0 = make_int4(0, 0, 0, 0), b1 = b0;
    if (two) {
        b0 = __ldcs(reinterpret_cast<const int4*>(src + (t0 + 1) * SSA_TREE_SPAN));
        b1 = __ldcs(reinterpret_cast<const int4*>(src + (t0 + 1) * SSA_TREE_SPAN + 4));
    }
    double mean = 0.0, m2 = 0.0;
    tree_block_full(a0, a1, mean, m2);
    if (threadIdx.x == 0) {
        const ssa_u64 o = row * out.row_stride + t0 * out.elem_stride + out.offset;
        out.n[o] = (double)SSA_TREE_SPAN; out.mean[o] = mean; out.m2[o] = m2;
    }
    if (two) {
        __syncthreads();                                   // shared scratch of tree_block_full reused
        tree_block_full(b0, b1, mean, m2);
        if (threadIdx.x == 0) {
            const ssa_u64 o = row * out.row_stride + (t0 + 1) * out.elem_stride + out.offset;
            out.n[o] = (double)SSA_TREE_SPAN; out.mean[o] = mean; out.m2[o] = m2;
        }
    }
}

// leaves: staging row r = blockIdx.y (+ 65535 * blockIdx.z), ids [0, count);
// blocks start at tile `first` (the tiles before it are full and reduced by
// ssa_tree_leaf_full)
__global__ void __launch_bounds__(SSA_TREE_BLOCK) ssa_tree_leaf(const int* __restrict__ staging, ssa_u64 stride,
                                                                ssa_u64 count, ssa_u64 rows, ssa_u64 first,
                                                                ssa_tree_out out)
{
    const ssa_u64 row = (ssa_u64)blockIdx.y + 65535ull * blockIdx.z;
    if (row >= rows) return;
    const ssa_u64 tile = first + blockIdx.x;
    const ssa_u64 base = tile * SSA_TREE_SPAN + (ssa_u64)threadIdx.x * 8;
    const int* src = staging + row * stride;
    ssa_welford v[8];
    if (base + 8 <= count && (((uintptr_t)(src + base)) & 15) == 0) {
        const int4 q0 = *reinterpret_cast<const int4*>(src + base);
        const int4 q1 = *reinterpret_cast<const int4*>(src + base + 4);
        v[0] = ssa_welford_leaf(q0.x); v[1] = ssa_welford_leaf(q0.y);
        v[2] = ssa_welford_leaf(q0.z); v[3] = ssa_welford_leaf(q0.w);
        v[4] = ssa_welford_leaf(q1.x); v[5] = ssa_welford_leaf(q1.y);
        v[6] = ssa_welford_leaf(q1.z); v[7] = ssa_welford_leaf(q1.w);
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            v[i] = (base + i < count) ? ssa_welford_leaf(src[base + i]) : ssa_welford_empty();
    }
    ssa_welford w = tree_block(fold8(v));
    if (threadIdx.x == 0) {
        const ssa_u64 o = row * out.row_stride + tile * out.elem_stride + out.offset;
        out.n[o] = w.n; out.mean[o] = w.mean; out.m2[o] = w.m2;
    }
}

// partials: element (row, i) at in.{n,mean,m2}[row*in.row_stride + i*in.elem_stride], i < count
__global__ void __launch_bounds__(SSA_TREE_BLOCK) ssa_tree_merge(const ssa_tree_in in, ssa_u64 count, ssa_u64 rows,
                                                                 ssa_tree_out out)
{
    const ssa_u64 row = (ssa_u64)blockIdx.y + 65535ull * blockIdx.z;
    if (row >= rows) return;
    const ssa_u64 base = (ssa_u64)blockIdx.x * SSA_TREE_SPAN + (ssa_u64)threadIdx.x * 8;
    ssa_welford v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (base + i < count) {
            const ssa_u64 a = row * in.row_stride + (base + i) * in.elem_stride;
            v[i].n = in.n[a]; v[i].mean = in.mean[a]; v[i].m2 = in.m2[a];
        } else {
            v[i] = ssa_welford_empty();
        }
    }
    ssa_welford w = tree_block(fold8(v));
    if (threadIdx.x == 0) {
        const ssa_u64 o = row * out.row_stride + (ssa_u64)blockIdx.x * out.elem_stride + out.offset;
        out.n[o] = w.n; out.mean[o] = w.mean; out.m2[o] = w.m2;
    }
}

// root (n, mean, m2) per cell -> mean, var = M2/n, m2, count
__global__ void ssa_finalize(const double* __restrict__ n, const double* __restrict__ mean,
                             const double* __restrict__ m2, ssa_u64 cells, double* o_mean, double* o_var,
                             double* o_m2, double* o_count)
{
    const ssa_u64 i = (ssa_u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cells) return;
    const double nn = n[i];
    if (o_mean) o_mean[i] = nn > 0.0 ? mean[i] : 0.0;
    if (o_var) o_var[i] = nn > 0.0 ? __ddiv_rn(m2[i], nn) : 0.0;
    if (o_m2) o_m2[i] = m2[i];
    if (o_count) o_count[i] = nn;
}

static dim3 tree_grid(ssa_u64 blocks_x, ssa_u64 rows)
{
    const ssa_u64 y = rows < 65535ull ? rows : 65535ull;
    const ssa_u64 z = (rows + 65534ull) / 65535ull;
    return dim3((unsigned)blocks_x, (unsigned)y, (unsigned)z);
}

cudaError_t ssa_tree_leaf_launch(const int* staging, ssa_u64 stride, ssa_u64 count, ssa_u64 rows,
                                 const ssa_tree_out& out, cudaStream_t st, int* launches)
{
    const ssa_u64 bx = (count + SSA_TREE_SPAN - 1) / SSA_TREE_SPAN;
    // full tiles through the division-free kernel (needs 16-byte aligned rows)
    const bool aligned = stride % 4 == 0 && ((uintptr_t)staging % 16) == 0;
    const ssa_u64 n_full = aligned ? count / SSA_TREE_SPAN : 0;
    if (n_full) {
        ssa_tree_leaf_full<<<tree_grid((n_full + 1) / 2, rows), SSA_TREE_BLOCK, 0, st>>>(staging, stride, n_full,
                                                                                          rows, out);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        ++*launches;
    }
    if (bx > n_full || bx == 0) {
        ++*launches;
        ssa_tree_leaf<<<tree_grid(bx ? bx - n_full : 1, rows), SSA_TREE_BLOCK, 0, st>>>(staging, stride, count, rows,
                                                                                       n_full, out);
    }
    return cudaGetLastError();
}

cudaError_t ssa_tree_merge_launch(const ssa_tree_in& in, ssa_u64 count, ssa_u64 rows, const ssa_tree_out& out,
                                  cudaStream_t st)
{
    const ssa_u64 bx = (count + SSA_TREE_SPAN - 1) / SSA_TREE_SPAN;
    ssa_tree_merge<<<tree_grid(bx ? bx : 1, rows), SSA_TREE_BLOCK, 0, st>>>(in, count, rows, out);
    return cudaGetLastError();
}

cudaError_t ssa_finalize_launch(const double* n, const double* mean, const double* m2, ssa_u64 cells,
                                double* o_mean, double* o_var, double* o_m2, double* o_count, cudaStream_t st)
{
    const unsigned b = 256;
    const ssa_u64 g = (cells + b - 1) / b;
    ssa_finalize<<<(unsigned)(g ? g : 1), b, 0, st>>>(n, mean, m2, cells, o_mean, o_var, o_m2, o_count);
    return cudaGetLastError();
}
