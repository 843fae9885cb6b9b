// kernels.cu -- nvcc-compiled kernels of the ensemble-SSA hot path (sm_100a):
//   K3  ssa_tree_leaf  canonical-tree Welford reduction of a chunk's staged
//                      grid samples (a9, no atomics: north_star (d)).
//   K4  ssa_tree_merge merge of partial roots (tiles -> chunk -> shard -> GPUs)
//       ssa_finalize   mean, population variance = M2/n (a10).
// K1 (thread path, k1_thread.cuh) and K2 (warp path, k2_warp.cuh) are
// model-specialised and compiled by NVRTC at run time (runtime.cu).
#include <cuda_runtime.h>
#include <stdint.h>

#include "ssa_device.cuh"
#include "ssa_kernels.h"


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

// The staged samples are trajectory-major (runtime.cu): trajectory i's grid samples form a row of
// `row` ints (cells rounded up to 8), element (i, cell) at i*row + cell.  A K3 block reduces one
// 2048-id tile for a group of 8 consecutive cells: thread t holds ids [8t, 8t+8), and each of its
// ids' 8 cells is one 32-byte sector (two 16-byte loads), so the tile's samples are read as whole
// sectors exactly once.  Per cell the reduction is the same canonical tree as before (8 adjacent
// leaves per thread, then the warp and block levels).
#define SSA_TREE_CG 8

// the 8-leaf fold of one cell over a thread's 8 ids, full leaves: the integer fast path when all
// counts are below 2^20 (exact: see below), else the division-free fp64 merges
static __device__ __forceinline__ void fold8_full(const int (&c)[8], double& mm, double& vv)
{
    const unsigned lim = 1u << 20;
    bool small = true;
#pragma unroll
    for (int i = 0; i < 8; ++i) small = small && (unsigned)c[i] < lim;
    if (small) {
        // Counts below 2^20: every operation of these three merge levels is exact in fp64
        // (means are multiples of 2^-3 below 2^20, deltas have <= 22 significant bits so
        // their squares <= 44, the M2 sums stay below 2^49 with <= 4 fractional bits), so the
        // tree yields the exact mean = S1/8 and M2 = (8 S2 - S1^2)/8 -- computed here in
        // integers, bitwise equal to the fp64 merges and without their FP64 work.
        unsigned long long s1 = 0, s2 = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            s1 += (unsigned long long)c[i];
            s2 += (unsigned long long)c[i] * (unsigned long long)c[i];
        }
        mm = __dmul_rn((double)s1, 0.125);
        vv = __dmul_rn((double)(8ull * s2 - s1 * s1), 0.125);
    } else {
        double m[8], v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) { m[i] = (double)c[i]; v[i] = 0.0; }
        wf_merge_full(m[0], v[0], m[1], v[1], 0.5);
        wf_merge_full(m[2], v[2], m[3], v[3], 0.5);
        wf_merge_full(m[4], v[4], m[5], v[5], 0.5);
        wf_merge_full(m[6], v[6], m[7], v[7], 0.5);
        wf_merge_full(m[0], v[0], m[2], v[2], 1.0);
        wf_merge_full(m[4], v[4], m[6], v[6], 1.0);
        wf_merge_full(m[0], v[0], m[4], v[4], 2.0);
        mm = m[0];
        vv = v[0];
    }
}

// Full tiles only: cell group = blockIdx.x, tile = blockIdx.y (+ 65535 * z) (< count / SPAN).  Consecutive
// blocks take consecutive cell groups of one tile, so the blocks resident together read whole
// trajectory rows front to back (DRAM page locality) instead of one 32-byte sector per row.
__global__ void __launch_bounds__(SSA_TREE_BLOCK, 2) ssa_tree_leaf_full(const int* __restrict__ staging,
                                                                       ssa_u64 row, ssa_u64 cells, ssa_tree_out out)
{
    __shared__ double shm[SSA_TREE_CG][SSA_TREE_BLOCK / 32], shq[SSA_TREE_CG][SSA_TREE_BLOCK / 32];
    const ssa_u64 cg = (ssa_u64)blockIdx.x;
    const ssa_u64 c0 = cg * SSA_TREE_CG;
    if (c0 >= cells) return;
    const ssa_u64 tile = (ssa_u64)blockIdx.y + 65535ull * blockIdx.z;
    const ssa_u64 id0 = tile * SSA_TREE_SPAN + (ssa_u64)threadIdx.x * 8;
    int v[SSA_TREE_CG][8];                                // [cell][leaf]
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        // one 32-byte load per id (LDG.256): the whole sector in one request (two 16-byte loads
        // sent 2.5x the bytes to L2, profiles/r2z_k3_summary.txt)
        asm volatile("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(v[0][i]), "=r"(v[1][i]), "=r"(v[2][i]), "=r"(v[3][i]), "=r"(v[4][i]), "=r"(v[5][i]),
                       "=r"(v[6][i]), "=r"(v[7][i])
                     : "l"(staging + (id0 + i) * row + c0));
    }
    double mm[SSA_TREE_CG], vv[SSA_TREE_CG];
#pragma unroll
    for (int c = 0; c < SSA_TREE_CG; ++c) fold8_full(v[c], mm[c], vv[c]);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // warp levels: subtrees of 8*o leaves, h/2 = 4*o
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
        for (int c = 0; c < SSA_TREE_CG; ++c) {
            const double mb = __shfl_down_sync(0xffffffffu, mm[c], o);
            const double vb = __shfl_down_sync(0xffffffffu, vv[c], o);
            if ((lane & (2 * o - 1)) == 0) wf_merge_full(mm[c], vv[c], mb, vb, 4.0 * o);
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int c = 0; c < SSA_TREE_CG; ++c) { shm[c][warp] = mm[c]; shq[c][warp] = vv[c]; }
    }
    __syncthreads();
    if (threadIdx.x < SSA_TREE_CG && c0 + threadIdx.x < cells) {
        const int c = threadIdx.x;
        double a[SSA_TREE_BLOCK / 32], b[SSA_TREE_BLOCK / 32];
#pragma unroll
        for (int i = 0; i < SSA_TREE_BLOCK / 32; ++i) { a[i] = shm[c][i]; b[i] = shq[c][i]; }
        // block levels: subtrees of 256*o leaves, h/2 = 128*o
#pragma unroll
        for (int o = 1; o < SSA_TREE_BLOCK / 32; o <<= 1)
#pragma unroll
            for (int i = 0; i + o < SSA_TREE_BLOCK / 32; i += 2 * o) wf_merge_full(a[i], b[i], a[i + o], b[i + o], 128.0 * o);
        const ssa_u64 o = (c0 + c) * out.row_stride + tile * out.elem_stride + out.offset;
        out.n[o] = (double)SSA_TREE_SPAN; out.mean[o] = a[0]; out.m2[o] = b[0];
    }
}

// General leaves (a tile with ids past `count`: empty leaves n = 0, the identity), tiles from `first`
__global__ void __launch_bounds__(SSA_TREE_BLOCK) ssa_tree_leaf(const int* __restrict__ staging, ssa_u64 row,
                                                                ssa_u64 cells, ssa_u64 count, ssa_u64 first,
                                                                ssa_tree_out out)
{
    const ssa_u64 cg = (ssa_u64)blockIdx.y + 65535ull * blockIdx.z;
    const ssa_u64 c0 = cg * SSA_TREE_CG;
    if (c0 >= cells) return;
    const ssa_u64 tile = first + blockIdx.x;
    const ssa_u64 id0 = tile * SSA_TREE_SPAN + (ssa_u64)threadIdx.x * 8;
    for (int c = 0; c < SSA_TREE_CG; ++c) {               // block-uniform loop (tree_block syncs)
        ssa_welford v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
            v[i] = (id0 + i < count && c0 + c < cells) ? ssa_welford_leaf(staging[(id0 + i) * row + c0 + c])
                                                        : ssa_welford_empty();
        ssa_welford w = tree_block(fold8(v));
        if (threadIdx.x == 0 && c0 + c < cells) {
            const ssa_u64 o = (c0 + c) * out.row_stride + tile * out.elem_stride + out.offset;
            out.n[o] = w.n; out.mean[o] = w.mean; out.m2[o] = w.m2;
        }
        __syncthreads();                                  // tree_block's shared scratch is reused
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

cudaError_t ssa_tree_leaf_launch(const int* staging, ssa_u64 row, ssa_u64 count, ssa_u64 cells,
                                 const ssa_tree_out& out, cudaStream_t st, int* launches)
{
    const ssa_u64 bx = (count + SSA_TREE_SPAN - 1) / SSA_TREE_SPAN;
    const ssa_u64 groups = (cells + SSA_TREE_CG - 1) / SSA_TREE_CG;
    // full tiles through the division-free kernel (32-byte aligned rows: one sector per id and group)
    const bool aligned = row % 8 == 0 && ((uintptr_t)staging % 32) == 0;
    const ssa_u64 n_full = aligned ? count / SSA_TREE_SPAN : 0;
    if (n_full) {
        const dim3 g((unsigned)groups, (unsigned)(n_full < 65535ull ? n_full : 65535ull),
                     (unsigned)((n_full + 65534ull) / 65535ull));
        ssa_tree_leaf_full<<<g, SSA_TREE_BLOCK, 0, st>>>(staging, row, cells, out);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        ++*launches;
    }
    if (bx > n_full || bx == 0) {
        ++*launches;
        ssa_tree_leaf<<<tree_grid(bx ? bx - n_full : 1, groups), SSA_TREE_BLOCK, 0, st>>>(staging, row, cells, count,
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
