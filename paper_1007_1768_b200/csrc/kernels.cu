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

static __device__ __forceinline__ void tree_block_full(const int4 q0, const int4 q1, double& mean, double& m2)
{
    __shared__ double shm[SSA_TREE_BLOCK / 32], shq[SSA_TREE_BLOCK / 32];
    // 8 adjacent leaves per thread: levels h = 1, 2, 4.
    double mm, vv;
    const unsigned lim = 1u << 20;
    if ((unsigned)q0.x < lim && (unsigned)q0.y < lim && (unsigned)q0.z < lim && (unsigned)q0.w < lim &&
        (unsigned)q1.x < lim && (unsigned)q1.y < lim && (unsigned)q1.z < lim && (unsigned)q1.w < lim) {
        // Counts below 2^20: every operation of these three merge levels is
        // exact in fp64 (means are multiples of 2^-3 below 2^20, deltas have
        // <= 22 significant bits so their squares <= 44, the M2 sums stay below
        // 2^49 with <= 4 fractional bits), so the tree yields the exact
        // mean = S1/8 and M2 = (8 S2 - S1^2)/8 -- computed here in integers,
        // bitwise equal to the fp64 merges and without their FP64 work.
        const unsigned long long s1 = (unsigned long long)q0.x + q0.y + q0.z + q0.w + q1.x + q1.y + q1.z + q1.w;
        const unsigned long long s2 =
            (unsigned long long)q0.x * q0.x + (unsigned long long)q0.y * q0.y + (unsigned long long)q0.z * q0.z +
            (unsigned long long)q0.w * q0.w + (unsigned long long)q1.x * q1.x + (unsigned long long)q1.y * q1.y +
            (unsigned long long)q1.z * q1.z + (unsigned long long)q1.w * q1.w;
        mm = __dmul_rn((double)s1, 0.125);
        vv = __dmul_rn((double)(8ull * s2 - s1 * s1), 0.125);
    } else {
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
        mm = m[0];
        vv = v[0];
    }
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
