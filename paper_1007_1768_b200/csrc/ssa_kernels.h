// ssa_kernels.h -- internal interface between the runtime (ssa_api.cpp) and
// the nvcc-compiled kernels (kernels.cu).  Not part of the public C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#ifndef SSA_DEVICE_TYPES
#define SSA_DEVICE_TYPES
typedef unsigned int ssa_u32;
typedef unsigned long long ssa_u64;
typedef long long ssa_i64;
#endif

#define SSA_K2_BLOCK 256
#define SSA_TREE_BLOCK 256
#define SSA_TREE_SPAN (8 * SSA_TREE_BLOCK)

struct ssa_dev_summary;
struct ssa_dev_stats;

struct ssa_k2_params {
    // model (device copies, see pack_k2)
    int S, R, P, PMAX, n_ent;
    const ssa_u64* pk;       // [R] packed reactant terms + modifier species
    const double* rate;      // [R]
    const double* modc;      // [R]
    const double* x0;        // [S]
    const int* nu_off;       // [R+1]
    const int* nu_ent;       // [n_ent] (species | delta << 16)
    int n_dep;
    const int* dep_off;      // [S+1] species -> reactions whose propensity reads it
    const int* dep_ent;      // [n_dep] reaction indices
    // run
    ssa_u64 id_begin, n_ids;
    int* staging;
    ssa_u64 stride;
    double dt;
    long long K;
    ssa_u32 key0, key1;
    ssa_u64* work;
    const ssa_u64* dump_ids;
    ssa_u64 n_dump;
    int* dump_states;
    ssa_u64* dump_e;
    double* dump_t;
    ssa_dev_summary* dump_sum;
    ssa_dev_stats* stats;
};

struct ssa_tree_in {
    const double *n, *mean, *m2;
    ssa_u64 row_stride, elem_stride;
};

struct ssa_tree_out {
    double *n, *mean, *m2;
    ssa_u64 row_stride, elem_stride, offset;
};

size_t ssa_k2_smem_bytes(int S, int R, int P, int n_ent, int n_dep, int block);
cudaError_t ssa_k2_launch(const ssa_k2_params& p, int grid, int block, cudaStream_t st);
int ssa_k2_max_blocks_per_sm(int pmax, int block, size_t smem);

cudaError_t ssa_tree_leaf_launch(const int* staging, ssa_u64 stride, ssa_u64 count, ssa_u64 rows,
                                 const ssa_tree_out& out, cudaStream_t st, int* launches);
cudaError_t ssa_tree_merge_launch(const ssa_tree_in& in, ssa_u64 count, ssa_u64 rows, const ssa_tree_out& out,
                                  cudaStream_t st);
cudaError_t ssa_finalize_launch(const double* n, const double* mean, const double* m2, ssa_u64 cells,
                                double* o_mean, double* o_var, double* o_m2, double* o_count, cudaStream_t st);
