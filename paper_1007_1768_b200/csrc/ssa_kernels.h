// ssa_kernels.h -- internal interface between the runtime (runtime.cu) and
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


struct ssa_tree_in {
    const double *n, *mean, *m2;
    ssa_u64 row_stride, elem_stride;
};

struct ssa_tree_out {
    double *n, *mean, *m2;
    ssa_u64 row_stride, elem_stride, offset;
};


// staging: trajectory-major, element (trajectory i, cell) at i*row + cell; reduces ids [0, count)
// of every cell into out (element (cell, tile))
cudaError_t ssa_tree_leaf_launch(const int* staging, ssa_u64 row, ssa_u64 count, ssa_u64 cells,
                                 const ssa_tree_out& out, cudaStream_t st, int* launches);
cudaError_t ssa_tree_merge_launch(const ssa_tree_in& in, ssa_u64 count, ssa_u64 rows, const ssa_tree_out& out,
                                  cudaStream_t st);
cudaError_t ssa_finalize_launch(const double* n, const double* mean, const double* m2, ssa_u64 cells,
                                double* o_mean, double* o_var, double* o_m2, double* o_count, cudaStream_t st);

// union-time selective memory (union.cu)
struct ssa_union_args {
    ssa_u64 E;                          // recorded events (valid rows)
    ssa_u64 rows;                       // reserved rows (>= E; the others have time +inf)
    const double* rec_t;                // [E] event times
    const int* rec_j;                   // [E] reactions
    const int* rec_pre;                 // [E][U] pre-event counts of the species each reaction changes
    int U;
    int S;
    const int* nu_sp;                   // [R][U] changed species (-1: none)
    const int* nu_d;                    // [R][U] their net change
    const long long* s0;                // [S] sum over the ensemble of x0
    const long long* s0sq;              // [S] sum over the ensemble of x0^2
    ssa_u64 k;                          // trajectories
    double t_end;
    ssa_u64 kx;                         // X-reduction: Y-points per output point
    ssa_u64 capacity;                   // output points the buffers hold
    double *times, *mean, *var, *count; // device outputs [capacity], [capacity][S], [capacity][S], [capacity]
};
cudaError_t ssa_union_reduce(ssa_union_args a, cudaStream_t st, ssa_u64* n_points, int* launches);

// stride-sampled trajectory output (union.cu): sort the recorded points by
// key and gather them (device outputs of `capacity` rows; *n_points = points)
cudaError_t ssa_points_gather(const ssa_u64* keys, const double* t, const int* states, ssa_u64 rows, int S,
                              ssa_u64 capacity, unsigned* o_traj, ssa_u64* o_event, double* o_time, int* o_state,
                              ssa_u64* n_points, cudaStream_t st, int* launches);

