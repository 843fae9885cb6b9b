// Pipe-throughput microbenchmark for the K1/K2 rooflines ("The B200 FP64 rate is
// not in MEASURED_PEAKS.json; measure it with a DFMA/DADD microbenchmark on the box before quoting
// pipe fractions").  Measurement tool only; not part of libssa.
//
// Each kernel runs 8 independent dependency chains per thread of one instruction kind in one wave
// of resident 256-thread blocks, and reports warp-instructions per SM per SM-clock
// (clock64 inside the kernel, so the figure is independent of the clock the box runs at) and
// instructions per second (CUDA events).  Build and run on the GPU box:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pipe_peaks scripts/pipe_peaks.cu && /tmp/pipe_peaks
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

enum { OP_DADD, OP_DMUL, OP_DFMA, OP_FFMA, OP_IADD3, OP_IMAD, OP_MIX };
static const char* kNames[] = {"DADD", "DMUL", "DFMA", "FFMA", "IADD3", "IMAD", "DADD+IADD3 pair"};

template <int OP>
__global__ void __launch_bounds__(256) pipe_kernel(int iters, double* sink, long long* cycles) {
    double d[8];
    float f[8];
    uint32_t u[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        d[c] = threadIdx.x + c;
        f[c] = threadIdx.x + c;
        u[c] = threadIdx.x * 7 + c;
    }
    const double db = 1.0000000001, dc = 1e-12;
    const float fb = 1.0001f, fc = 1e-6f;
    const uint32_t ub = blockIdx.x | 1u;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (OP == OP_DADD) d[c] = __dadd_rn(d[c], db);
            if (OP == OP_DMUL) d[c] = __dmul_rn(d[c], db);
            if (OP == OP_DFMA) d[c] = __fma_rn(d[c], db, dc);
            if (OP == OP_FFMA) f[c] = __fmaf_rn(f[c], fb, fc);
            if (OP == OP_IADD3) u[c] = u[c] + ub + (uint32_t)i;
            if (OP == OP_IMAD) u[c] = u[c] * ub + (uint32_t)c;
            if (OP == OP_MIX) {
                d[c] = __dadd_rn(d[c], db);
                u[c] = u[c] + ub + (uint32_t)i;
            }
        }
    }
    const long long t1 = clock64();
    double acc = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) acc += d[c] + f[c] + (double)u[c];
    if (acc == 1.2345) sink[0] = acc;  // keeps the chains live
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
static void run(int sms) {
    // exactly one wave: the resident blocks per SM at this kernel's register use
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pipe_kernel<OP>, 256, 0);
    const int blocks = sms * per_sm, threads = 256, iters = 1 << 14;
    double* sink;
    long long* cyc;
    cudaMalloc(&sink, 8);
    cudaMalloc(&cyc, blocks * sizeof(long long));
    pipe_kernel<OP><<<blocks, threads>>>(1 << 12, sink, cyc);  // warm-up
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    pipe_kernel<OP><<<blocks, threads>>>(iters, sink, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    long long* h = new long long[blocks];
    cudaMemcpy(h, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    double avg = 0;
    for (int i = 0; i < blocks; ++i) {
        mx = h[i] > mx ? h[i] : mx;
        avg += h[i];
    }
    avg /= blocks;
    // warp-instructions of the measured kind per SM: resident blocks x 8 warps x iters x 8 chains
    // (the mix kernel issues one DADD and one IADD3 per chain step; counted as pairs); all blocks
    // of the wave run concurrently, so the per-SM rate is over the longest block's cycles
    const double winst_per_sm = (double)per_sm * 8.0 * iters * 8.0;
    const double per_clk = winst_per_sm / (double)mx;
    const double per_s = winst_per_sm * sms / (ms * 1e-3);
    printf("%-16s %d blocks/SM  %7.3f warp-inst/SM/clk (%.3f per SMSP)  %8.1f G warp-inst/s  "
           "kernel %.3f ms  block cycles avg %.0f max %lld  => SM clock %.0f MHz\n",
           kNames[OP], per_sm, per_clk, per_clk / 4, per_s * 1e-9, ms, avg, mx, mx / (ms * 1e3));
    delete[] h;
    cudaFree(sink);
    cudaFree(cyc);
}

int main() {
    cudaFree(0);
    {   // ~0.5 s of load first, so the SM clock has ramped up before the measured kernels
        double* sink;
        long long* cyc;
        cudaMalloc(&sink, 8);
        cudaMalloc(&cyc, 148 * 64 * sizeof(long long));
        for (int i = 0; i < 20; ++i) pipe_kernel<OP_DADD><<<148 * 4, 256>>>(1 << 14, sink, cyc);
        cudaDeviceSynchronize();
    }
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    printf("device %s, %d SMs, cc %d.%d\n", p.name, p.multiProcessorCount, p.major, p.minor);
    const int sms = p.multiProcessorCount;
    run<OP_DADD>(sms);
    run<OP_DMUL>(sms);
    run<OP_DFMA>(sms);
    run<OP_FFMA>(sms);
    run<OP_IADD3>(sms);
    run<OP_IMAD>(sms);
    run<OP_MIX>(sms);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
