// Is the FP64 tensor-core path (mma.sync m8n8k4 f64, DMMA) extra throughput beside DFMA on B200?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_bench tools/dev/dmma_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MODE>  // 0: DFMA only, 1: DMMA only, 2: both interleaved
__global__ void k(double *out, int iters)
{
    double a = threadIdx.x * 1e-3, b = 1.0000001;
    double f[8], d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0};
    for (int i = 0; i < 8; ++i) f[i] = a + i;
    for (int it = 0; it < iters; ++it) {
        if (MODE != 1) {
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = fma(f[i], b, a);
        }
        if (MODE != 0) {
#pragma unroll
            for (int i = 0; i < 4; ++i) dmma(d0[i], d1[i], a, b);
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += f[i];
    for (int i = 0; i < 4; ++i) s += d0[i] + d1[i];
    if (s == 12345.678) out[0] = s;
}

int main()
{
    double *o;
    cudaMalloc(&o, 8);
    const int iters = 20000, blocks = 148 * 4, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<blocks, threads>>>(o, iters);
            if (mode == 1) k<1><<<blocks, threads>>>(o, iters);
            if (mode == 2) k<2><<<blocks, threads>>>(o, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double th = (double)blocks * threads * iters;
            const double dfma = mode != 1 ? th * 8 : 0;           // thread-level DFMA
            const double dmma = mode != 0 ? th / 32 * 4 * 256 : 0; // MACs (8x8x4 per warp-instr)
            if (rep)
                printf("mode %d: %.3f ms  DFMA %.2f Tflop/s  DMMA %.2f Tflop/s  total %.2f\n", mode, ms,
                       2 * dfma / ms / 1e9, 2 * dmma / ms / 1e9, 2 * (dfma + dmma) / ms / 1e9);
        }
    }
    return 0;
}
