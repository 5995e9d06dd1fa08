// microbench.cu -- measured B200 constants that decide route (a)'s design.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench.cu && ./mb
// 1. FP64 DFMA / DADD issue rate per SM per clock
// 2. int32 IMAD / IADD3 / LOP3 rates
// 3. HBM copy bandwidth with contiguous vs strided runs of 16/32/64/128/256 bytes
// 4. DSMEM all-to-all bandwidth inside an 8-CTA cluster
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_dfma(double *out, int iters)
{
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 1.0000001, c = 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_dadd(double *out, int iters)
{
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double c = 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            a0 += c; a1 += c; a2 += c; a3 += c; a4 += c; a5 += c; a6 += c; a7 += c;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_imad(unsigned *out, int iters)
{
    unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    unsigned b = out[0] | 3, c = out[1];
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            a0 = a0 * b + c; a1 = a1 * b + c; a2 = a2 * b + c; a3 = a3 * b + c;
            a4 = a4 * b + c; a5 = a5 * b + c; a6 = a6 * b + c; a7 = a7 * b + c;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_lop3(unsigned *out, int iters)
{
    unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    unsigned b = out[0], c = out[1];
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            a0 ^= b & (c + k); a1 ^= b & (a0 >> 1); a2 ^= c & a1; a3 ^= b & a2;
            a4 ^= c & a3; a5 ^= b & a4; a6 ^= c & a5; a7 ^= b & a6;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_shf(unsigned *out, int iters)
{
    unsigned acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned A = out[0] + threadIdx.x, B = out[1], X = out[2];
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int b = 0; b < 32; ++b) acc[b & 7] ^= X & __funnelshift_r(A, B, b);
        A = B ^ i; B = A + X;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] ^ acc[1] ^ acc[2] ^ acc[3] ^ acc[4] ^ acc[5] ^ acc[6] ^ acc[7];
}

// copy with runs of RUN bytes: element e of run r at src[(r * stride) + e]
template <int RUN>
__global__ void k_strided_copy(const double2 *__restrict__ src, double2 *__restrict__ dst, size_t nruns, size_t stride_elems)
{
    constexpr int E = RUN / 16;
    size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    size_t nthreads = (size_t)gridDim.x * blockDim.x;
    for (size_t i = tid; i < nruns * E; i += nthreads) {
        size_t r = i / E, e = i % E;
        // runs are visited in a scattered order: consecutive warps hit distant rows
        size_t rr = (r * 2654435761ull) % nruns;
        dst[rr * stride_elems + e] = src[rr * stride_elems + e];
    }
}

__global__ void k_dsmem(double2 *out, int iters)
{
    extern __shared__ double2 sm[];
    cg::cluster_group cl = cg::this_cluster();
    const int n = 4096;  // 64 KB per CTA
    for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = make_double2(i, blockIdx.x);
    cl.sync();
    double2 acc = make_double2(0, 0);
    unsigned r = cl.block_rank(), cs = cl.num_blocks();
    for (int it = 0; it < iters; ++it) {
        for (unsigned p = 1; p < cs; ++p) {
            double2 *peer = cl.map_shared_rank(sm, (r + p) % cs);
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                double2 v = peer[i];
                acc.x += v.x;
                acc.y += v.y;
            }
        }
    }
    cl.sync();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main2();
int main()
{
    if (main2()) return 1;
    int dev = 0, sms = 0, clk = 0;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    printf("SMs %d, max clock %.0f MHz\n", sms, clk / 1000.0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    double *dout;
    CK(cudaMalloc(&dout, 1 << 26));
    CK(cudaMemset(dout, 0, 1 << 26));
    int blocks = sms * 4, threads = 512, iters = 2000;
    auto rate = [&](const char *name, double ops_per_thread_iter, auto launch) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)blocks * threads * iters * ops_per_thread_iter;
        printf("%-8s %.3f Tops/s -> %.1f ops/clk/SM at 1965 MHz (%.3f ms)\n", name, ops / ms / 1e9,
               ops / (ms * 1e-3) / sms / 1.965e9, ms);
    };
    rate("DFMA", 128, [&] { k_dfma<<<blocks, threads>>>(dout, iters); });
    rate("DADD", 128, [&] { k_dadd<<<blocks, threads>>>(dout, iters); });
    rate("IMAD", 128, [&] { k_imad<<<blocks, threads>>>((unsigned *)dout, iters); });
    rate("LOP3", 128 * 1.5, [&] { k_lop3<<<blocks, threads>>>((unsigned *)dout, iters); });
    rate("SHF+LOP", 64, [&] { k_shf<<<blocks, threads>>>((unsigned *)dout, iters); });
    CK(cudaGetLastError());

    size_t bytes = (size_t)1 << 31;  // 2 GiB buffers
    double2 *src, *dst;
    CK(cudaMalloc(&src, bytes));
    CK(cudaMalloc(&dst, bytes));
    CK(cudaMemset(src, 1, bytes));
    auto bw = [&](int run, auto launch) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        return ms / 3;
    };
    // runs of RUN bytes, rows spaced by 64 KiB (stride), covering 1/ (stride/RUN) of the buffer
    size_t total_elems = bytes / 16;
#define RUNBW(RUN)                                                                                 \
    {                                                                                              \
        size_t stride = 4096; /* elements (64 KiB) between runs */                                  \
        size_t nruns = total_elems / stride * (stride / (RUN / 16));                               \
        /* pack runs densely: stride_elems = RUN/16 means contiguous */                            \
        size_t se = (size_t)RUN / 16 * 1;                                                          \
        (void)stride;                                                                              \
        nruns = total_elems / se;                                                                  \
        float t = bw(RUN, [&] { k_strided_copy<RUN><<<sms * 8, 512>>>(src, dst, nruns, se); });    \
        printf("scattered runs of %4d B: %.0f GB/s (read+write)\n", RUN, 2.0 * nruns * RUN / t / 1e6); \
    }
    RUNBW(16) RUNBW(32) RUNBW(64) RUNBW(128) RUNBW(256)
    {
        float t = bw(0, [&] { cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice); });
        printf("cudaMemcpy D2D: %.0f GB/s (read+write)\n", 2.0 * bytes / t / 1e6);
    }
    CK(cudaGetLastError());

    // DSMEM
    for (int cs : {2, 4, 8}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(sms / cs * cs);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = 65536;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
        int it = 20;
        CK(cudaLaunchKernelEx(&cfg, k_dsmem, (double2 *)dout, it));
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        CK(cudaLaunchKernelEx(&cfg, k_dsmem, (double2 *)dout, it));
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double b = (double)cfg.gridDim.x * (cs - 1) * 65536.0 * it;
        printf("DSMEM cluster %d: %.0f GB/s total remote reads = %.1f B/clk/SM\n", cs, b / ms / 1e6,
               b / (ms * 1e-3) / cfg.gridDim.x / 1.965e9);
    }
    CK(cudaGetLastError());
    return 0;
}

// ---- column-group pattern: CTA owns C adjacent columns of an [N2][N1] array of
// double2, copies its tile to another array with the same layout.  One CTA per SM
// (smem tile) vs register streaming.
template <int C>
__global__ void k_colgroup(const double2 *__restrict__ src, double2 *__restrict__ dst, int N1, int N2)
{
    size_t a0 = (size_t)blockIdx.x * C;
    int tot = N2 * C;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        int p = e / C, c = e % C;
        size_t off = (size_t)p * N1 + a0 + c;
        dst[off] = __ldg(src + off);
    }
}

template <int C>
__global__ void k_colgroup_smem(const double2 *__restrict__ src, double2 *__restrict__ dst, int N1, int N2)
{
    extern __shared__ double2 sm[];
    size_t a0 = (size_t)blockIdx.x * C;
    int tot = N2 * C;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        int p = e / C, c = e % C;
        size_t off = (size_t)p * N1 + a0 + c;
        unsigned sa = (unsigned)__cvta_generic_to_shared(sm + e);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src + off));
    }
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
        int p = e / C, c = e % C;
        size_t off = (size_t)p * N1 + a0 + c;
        dst[off] = sm[e];
    }
}

int main2()
{
    int sms = 148;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    const int N1 = 9600, N2 = 6250;
    size_t bytes = (size_t)N1 * N2 * 16;
    double2 *src, *dst;
    CK(cudaMalloc(&src, bytes));
    CK(cudaMalloc(&dst, bytes));
    CK(cudaMemset(src, 1, bytes));
    auto tm = [&](auto launch) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        return ms / 3;
    };
#define CG(C)                                                                                       \
    {                                                                                               \
        float t = tm([&] { k_colgroup<C><<<N1 / C, 1024>>>(src, dst, N1, N2); });                  \
        printf("colgroup C=%d regs: %.0f GB/s\n", C, 2.0 * bytes / t / 1e6);                       \
        int sb = N2 * C * 16;                                                                       \
        if (sb <= 232448) {                                                                         \
            CK(cudaFuncSetAttribute(k_colgroup_smem<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448)); \
            t = tm([&] { k_colgroup_smem<C><<<N1 / C, 1024, sb>>>(src, dst, N1, N2); });           \
            printf("colgroup C=%d smem tile %d KB: %.0f GB/s\n", C, sb / 1024, 2.0 * bytes / t / 1e6); \
        }                                                                                           \
    }
    CG(1) CG(2) CG(4) CG(8) CG(16)
    CK(cudaGetLastError());
    // row tiles: CTA copies one contiguous row of N1 via smem (1 row per CTA)
    return 0;
}
