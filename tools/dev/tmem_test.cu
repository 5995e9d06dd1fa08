// TMEM round trip check (developer tool): allocate all 512 columns, every warp writes a
// known pattern into its lane quarter with tcgen05.st.32x32b, reads it back with
// tcgen05.ld.32x32b, and counts mismatches.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void tm_st32(uint32_t taddr, const uint32_t (&r)[32])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
__device__ __forceinline__ void tm_ld32(uint32_t taddr, uint32_t (&r)[32])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

__global__ void k_tmem_roundtrip(unsigned *bad, unsigned long long *cycles)
{
    __shared__ uint32_t base_s;
    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&base_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = base_s;
    const uint32_t q = warp % 4;                 // lane quarter this warp may touch
    const uint32_t nq = blockDim.x / 128;        // warps sharing a quarter
    const uint32_t part = warp / 4;              // which slice of the 512 columns
    const uint32_t cols = 512 / nq;
    unsigned long long t0 = clock64();
    for (uint32_t c0 = part * cols; c0 < (part + 1) * cols; c0 += 32) {
        uint32_t r[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = (blockIdx.x << 24) ^ ((32 * q + lane) << 12) ^ (c0 + i);
        tm_st32(base + ((32 * q) << 16) + c0, r);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    unsigned nbad = 0;
    // read back the slice of another warp of the same quarter (crosses warps)
    const uint32_t rpart = (part + 1) % nq;
    for (uint32_t c0 = rpart * cols; c0 < (rpart + 1) * cols; c0 += 32) {
        uint32_t r[32];
        tm_ld32(base + ((32 * q) << 16) + c0, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int i = 0; i < 32; ++i) nbad += r[i] != ((blockIdx.x << 24) ^ ((32 * q + lane) << 12) ^ (c0 + i));
    }
    unsigned long long t1 = clock64();
    atomicAdd(bad, nbad);
    if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

int main()
{
    unsigned *bad;
    unsigned long long *cyc;
    cudaMalloc(&bad, 4);
    cudaMalloc(&cyc, 8);
    cudaMemset(bad, 0, 4);
    cudaFuncSetAttribute(k_tmem_roundtrip, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
    for (int threads : {128, 256, 512}) {
        cudaMemset(bad, 0, 4);
        k_tmem_roundtrip<<<296, threads, 150 * 1024>>>(bad, cyc);  // big smem: one CTA per SM at a time
        cudaError_t e = cudaDeviceSynchronize();
        unsigned hb = 0;
        unsigned long long hc = 0;
        cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
        printf("threads=%d err=%s mismatches=%u cycles(st+ld of 256 KB)=%llu\n", threads, cudaGetErrorString(e), hb, hc);
    }
    return 0;
}
