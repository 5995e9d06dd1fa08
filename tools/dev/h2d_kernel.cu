// Experiment (developer tool): moving a small key in and a small result out of pinned host
// memory with the copy engines (cudaMemcpyAsync nodes) vs with copy kernels that read / write
// the mapped host pages directly.  Each variant is a CUDA graph of H2D + a stand-in kernel +
// D2H, timed with events over back-to-back launches.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/h2d tools/dev/h2d_kernel.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__global__ void k_copy16(const uint4 *__restrict__ src, uint4 *__restrict__ dst, size_t n16)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

__global__ void k_work(const uint32_t *key, uint32_t *out, size_t kw, size_t ow, int spin)
{
    // stand-in for the hash: touch the key, produce the output, burn ~spin ns
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    long long t0 = clock64();
    while (clock64() - t0 < spin) {}
    if (i < ow) out[i] = key[i % kw] ^ 0x5a5a5a5au;
}

static float time_graph(cudaGraphExec_t ex, cudaStream_t s, int iters)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 5; ++i) cudaGraphLaunch(ex, s);
    cudaStreamSynchronize(s);
    std::vector<float> ts;
    for (int i = 0; i < iters; ++i) {
        cudaEventRecord(a, s);
        cudaGraphLaunch(ex, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ts.push_back(ms * 1e3f);
    }
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
}

int main()
{
    const size_t kb = 125008, ob = 31264;  // C2: n = 1,000,003 bits in, m = 250,000 bits out
    const size_t kw = kb / 4, ow = ob / 4;
    uint32_t *hk, *ho, *dk, *dout;
    cudaHostAlloc(&hk, kb, cudaHostAllocDefault);
    cudaHostAlloc(&ho, ob, cudaHostAllocDefault);
    cudaMalloc(&dk, kb);
    cudaMalloc(&dout, ob);
    for (size_t i = 0; i < kw; ++i) hk[i] = (uint32_t)(i * 2654435761u);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int spin : {0, 20000}) {
        for (int variant = 0; variant < 4; ++variant) {
            cudaGraph_t g;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
            if (variant & 1) k_copy16<<<148, 256, 0, s>>>((const uint4 *)hk, (uint4 *)dk, kb / 16);
            else cudaMemcpyAsync(dk, hk, kb, cudaMemcpyHostToDevice, s);
            k_work<<<(ow + 255) / 256, 256, 0, s>>>(dk, dout, kw, ow, spin);
            if (variant & 2) k_copy16<<<16, 128, 0, s>>>((const uint4 *)dout, (uint4 *)ho, ob / 16);
            else cudaMemcpyAsync(ho, dout, ob, cudaMemcpyDeviceToHost, s);
            cudaStreamEndCapture(s, &g);
            cudaGraphExec_t ex;
            cudaGraphInstantiate(&ex, g, 0);
            float us = time_graph(ex, s, 200);
            cudaError_t e = cudaStreamSynchronize(s);
            bool ok = true;
            for (size_t i = 0; i < ow; ++i) ok &= ho[i] == (hk[i % kw] ^ 0x5a5a5a5au);
            printf("spin=%d in=%s out=%s: %.1f us  ok=%d err=%s\n", spin, variant & 1 ? "kernel" : "memcpy",
                   variant & 2 ? "kernel" : "memcpy", us, ok, cudaGetErrorString(e));
            cudaGraphExecDestroy(ex);
            cudaGraphDestroy(g);
            for (size_t i = 0; i < ow; ++i) ho[i] = 0;
        }
    }
    // the work kernel alone
    cudaGraph_t g;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    k_work<<<(ow + 255) / 256, 256, 0, s>>>(dk, dout, kw, ow, 20000);
    cudaStreamEndCapture(s, &g);
    cudaGraphExec_t ex;
    cudaGraphInstantiate(&ex, g, 0);
    printf("work kernel alone (spin=20000): %.1f us\n", time_graph(ex, s, 200));
    return 0;
}
