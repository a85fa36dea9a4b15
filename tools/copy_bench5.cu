// copy_bench5 -- D2H right after a kernel wrote the source (dirty L2) vs a cold source.
#include <cuda_runtime.h>
#include <cstdio>
__global__ void fill(uint4* p, size_t n, unsigned v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(v, (unsigned)i, v ^ (unsigned)i, 7u);
}
__global__ void fill32(unsigned* p, size_t n, unsigned v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v + (unsigned)i;
}
int main() {
    const size_t bytes = 21 << 20;
    void *d, *h; cudaMalloc(&d, bytes); cudaMallocHost(&h, bytes);
    cudaStream_t s, o; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&o, cudaStreamNonBlocking);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 4; ++mode)
        for (int rep = 0; rep < 3; ++rep) {
            if (mode == 1) fill<<<1184, 256, 0, s>>>((uint4*)d, bytes / 16, rep);
            if (mode == 2) fill32<<<1184, 256, 0, s>>>((unsigned*)d, bytes / 4, rep);
            if (mode == 3) { fill<<<1184, 256, 0, s>>>((uint4*)d, bytes / 16, rep); cudaStreamSynchronize(s); }
            cudaStreamSynchronize(s);
            cudaEventRecord(a, o);
            cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, o);
            cudaEventRecord(b, o);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep == 2) printf("mode %d (%s): %.1f GB/s\n", mode, mode == 0 ? "cold" : mode == 1 ? "uint4 writes" : mode == 2 ? "u32 writes" : "uint4+sync", bytes / ms / 1e6);
        }
}
