// copy_bench -- D2H into differently allocated pinned buffers, alone and beside an H2D copy on
// another stream (diagnosing the host-buffer pipeline).  nvcc -O2 tools/copy_bench.cu -o /tmp/cb
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
int main() {
    const size_t N = 24 << 20, M = 4 << 20;
    void *d_out, *d_in, *h_in;
    cudaMalloc(&d_out, N); cudaMalloc(&d_in, M); cudaMallocHost(&h_in, M);
    void* h[3];
    cudaMallocHost(&h[0], N);
    cudaHostAlloc(&h[1], N, cudaHostAllocPortable);
    h[2] = aligned_alloc(4096, N); cudaHostRegister(h[2], N, cudaHostRegisterDefault);
    const char* names[3] = {"cudaMallocHost", "HostAllocPortable", "HostRegister"};
    cudaStream_t a, b; cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    cudaEvent_t e[4]; for (auto& x : e) cudaEventCreate(&x);
    for (int k = 0; k < 3; ++k)
        for (int with_h2d = 0; with_h2d < 2; ++with_h2d)
            for (int rep = 0; rep < 3; ++rep) {
                cudaDeviceSynchronize();
                cudaEventRecord(e[0], a);
                cudaMemcpyAsync(h[k], d_out, N, cudaMemcpyDeviceToHost, a);
                cudaEventRecord(e[1], a);
                if (with_h2d) {
                    cudaEventRecord(e[2], b);
                    cudaMemcpyAsync(d_in, h_in, M, cudaMemcpyHostToDevice, b);
                    cudaEventRecord(e[3], b);
                }
                cudaDeviceSynchronize();
                float t = 0, s = 0, f = 0;
                cudaEventElapsedTime(&t, e[0], e[1]);
                if (with_h2d) { cudaEventElapsedTime(&s, e[0], e[2]); cudaEventElapsedTime(&f, e[0], e[3]); }
                if (rep == 2) printf("%-18s h2d=%d  d2h %.3f ms (%.1f GB/s)  h2d start %.3f end %.3f\n", names[k], with_h2d, t, N / t / 1e6, s, f);
            }
}
