// copy_bench2 -- does an H2D copy issued on stream M after D2H copies on stream O wait for them?
// (order A: D2H first, then H2D; order B: H2D first)  nvcc -O2 tools/copy_bench2.cu -o /tmp/cb2
#include <cuda_runtime.h>
#include <cstdio>
__global__ void spin(long long cycles) {
    const long long t0 = clock64();
    while (clock64() - t0 < cycles) {}
}
int main() {
    const size_t NO = 128 << 20, NI = 4 << 20;
    void *d_o, *d_i, *h_o, *h_i;
    cudaMalloc(&d_o, NO); cudaMalloc(&d_i, NI); cudaMallocHost(&h_o, NO); cudaMallocHost(&h_i, NI);
    cudaStream_t m, o;
    cudaStreamCreateWithFlags(&m, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&o, cudaStreamNonBlocking);
    cudaEvent_t t0, a, b, c, d;
    for (auto* e : {&t0, &a, &b, &c, &d}) cudaEventCreate(e);
    for (size_t no : {size_t(8) << 20, size_t(24) << 20, size_t(64) << 20, size_t(128) << 20})
    for (int order = 0; order < 2; ++order)
        for (int rep = 0; rep < 2; ++rep) {
            cudaDeviceSynchronize();
            cudaEventRecord(t0, m);
            spin<<<1, 1, 0, m>>>(200000);
            cudaStreamSynchronize(m);
            if (order == 0) {
                cudaEventRecord(a, o);
                cudaMemcpyAsync(h_o, d_o, no, cudaMemcpyDeviceToHost, o);
                cudaEventRecord(b, o);
                cudaEventRecord(c, m);
                cudaMemcpyAsync(d_i, h_i, NI, cudaMemcpyHostToDevice, m);
                cudaEventRecord(d, m);
            } else {
                cudaEventRecord(c, m);
                cudaMemcpyAsync(d_i, h_i, NI, cudaMemcpyHostToDevice, m);
                cudaEventRecord(d, m);
                cudaEventRecord(a, o);
                cudaMemcpyAsync(h_o, d_o, no, cudaMemcpyDeviceToHost, o);
                cudaEventRecord(b, o);
            }
            cudaDeviceSynchronize();
            float fa, fb, fc, fd;
            cudaEventElapsedTime(&fa, t0, a); cudaEventElapsedTime(&fb, t0, b);
            cudaEventElapsedTime(&fc, t0, c); cudaEventElapsedTime(&fd, t0, d);
            printf("%3zu MB order %s: d2h %.3f-%.3f  h2d %.3f-%.3f ms\n", no >> 20, order ? "H2D first" : "D2H first", fa, fb, fc, fd);
        }
}
