// copy_bench3 -- the host-buffer pipeline's stream pattern with dummy kernels:
//   main: H2D(c) -> wait(out_done) -> kernel -> small D2H;  host: sync main;
//   out:  D2H(c) 64 MB -> record out_done;  then the next chunk's H2D on main.
// Prints when each H2D starts relative to the previous chunk's D2H.  (diagnostic)
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
__global__ void spin(long long cycles) {
    const long long t0 = clock64();
    while (clock64() - t0 < cycles) {}
}
int main(int argc, char** argv) {
    const int use_wait = argc > 1 ? atoi(argv[1]) : 1;
    const int use_kernel = argc > 2 ? atoi(argv[2]) : 1;
    const int small = argc > 3 ? atoi(argv[3]) : 1;  // small D2H: 0 none, 1 on main, 2 on its own stream
    const int in_stream = argc > 4 ? atoi(argv[4]) : 0;  // H2D on its own stream (main waits on an event)
    const size_t NO = 64 << 20, NI = 4 << 20;
    void *d_o, *d_i, *h_o, *h_i, *h_s, *d_s;
    cudaMalloc(&d_o, NO); cudaMalloc(&d_i, NI); cudaMallocHost(&h_o, NO); cudaMallocHost(&h_i, NI);
    cudaMalloc(&d_s, 4096); cudaMallocHost(&h_s, 4096);
    cudaStream_t m, o;
    cudaStreamCreateWithFlags(&m, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&o, cudaStreamNonBlocking);
    cudaEvent_t t0, done, done2; cudaEventCreate(&t0); cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&done2, cudaEventDisableTiming);
    cudaStream_t sd, si; cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&si, cudaStreamNonBlocking);
    const int C = 6;
    cudaEvent_t h0[C], h1[C], o0[C], o1[C];
    for (int c = 0; c < C; ++c) { cudaEventCreate(&h0[c]); cudaEventCreate(&h1[c]); cudaEventCreate(&o0[c]); cudaEventCreate(&o1[c]); }
    cudaEventRecord(t0, m);
    bool have_done = false;
    for (int c = 0; c < C; ++c) {
        cudaStream_t hs = in_stream ? si : m;
        cudaEventRecord(h0[c], hs);
        cudaMemcpyAsync(d_i, h_i, NI, cudaMemcpyHostToDevice, hs);
        cudaEventRecord(h1[c], hs);
        if (in_stream) cudaStreamWaitEvent(m, h1[c], 0);
        if (use_wait && have_done) cudaStreamWaitEvent(m, done, 0);
        if (use_kernel) spin<<<148, 128, 0, m>>>(400000);
        if (small == 1) cudaMemcpyAsync(h_s, d_s, 4096, cudaMemcpyDeviceToHost, m);
        if (small == 2) {
            cudaEventRecord(done2, m);
            cudaStreamWaitEvent(sd, done2, 0);
            cudaMemcpyAsync(h_s, d_s, 4096, cudaMemcpyDeviceToHost, sd);
            cudaStreamSynchronize(sd);
        }
        cudaStreamSynchronize(m);
        cudaEventRecord(o0[c], o);
        cudaMemcpyAsync(h_o, d_o, NO, cudaMemcpyDeviceToHost, o);
        cudaEventRecord(o1[c], o);
        cudaEventRecord(done, o);
        have_done = true;
    }
    cudaDeviceSynchronize();
    for (int c = 0; c < C; ++c) {
        float a, b, x, y;
        cudaEventElapsedTime(&a, t0, h0[c]); cudaEventElapsedTime(&b, t0, h1[c]);
        cudaEventElapsedTime(&x, t0, o0[c]); cudaEventElapsedTime(&y, t0, o1[c]);
        printf("in=%d small=%d wait=%d kernel=%d chunk %d: h2d %.3f-%.3f  d2h %.3f-%.3f\n", in_stream, small, use_wait, use_kernel, c, a, b, x, y);
    }
}
