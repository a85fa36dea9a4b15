// Microbenchmark: shared-memory load/store/atomic throughput on the GPU (per SM).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/ubench_smem.cu -o /tmp/ubench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int MODE>
__global__ void k(uint32_t* out, int stride) {
    __shared__ uint32_t s32[8192];  // 32 KB
    __shared__ unsigned long long s64[2048];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) s32[i] = i;
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s64[i] = i;
    __syncthreads();
    uint32_t acc = 0;
    uint32_t idx = (threadIdx.x * stride) & 4095;
    for (int it = 0; it < ITERS; ++it) {
        if (MODE == 0) acc += s32[(idx + it) & 8191];                          // LDS
        if (MODE == 1) s32[(idx + it * 33) & 8191] = it;                       // STS
        if (MODE == 2) atomicAdd(&s32[(idx + it * 33) & 8191], 1u);            // ATOMS add spread
        if (MODE == 3) atomicMin(&s32[(idx + it * 33) & 8191], (uint32_t)it);  // ATOMS min spread
        if (MODE == 4) atomicAdd(&s64[(idx + it * 33) & 2047], 1ull);          // ATOMS add 64
        if (MODE == 5) atomicAdd(&s32[it & 7], 1u);                            // same address
        if (MODE == 6) acc += atomicMin(&s32[(idx + it * 33) & 8191], (uint32_t)it);  // with return
    }
    if (acc == 0xFFFFFFFF) out[0] = acc;
    if (MODE == 1 || MODE >= 2) { __syncthreads(); if (threadIdx.x == 0) out[blockIdx.x] = s32[blockIdx.x & 8191]; }
}

int main() {
    uint32_t* out;
    cudaMalloc(&out, 1 << 20);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char* names[] = {"LDS", "STS", "ATOMS.ADD spread", "ATOMS.MIN spread", "ATOMS.ADD.64 spread",
                           "ATOMS.ADD same-8", "ATOMS.MIN ret"};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 7; ++mode) {
        for (int bpsm : {1, 4}) {
            const int blocks = sms * bpsm, threads = 256;
            auto launch = [&] {
                switch (mode) {
                    case 0: k<0><<<blocks, threads>>>(out, 1); break;
                    case 1: k<1><<<blocks, threads>>>(out, 1); break;
                    case 2: k<2><<<blocks, threads>>>(out, 1); break;
                    case 3: k<3><<<blocks, threads>>>(out, 1); break;
                    case 4: k<4><<<blocks, threads>>>(out, 1); break;
                    case 5: k<5><<<blocks, threads>>>(out, 1); break;
                    case 6: k<6><<<blocks, threads>>>(out, 1); break;
                }
            };
            launch();
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double ops = (double)blocks * threads * ITERS;  // lane-ops
            const double cyc = ms * 1e-3 * 1.965e9;                 // at max clock
            printf("%-22s warps/SM=%2d  %8.3f ms  lane-ops/cycle/SM = %6.2f\n", names[mode], bpsm * 8, ms,
                   ops / sms / cyc);
        }
    }
    return 0;
}
