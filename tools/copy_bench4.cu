// copy_bench4 -- D2H bandwidth into the same pinned region repeatedly vs cycling through a large
// pinned buffer (IOMMU/IOTLB reach), for cudaMallocHost and for THP-backed + cudaHostRegister.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
int main() {
    const size_t piece = 24 << 20, big = size_t(1) << 30;
    void* d; cudaMalloc(&d, piece);
    void* hm; cudaMallocHost(&hm, big);
    void* ht = nullptr; posix_memalign(&ht, 2 << 20, big); madvise(ht, big, MADV_HUGEPAGE); memset(ht, 0, big);
    cudaHostRegister(ht, big, cudaHostRegisterDefault);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const char* names[2] = {"cudaMallocHost", "THP+HostRegister"};
    void* bufs[2] = {hm, ht};
    for (int k = 0; k < 2; ++k)
        for (int cyc = 0; cyc < 2; ++cyc) {
            const int n = 40;
            cudaEventRecord(a, s);
            for (int i = 0; i < n; ++i) {
                const size_t off = cyc ? (size_t)(i % (big / piece)) * piece : 0;
                cudaMemcpyAsync((char*)bufs[k] + off, d, piece, cudaMemcpyDeviceToHost, s);
            }
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("%-18s %-8s %.1f GB/s\n", names[k], cyc ? "cycling" : "same", n * piece / ms / 1e6);
        }
    char line[256]; FILE* f = fopen("/sys/kernel/mm/transparent_hugepage/enabled", "r");
    if (f && fgets(line, sizeof line, f)) printf("THP: %s", line);
}
