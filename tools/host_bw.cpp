// host_bw -- host-memory write bandwidth of the machine the GPU hangs off, regular stores vs
// non-temporal (streaming) stores, by thread count.  The host-buffer path (into.cu) expands
// packed outputs into the caller's buffers with host threads; this is its ceiling.
//
//   g++ -O3 -pthread tools/host_bw.cpp -o /tmp/host_bw && /tmp/host_bw
#include <emmintrin.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double run(int threads, size_t bytes, uint8_t* buf, int mode) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> ts;
    for (int t = 0; t < threads; ++t)
        ts.emplace_back([=] {
            const size_t a = bytes * t / threads & ~size_t{63}, b = bytes * (t + 1) / threads & ~size_t{63};
            if (mode == 0) {
                std::memset(buf + a, t + 1, b - a);
            } else {
                const __m128i v = _mm_set1_epi8((char)(t + 1));
                for (size_t i = a; i < b; i += 64) {
                    _mm_stream_si128((__m128i*)(buf + i), v);
                    _mm_stream_si128((__m128i*)(buf + i + 16), v);
                    _mm_stream_si128((__m128i*)(buf + i + 32), v);
                    _mm_stream_si128((__m128i*)(buf + i + 48), v);
                }
                _mm_sfence();
            }
        });
    for (auto& t : ts) t.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int main() {
    const size_t bytes = size_t{1} << 30;
    uint8_t* buf = (uint8_t*)std::aligned_alloc(64, bytes);
    std::memset(buf, 0, bytes);
    const unsigned hw = std::thread::hardware_concurrency();
    std::printf("hardware threads %u\n", hw);
    for (int threads : {1, 2, 4, 8, 12, 16})
        for (int mode : {0, 1}) {
            double best = 1e9;
            for (int r = 0; r < 3; ++r) best = std::min(best, run(threads, bytes, buf, mode));
            std::printf("threads %2d %-9s %6.1f GB/s\n", threads, mode ? "streaming" : "memset", bytes / best / 1e9);
        }
    std::free(buf);
}
