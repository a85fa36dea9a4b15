// generate.cu -- device-side input generators (BASELINE configs), bit-identical to the
// reference's host generator.
//
//   rl_generate        generator.hpp:46-83: g x g blocks, FG iff splitmix64 block draw
//                      (generator.hpp:28-41) < density * 2^64; d = 1 accepts every draw.
//   rl_generate_rings  config 3 (new; SURVEY App. B interpretation, same recipe as the
//                      oracle's orc_generate_rings): nested square rings per tile + salt.
//   rl_cfg4_params     config 4 per-image (density, granularity) draws.
#include <cuda_runtime.h>

#include <cstdint>

#include "runlab_gpu.h"

namespace {

__host__ __device__ __forceinline__ uint64_t sm_step(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t block_draw(uint64_t seed, uint64_t br, uint64_t bc) {
    return sm_step(sm_step(sm_step(seed) ^ br) ^ bc);
}

// one thread per 16 pixels of a row (16-byte stores when the row is aligned)
// rows [y0, y0 + h) of the image (out holds just those rows)
__global__ void k_generate(uint8_t* out, int32_t w, int32_t h, int32_t g, uint64_t seed, uint64_t thr,
                           int always, int32_t y0) {
    const int32_t vpr = (w + 15) / 16;
    const int64_t total = (int64_t)vpr * h;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t yo = (int32_t)(i / vpr), y = y0 + yo;
        const int32_t x0 = (int32_t)(i % vpr) * 16;
        const uint64_t sr = sm_step(sm_step(seed) ^ (uint64_t)(y / g));
        uint8_t v[16];
        int32_t last_bc = -1;
        uint8_t last = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int32_t x = x0 + k;
            const int32_t bc = x / g;
            if (bc != last_bc) {
                last = (always || sm_step(sr ^ (uint64_t)bc) < thr) ? 1 : 0;
                last_bc = bc;
            }
            v[k] = x < w ? last : 0;
        }
        uint8_t* dst = out + (int64_t)yo * w + x0;
        if ((w % 16) == 0 && (reinterpret_cast<uintptr_t>(out) % 16) == 0) {
            uint4 q;
            q.x = v[0] | (v[1] << 8) | (v[2] << 16) | ((uint32_t)v[3] << 24);
            q.y = v[4] | (v[5] << 8) | (v[6] << 16) | ((uint32_t)v[7] << 24);
            q.z = v[8] | (v[9] << 8) | (v[10] << 16) | ((uint32_t)v[11] << 24);
            q.w = v[12] | (v[13] << 8) | (v[14] << 16) | ((uint32_t)v[15] << 24);
            *reinterpret_cast<uint4*>(dst) = q;
        } else {
            for (int k = 0; k < 16 && x0 + k < w; ++k) dst[k] = v[k];
        }
    }
}

// config 3: rings, one thread per pixel
__global__ void k_rings(uint8_t* out, int32_t w, int32_t h, int32_t tile, uint64_t seed, uint64_t salt_thr,
                        int salt) {
    const int64_t total = (int64_t)w * h;
    const int32_t ntc = (w + tile - 1) / tile;
    const int32_t half = tile / 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t y = (int32_t)(i / w), x = (int32_t)(i % w);
        const int32_t tr = y / tile, tc = x / tile;
        const int32_t ly = y - tr * tile, lx = x - tc * tile;
        const uint64_t tile_id = (uint64_t)tr * (uint64_t)ntc + (uint64_t)tc;
        const int32_t k = 1 + (int32_t)(block_draw(seed, (uint64_t)tr, (uint64_t)tc) % 16u);
        // distance of the pixel to the tile border (square annuli)
        int32_t d = ly;
        d = min(d, lx);
        d = min(d, tile - 1 - ly);
        d = min(d, tile - 1 - lx);
        uint8_t v = 0;
        int32_t off = 1;
        for (int32_t r = 0; r < k; ++r) {
            const int32_t rw = 1 + (int32_t)(block_draw(seed ^ 0xABCDull, tile_id, (uint64_t)r) % 3u);
            if (off + rw > half) break;
            if (d >= off && d < off + rw) {
                v = (r & 1) == 0 ? 1 : 0;
                break;
            }
            off += rw;
        }
        if (salt && block_draw(seed ^ 0x5A17ull, (uint64_t)y, (uint64_t)x) < salt_thr) v ^= 1;
        out[i] = v;
    }
}

int grid_of(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 32) g = 148 * 32;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" {

// generator.hpp:46-83 on the device; d_out holds w*h bytes; stream = cudaStream_t or NULL
int rl_generate_rows(void* stream, uint8_t* d_out, int32_t w, int32_t h, int32_t y0, int32_t rows, double density,
                     int32_t g, uint64_t seed) {
    if (w < 1 || h < 1 || y0 < 0 || rows < 1 || y0 + rows > h) return RL_EINVAL;
    if (density < 0.0 || density > 1.0) return RL_EINVAL;
    if (g < 1 || g > (w < h ? w : h)) return RL_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    if (density <= 0.0) return cudaMemsetAsync(d_out, 0, (size_t)w * rows, s) == cudaSuccess ? RL_OK : RL_ECUDA;
    const double scaled = density * 18446744073709551616.0;
    const int always = scaled >= 18446744073709551616.0;
    const uint64_t thr = always ? 0 : (uint64_t)scaled;
    const int64_t n = (int64_t)((w + 15) / 16) * rows;
    k_generate<<<grid_of(n), 256, 0, s>>>(d_out, w, rows, g, seed, thr, always, y0);
    return cudaGetLastError() == cudaSuccess ? RL_OK : RL_ECUDA;
}

int rl_generate(void* stream, uint8_t* d_out, int32_t w, int32_t h, double density, int32_t g, uint64_t seed) {
    return rl_generate_rows(stream, d_out, w, h, 0, h, density, g, seed);
}

// host-buffer variant (generated on the device, copied back)
int rl_generate_host(uint8_t* out, int32_t w, int32_t h, double density, int32_t g, uint64_t seed) {
    if (!out || w < 1 || h < 1) return RL_EINVAL;
    uint8_t* d = nullptr;
    const size_t n = (size_t)w * h;
    if (cudaMalloc(&d, n) != cudaSuccess) {
        cudaGetLastError();
        return RL_ENOMEM;
    }
    int rc = rl_generate(nullptr, d, w, h, density, g, seed);
    if (rc == RL_OK && cudaMemcpy(out, d, n, cudaMemcpyDeviceToHost) != cudaSuccess) rc = RL_ECUDA;
    cudaFree(d);
    return rc;
}

int rl_generate_rings(void* stream, uint8_t* d_out, int32_t w, int32_t h, int32_t tile, uint64_t seed,
                      double salt) {
    if (w < 1 || h < 1 || tile < 4 || salt < 0.0 || salt >= 1.0) return RL_EINVAL;
    const uint64_t thr = (uint64_t)(salt * 18446744073709551616.0);
    k_rings<<<grid_of((int64_t)w * h), 256, 0, (cudaStream_t)stream>>>(d_out, w, h, tile, seed, thr, salt > 0.0);
    return cudaGetLastError() == cudaSuccess ? RL_OK : RL_ECUDA;
}

void rl_cfg4_params(uint64_t i, double* density, int32_t* g) {
    *density = 0.1 + 0.8 * ((double)(block_draw(42, i, 0) >> 11) * (1.0 / 9007199254740992.0));
    *g = 1 + (int32_t)(block_draw(42, i, 1) % 8u);
}

}  // extern "C"
