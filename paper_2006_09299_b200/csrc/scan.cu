// scan.cu -- single-pass exclusive prefix sum of u32 counts (decoupled look-back), used for the
// canonical-id offsets of the (image, row, tile column) cells and for the densify / compaction
// ranks.  One launch: each CTA scans a 4096-element block in registers and shared memory,
// publishes its block total, and gets the total of everything before it by walking back over the
// predecessors' published totals (a predecessor that already knows its inclusive prefix ends the
// walk).  Blocks take their index from an atomic ticket, so every predecessor of a running block
// has started: the walk cannot wait on a block that is not resident.
#include <cuda_runtime.h>

#include <cstdint>

#include "ctx.hpp"

namespace rlg {

namespace {

constexpr int SCAN_T = 256;              // threads per block
constexpr int SCAN_V = 4;                // uint4 vectors per thread
constexpr int SCAN_ITEMS = 4 * SCAN_V;   // elements per thread
constexpr int SCAN_BLOCK = SCAN_T * SCAN_ITEMS;

// status word of a block: (flag << 62) | value; flag 1 = block total, 2 = inclusive prefix
constexpr unsigned long long ST_AGG = 1ull << 62, ST_INC = 2ull << 62, ST_VAL = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// state[0] = ticket counter, state[1 + b] = status of block b (zeroed before the launch)
__global__ void __launch_bounds__(SCAN_T) k_scan(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                 int64_t n, uint32_t init, unsigned long long* state) {
    __shared__ uint32_t s_warp[SCAN_T / 32];
    __shared__ uint32_t s_prefix;
    __shared__ uint32_t s_block;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_block = (uint32_t)atomicAdd(state, 1ull);
    __syncthreads();
    const int64_t blk = s_block;
    const int64_t base = blk * SCAN_BLOCK + (int64_t)tid * SCAN_ITEMS;
    uint32_t v[SCAN_ITEMS];
    const bool full = base + SCAN_ITEMS <= n && ((reinterpret_cast<uintptr_t>(in) & 15) == 0) &&
                      ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
    if (full) {
#pragma unroll
        for (int k = 0; k < SCAN_V; ++k) {
            const uint4 q = __ldcs(reinterpret_cast<const uint4*>(in + base) + k);
            v[4 * k] = q.x;
            v[4 * k + 1] = q.y;
            v[4 * k + 2] = q.z;
            v[4 * k + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; ++k) v[k] = base + k < n ? in[base + k] : 0u;
    }
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) sum += v[k];
    // block-wide exclusive scan of the thread sums
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = lane < SCAN_T / 32 ? s_warp[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < SCAN_T / 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, wi, o);
            if (lane >= o) wi += t;
        }
        const uint32_t total = __shfl_sync(0xFFFFFFFFu, wi, SCAN_T / 32 - 1);
        if (lane < SCAN_T / 32) s_warp[lane] = wi - w;  // exclusive warp offsets
        // everything before this block: the predecessors' totals, walked back by lane 0
        uint32_t prefix = init;
        unsigned long long* st = state + 1;
        if (blk == 0) {
            if (lane == 0) st_status(st, ST_INC | (unsigned long long)(init + total));
        } else {
            if (lane == 0) st_status(st + blk, ST_AGG | total);
            uint32_t acc = 0;
            for (int64_t p = blk - 1;; p -= 32) {  // 32 predecessors per step, one per lane
                const int64_t q = p - lane;
                unsigned long long s = 0;
                if (q >= 0)
                    do s = ld_status(st + q);
                    while ((s & ~ST_VAL) == 0);
                else
                    s = ST_INC;  // before block 0: nothing (init is block 0's)
                const uint32_t inc_lanes = __ballot_sync(0xFFFFFFFFu, (s & ~ST_VAL) == ST_INC);
                // lanes up to and including the first one holding an inclusive prefix count
                const int stop = inc_lanes ? __ffs(inc_lanes) - 1 : 31;
                uint32_t val = lane <= stop && q >= 0 ? (uint32_t)(s & ST_VAL) : 0u;
                if (q < 0 && lane == stop) val = 0;
#pragma unroll
                for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(0xFFFFFFFFu, val, o);
                acc += val;
                if (inc_lanes) break;
            }
            prefix = acc;
            if (lane == 0) st_status(st + blk, ST_INC | (unsigned long long)(prefix + total));
        }
        if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();
    uint32_t run = s_prefix + s_warp[warp] + incl - sum;
    if (full) {
#pragma unroll
        for (int k = 0; k < SCAN_V; ++k) {
            uint4 q;
            q.x = run;
            run += v[4 * k];
            q.y = run;
            run += v[4 * k + 1];
            q.z = run;
            run += v[4 * k + 2];
            q.w = run;
            run += v[4 * k + 3];
            reinterpret_cast<uint4*>(out + base)[k] = q;
        }
    } else {
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; ++k) {
            if (base + k < n) out[base + k] = run;
            run += v[k];
        }
    }
}

}  // namespace

size_t scan_state_bytes(int64_t n) { return (size_t)(1 + (n + SCAN_BLOCK - 1) / SCAN_BLOCK) * 8; }

// out[i] = init + sum(in[0 .. i)), i < n; `state` holds scan_state_bytes(n) bytes of device memory
// (zeroed here unless the caller already did, `zeroed`)
void launch_scan(const uint32_t* in, uint32_t* out, int64_t n, uint32_t init, void* state, cudaStream_t s,
                 bool zeroed) {
    if (n <= 0) return;
    const int64_t blocks = (n + SCAN_BLOCK - 1) / SCAN_BLOCK;
    if (!zeroed) cudaMemsetAsync(state, 0, scan_state_bytes(n), s);
    k_scan<<<(unsigned)blocks, SCAN_T, 0, s>>>(in, out, n, init, static_cast<unsigned long long*>(state));
}

}  // namespace rlg
