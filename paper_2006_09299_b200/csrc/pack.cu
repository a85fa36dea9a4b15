// pack.cu -- device side of the compact component slots (pack.cuh) for rl_label_into.
//
// Both kernels run at the end of the captured pipeline, after the component count of the batch
// is known on the device (cbase[B]); their escape counts land in the summary row B + 1, which
// the pipeline's last copy brings to the host with the rest of the summary.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "pack.cuh"

namespace rlg {
namespace {

__device__ __forceinline__ rlp::Slot esc_slot(uint32_t k) { return rlp::Slot{k, 0u, rlp::ESC, 0u}; }

__device__ __forceinline__ void store_slot(rlp::Slot* p, const rlp::Slot& o) {
    *reinterpret_cast<uint4*>(p) = make_uint4(o.x, o.y, o.z, o.w);
}

// pre-fill records: slots[i] + parent[i]; records that do not fit go to esc[]
__global__ void k_pack_comps(const rl_component* __restrict__ comps, const uint64_t* __restrict__ total_p,
                             uint64_t cap, rlp::Slot* __restrict__ slots, uint32_t* __restrict__ parent,
                             rl_component* __restrict__ esc, unsigned long long* nesc) {
    const uint64_t total = *total_p;
    if (total > cap) return;  // components overflowed (nothing was emitted): the host re-runs
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const rl_component c = comps[i];
        rlp::Slot o;
        if (!rlp::encode(c.f, c.flags, o)) {
            const uint32_t k = (uint32_t)atomicAdd(nesc, 1ull);
            esc[k] = c;
            o = esc_slot(k);
        }
        store_slot(slots + i, o);
        parent[i] = c.parent;
    }
}

// post-fill features of the survivors (rank order, cf. k_compact_filled)
__global__ void k_pack_filled(const Acc* __restrict__ filled, const uint32_t* __restrict__ flag,
                              const uint32_t* __restrict__ rank, const uint64_t* __restrict__ total_p, uint64_t cap,
                              rlp::Slot* __restrict__ slots, Acc* __restrict__ esc, unsigned long long* nesc) {
    const uint64_t total = *total_p;
    if (total > cap) return;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        if (!flag[i]) continue;
        const Acc f = filled[i];
        rlp::Slot o;
        if (!rlp::encode(f, 0u, o)) {
            const uint32_t k = (uint32_t)atomicAdd(nesc, 1ull);
            esc[k] = f;
            o = esc_slot(k);
        }
        store_slot(slots + rank[i], o);
    }
}

int grid_of(uint64_t n, int sms) {
    const uint64_t g = n / 256 + 1, m = (uint64_t)sms * 8;
    return (int)(g < m ? g : m);
}

}  // namespace

void launch_pack_comps(const rl_component* comps, const uint64_t* total_p, uint64_t cap, void* slots, uint32_t* parent,
                       rl_component* esc, int64_t* nesc, cudaStream_t s, int sms) {
    k_pack_comps<<<grid_of(cap, sms), 256, 0, s>>>(comps, total_p, cap, static_cast<rlp::Slot*>(slots), parent, esc,
                                                   reinterpret_cast<unsigned long long*>(nesc));
}

void launch_pack_filled(const Acc* filled, const uint32_t* flag, const uint32_t* rank, const uint64_t* total_p,
                        uint64_t cap, void* slots, Acc* esc, int64_t* nesc, cudaStream_t s, int sms) {
    k_pack_filled<<<grid_of(cap, sms), 256, 0, s>>>(filled, flag, rank, total_p, cap, static_cast<rlp::Slot*>(slots),
                                                    esc, reinterpret_cast<unsigned long long*>(nesc));
}

}  // namespace rlg
