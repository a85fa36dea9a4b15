// filter.cu -- connected-operator filtering of a labeled image's component table
// (analysis.hpp:89-125 filter_components), SURVEY §8(f) first "next" row.
//
// The reference walks the components in ascending id (parents before children): a component
// merges into target[parent] when its parent merged, else into its parent when selected.  So
// a merged component's target is the parent of the HIGHEST selected component on its path to
// the exterior.  On the device that is pointer jumping over the parent map, carrying for each
// component the pair (ancestor a, highest selected component on [c, a)); combining two
// consistent pairs keeps the upper segment's choice.  Survivors then accumulate the features
// of the components they absorb (global atomics), and the tables are written per component.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "runlab_gpu.h"

using namespace rlg;

namespace {

constexpr uint32_t NONE = 0xFFFFFFFFu;

__device__ __forceinline__ unsigned long long pack(uint32_t anc, uint32_t best) {
    return ((unsigned long long)anc << 32) | best;
}

__global__ void k_filt_init(const rl_component* __restrict__ comps, int64_t n, const uint8_t* __restrict__ sel,
                            unsigned long long* st, uint32_t* flags) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
        if (c == 0) {
            st[0] = pack(0, NONE);
            if (sel[0]) flags[1] = 1;  // the exterior may not be selected (analysis.hpp:92-94)
        } else {
            st[c] = pack(comps[c].parent, sel[c] ? (uint32_t)c : NONE);
        }
    }
}

// one jump for every component; flags[0] = some ancestor is still above the exterior
__global__ void k_filt_jump(int64_t n, unsigned long long* st, uint32_t* flags) {
    int more = 0;
    for (int64_t c = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long v = st[c];
        const uint32_t a = (uint32_t)(v >> 32);
        if (a == 0) continue;
        const unsigned long long w = st[a];
        const uint32_t bw = (uint32_t)w, nb = bw != NONE ? bw : (uint32_t)v;
        const uint32_t na = (uint32_t)(w >> 32);
        st[c] = pack(na, nb);
        more |= na != 0;
    }
    if (__syncthreads_or(more) && threadIdx.x == 0) flags[0] = 1;
}

__global__ void k_filt_targets(const rl_component* __restrict__ comps, int64_t n, const unsigned long long* st,
                               uint32_t* parent_out, rl_features* feat_out) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t b = (uint32_t)st[c];
        parent_out[c] = b != NONE ? comps[b].parent : (uint32_t)c;
        feat_out[c] = comps[c].f;
    }
}

// survivors absorb the (own) features of the components merged into them (analysis.hpp:108-110)
__global__ void k_filt_fold(const rl_component* __restrict__ comps, int64_t n, const uint32_t* parent_out,
                            rl_features* feat_out) {
    for (int64_t c = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t t = parent_out[c];
        if (t != (uint32_t)c) acc_atomic_fold(feat_out + t, comps[c].f);
    }
}

// adjacency of components that are still roots, redirected into survivors (analysis.hpp:117-121)
__global__ void k_filt_adjacency(const rl_component* __restrict__ comps, int64_t n, const uint32_t* parent_out,
                                 uint32_t* adj_out) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
        if (c == 0) {
            adj_out[0] = NONE;
            continue;
        }
        const uint32_t pr = comps[c].parent;
        adj_out[c] = (parent_out[c] == (uint32_t)c && parent_out[pr] != pr) ? parent_out[pr] : pr;
    }
}

int grid_n(int64_t n) { return (int)(n / 256 + 1 < 148 * 16 ? n / 256 + 1 : 148 * 16); }

}  // namespace

extern "C" int rl_filter_components(void* stream, const rl_component* d_comps, int64_t n, const uint8_t* d_selected,
                                    uint32_t* d_parent, rl_features* d_features, uint32_t* d_adjacency) {
    if (n < 1 || !d_comps || !d_selected || !d_parent || !d_features || !d_adjacency) return RL_EINVAL;
    if (n >= (int64_t)NONE) return RL_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long* st = nullptr;
    uint32_t* flags = nullptr;
    if (cudaMallocAsync(&st, (size_t)n * 8, s) != cudaSuccess || cudaMallocAsync(&flags, 8, s) != cudaSuccess) {
        cudaGetLastError();
        return RL_ENOMEM;
    }
    int rc = RL_OK;
    uint32_t h[2] = {0, 0};
    cudaMemsetAsync(flags, 0, 8, s);
    k_filt_init<<<grid_n(n), 256, 0, s>>>(d_comps, n, d_selected, st, flags);
    // pointer jumping: rounds double the covered path; check every other round
    for (int round = 0; round < 64; round += 2) {
        cudaMemsetAsync(flags, 0, 4, s);
        k_filt_jump<<<grid_n(n), 256, 0, s>>>(n, st, flags);
        k_filt_jump<<<grid_n(n), 256, 0, s>>>(n, st, flags);
        cudaMemcpyAsync(h, flags, 8, cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) {
            rc = RL_ECUDA;
            break;
        }
        if (h[1]) {
            rc = RL_EINVAL;
            break;
        }
        if (!h[0]) break;
    }
    if (rc == RL_OK) {
        k_filt_targets<<<grid_n(n), 256, 0, s>>>(d_comps, n, st, d_parent, d_features);
        k_filt_fold<<<grid_n(n), 256, 0, s>>>(d_comps, n, d_parent, d_features);
        k_filt_adjacency<<<grid_n(n), 256, 0, s>>>(d_comps, n, d_parent, d_adjacency);
    }
    cudaFreeAsync(st, s);
    cudaFreeAsync(flags, s);
    if (cudaStreamSynchronize(s) != cudaSuccess && rc == RL_OK) rc = RL_ECUDA;
    return rc;
}

// host-buffer variant (the C++ drop-in's filter_components)
extern "C" int rl_filter_components_host(const rl_component* comps, int64_t n, const uint8_t* selected,
                                         uint32_t* parent, rl_features* features, uint32_t* adjacency) {
    if (n < 1 || !comps || !selected || !parent || !features || !adjacency) return RL_EINVAL;
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        return RL_ECUDA;
    }
    uint8_t* d = nullptr;
    const size_t bc = (size_t)n * sizeof(rl_component), bf = (size_t)n * sizeof(rl_features);
    const size_t total = bc + bf + (size_t)n * 9 + 64;
    int rc = RL_OK;
    if (cudaMallocAsync(&d, total, s) != cudaSuccess) {
        cudaGetLastError();
        cudaStreamDestroy(s);
        return RL_ENOMEM;
    }
    rl_component* d_comps = reinterpret_cast<rl_component*>(d);
    rl_features* d_feat = reinterpret_cast<rl_features*>(d + bc);
    uint32_t* d_parent = reinterpret_cast<uint32_t*>(d + bc + bf);
    uint32_t* d_adj = d_parent + n;
    uint8_t* d_sel = reinterpret_cast<uint8_t*>(d_adj + n);
    cudaMemcpyAsync(d_comps, comps, bc, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d_sel, selected, (size_t)n, cudaMemcpyHostToDevice, s);
    rc = rl_filter_components(s, d_comps, n, d_sel, d_parent, d_feat, d_adj);
    if (rc == RL_OK) {
        cudaMemcpyAsync(parent, d_parent, (size_t)n * 4, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(adjacency, d_adj, (size_t)n * 4, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(features, d_feat, bf, cudaMemcpyDeviceToHost, s);
    }
    cudaFreeAsync(d, s);
    if (cudaStreamSynchronize(s) != cudaSuccess && rc == RL_OK) rc = RL_ECUDA;
    cudaStreamDestroy(s);
    return rc;
}
