// Online decoding for n = k + 1 (App. C).
// One "wave" = at most one completion event per group.  k_online_est applies the update rule
// to the estimates (HBM-bound, float4 over d), k_online_state then advances the per-group
// received / finalised masks.  Two kernels, so every thread of the first reads the state from
// before the wave.  State word: bits 0..k = tasks received, bits 32..32+k-1 = finalised.
#include "ci_internal.h"

namespace ci {
namespace {

__device__ __forceinline__ bool event_applies(uint64_t st, int j, int k, bool& dup) {
    const uint32_t R = (uint32_t)st;
    dup = (R >> j) & 1u;
    return !dup && __popc(R) < k;   // already decoded: nothing changes
}

template <bool VEC>
__global__ void __launch_bounds__(256) k_online_est(float* __restrict__ est, const uint64_t* __restrict__ state,
                                                    const int32_t* __restrict__ task,
                                                    const float* __restrict__ value, int k, int64_t B,
                                                    int64_t dv, int* __restrict__ flag) {
    const float fk = (float)k;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < B * dv;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = idx / dv, e = idx - b * dv;
        const int j = __ldg(task + b);
        if (j < 0 || j > k) continue;
        const uint64_t st = __ldg(state + b);
        bool dup;
        if (!event_applies(st, j, k, dup)) {
            if (dup && e == 0) atomicAdd(flag, 1);
            continue;
        }
        const uint32_t F = (uint32_t)(st >> 32);
        if (VEC) {
            const float4 v = reinterpret_cast<const float4*>(value)[b * dv + e];
            float4* g = reinterpret_cast<float4*>(est) + b * k * dv + e;
            for (int i = 0; i < k; i++) {
                if ((F >> i) & 1u) continue;
                if (j < k) {
                    if (i == j) { g[i * dv] = v; continue; }
                    float4 t = g[i * dv];
                    t.x = __fsub_rn(t.x, v.x); t.y = __fsub_rn(t.y, v.y); t.z = __fsub_rn(t.z, v.z); t.w = __fsub_rn(t.w, v.w);
                    g[i * dv] = t;
                } else {
                    float4 t = g[i * dv];
                    t.x = __fmaf_rn(fk, v.x, t.x); t.y = __fmaf_rn(fk, v.y, t.y);
                    t.z = __fmaf_rn(fk, v.z, t.z); t.w = __fmaf_rn(fk, v.w, t.w);
                    g[i * dv] = t;
                }
            }
        } else {
            const float v = value[b * dv + e];
            float* g = est + b * k * dv + e;
            for (int i = 0; i < k; i++) {
                if ((F >> i) & 1u) continue;
                if (j < k) g[i * dv] = i == j ? v : __fsub_rn(g[i * dv], v);
                else g[i * dv] = __fmaf_rn(fk, v, g[i * dv]);
            }
        }
    }
}

__global__ void k_online_state(uint64_t* __restrict__ state, const int32_t* __restrict__ task, int k, int64_t B) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x) {
        const int j = task[b];
        if (j < 0 || j > k) continue;
        uint64_t st = state[b];
        bool dup;
        if (dup = ((uint32_t)st >> j) & 1u, dup) continue;
        uint32_t R = (uint32_t)st | (1u << j), F = (uint32_t)(st >> 32);
        if (__popc((uint32_t)st) < k) {
            if (j < k) F |= 1u << j;
            if (__popc(R) == k) F = (k >= 32) ? 0xFFFFFFFFu : ((1u << k) - 1u);
        }
        state[b] = ((uint64_t)F << 32) | R;
    }
}
}  // namespace

cudaError_t launch_online_update(int k, int64_t B, int64_t d, float* est, uint64_t* state, const int32_t* task,
                                 const float* value, int* flag, cudaStream_t s) {
    if (B == 0) return cudaSuccess;
    const bool vec = d % 4 == 0;
    const int64_t dv = vec ? d / 4 : d;
    int64_t g = (B * dv + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    if (vec) k_online_est<true><<<(unsigned)g, 256, 0, s>>>(est, state, task, value, k, B, dv, flag);
    else k_online_est<false><<<(unsigned)g, 256, 0, s>>>(est, state, task, value, k, B, dv, flag);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_online_state<<<(unsigned)std::min<int64_t>((B + 255) / 256, 148 * 8), 256, 0, s>>>(state, task, k, B);
    count_launch();
    return cudaGetLastError();
}

}  // namespace ci
