// Stage-boundary layouts for the TS stage kernels: the 2x2 squeeze psi between stages
// (pixel_unshuffle channel order) applied while an image's state moves
// between global memory and shared memory, instead of a separate permutation pass.
//
// Element g (0 .. C H W - 1) of one image in global memory, for a stage whose state is [C][H][W]
// in shared memory (index ch H W + y W + x):
//   layout 0: [C][H][W]                 (the stage's own layout)
//   layout 1: [C/4][2H][2W]             (the previous stage's layout: psi is applied on load,
//                                        psi^-1 on store)
//   layout 2: [4C][H/2][W/2]            (the next stage's layout: psi^-1 on load, psi on store)
#pragma once
#include <stdint.h>

namespace ci {

template <int C, int H, int W>
__device__ __forceinline__ int io_smem_index(int layout, int g) {
    constexpr int HW = H * W;
    if (layout == 1) {   // g = c' (4HW) + Y (2W) + X  ->  ch = 4c' + 2(Y&1) + (X&1), y = Y/2, x = X/2
        const int cq = g / (4 * HW), rem = g - cq * (4 * HW), Y = rem / (2 * W), X = rem - Y * (2 * W);
        return (4 * cq + 2 * (Y & 1) + (X & 1)) * HW + (Y >> 1) * W + (X >> 1);
    }
    if (layout == 2) {   // g = C4 (HW/4) + Y' (W/2) + X'  ->  ch = C4/4, y = 2Y' + (C4/2 & 1), x = 2X' + (C4 & 1)
        const int c4 = g / (HW / 4), rem = g - c4 * (HW / 4), Y = rem / (W / 2), X = rem - Y * (W / 2);
        return (c4 >> 2) * HW + (2 * Y + ((c4 >> 1) & 1)) * W + 2 * X + (c4 & 1);
    }
    return g;
}

// global -> shared (one image), layout of the global copy; threads t of nt, float4 loads
template <int C, int H, int W>
__device__ __forceinline__ void io_load(const float* __restrict__ src, int layout, float* st, int t, int nt) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    for (int q = t; q < C * H * W / 4; q += nt) {
        const float4 v = __ldcg(s4 + q);
        if (layout == 0) {
            reinterpret_cast<float4*>(st)[q] = v;
        } else {
            st[io_smem_index<C, H, W>(layout, 4 * q + 0)] = v.x;
            st[io_smem_index<C, H, W>(layout, 4 * q + 1)] = v.y;
            st[io_smem_index<C, H, W>(layout, 4 * q + 2)] = v.z;
            st[io_smem_index<C, H, W>(layout, 4 * q + 3)] = v.w;
        }
    }
}

// shared -> global (one image) in `layout`, float4 stores
template <int C, int H, int W>
__device__ __forceinline__ void io_store(float* __restrict__ dst, int layout, const float* st, int t, int nt) {
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (int q = t; q < C * H * W / 4; q += nt) {
        float4 v;
        if (layout == 0) {
            v = reinterpret_cast<const float4*>(st)[q];
        } else {
            v.x = st[io_smem_index<C, H, W>(layout, 4 * q + 0)];
            v.y = st[io_smem_index<C, H, W>(layout, 4 * q + 1)];
            v.z = st[io_smem_index<C, H, W>(layout, 4 * q + 2)];
            v.w = st[io_smem_index<C, H, W>(layout, 4 * q + 3)];
        }
        __stcg(d4 + q, v);
    }
}

// global -> shared with cp.async (completes on cp.async.wait_all): 16-B copies in layout 0,
// 4-B copies to the permuted positions otherwise
template <int C, int H, int W>
__device__ __forceinline__ void io_fetch_async(const float* __restrict__ src, int layout, float* st, int t, int nt) {
    if (layout == 0) {
        for (int q = t; q < C * H * W / 4; q += nt)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(st + 4 * q)),
                         "l"(src + 4 * q)
                         : "memory");
    } else {
        for (int g = t; g < C * H * W; g += nt)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(st + io_smem_index<C, H, W>(layout, g))),
                         "l"(src + g)
                         : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

}  // namespace ci
