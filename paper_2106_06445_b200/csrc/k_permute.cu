// Stage-boundary permutations of the fp32 state: psi (space-to-depth r = 2, torch
// pixel_unshuffle order), psi^-1 and the identity copy (i-RevNet's squeeze).
#include "ci_internal.h"

namespace ci {

// mode 1 psi: in [C][H][W] -> out [4C][H/2][W/2], out[c*4+2dy+dx][y][x] = in[c][2y+dy][2x+dx]
// mode 2 psi^-1: in [C4][Ho][Wo] -> out [C4/4][2Ho][2Wo] (exact inverse of mode 1)
// mode 0 identity copy.  One thread per SOURCE element (coalesced reads).
__global__ void k_permute(const float* __restrict__ in, float* __restrict__ out, int64_t total,
                          int C, int H, int W, int mode) {
    const int64_t per = (int64_t)C * H * W;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t img = idx / per;
        int64_t r = idx - img * per;
        int c = (int)(r / (H * W));
        int rem = (int)(r - (int64_t)c * H * W);
        int i = rem / W, j = rem - (rem / W) * W;
        int64_t o;
        if (mode == 1) {
            int Ho = H >> 1, Wo = W >> 1;
            int oc = c * 4 + 2 * (i & 1) + (j & 1);
            o = ((int64_t)oc * Ho + (i >> 1)) * Wo + (j >> 1);
        } else if (mode == 2) {
            int oc = c >> 2, dy = (c >> 1) & 1, dx = c & 1;
            int Hn = H * 2, Wn = W * 2;
            o = ((int64_t)oc * Hn + 2 * i + dy) * Wn + 2 * j + dx;
        } else {
            o = r;
        }
        out[img * per + o] = in[idx];
    }
}

// Vectorised stage-boundary permutation: one thread per 4 consecutive elements of a row.
//   mode 0: copy (float4);  mode 1 (psi): a float4 of source row (c, i) splits into its even /
//   odd columns -> float2 stores into channels 4c + 2(i&1) + {0, 1};  mode 2 (psi^-1): a float4 of
//   destination row (c, 2y+dy) interleaves float2 loads of source channels 4c + 2dy + {0, 1}.
//   C, H, W: the SOURCE shape; requires W % 4 == 0 (mode 0/1) or 2W % 4 == 0 (mode 2).
__global__ void __launch_bounds__(256) k_permute4(const float* __restrict__ in, float* __restrict__ out,
                                                  int64_t units, int C, int H, int W, int mode) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < units;
         u += (int64_t)gridDim.x * blockDim.x) {
        if (mode == 0) {
            reinterpret_cast<float4*>(out)[u] = __ldcs(reinterpret_cast<const float4*>(in) + u);
        } else if (mode == 1) {
            const int w4 = W >> 2;
            const int64_t row = u / w4;               // (img, c, i)
            const int j = (int)(u - row * w4) * 4;
            const int i = (int)(row % H);
            const int64_t ic = row / H;               // img * C + c
            const int64_t img = ic / C;
            const int c = (int)(ic - img * C);
            const int Ho = H >> 1, Wo = W >> 1;
            const float4 v = __ldcs(reinterpret_cast<const float4*>(in) + u);
            const int oc = c * 4 + 2 * (i & 1);
            float* ob = out + ((img * (int64_t)(4 * C) + oc) * Ho + (i >> 1)) * Wo + (j >> 1);
            __stcs(reinterpret_cast<float2*>(ob), make_float2(v.x, v.z));
            __stcs(reinterpret_cast<float2*>(ob + (int64_t)Ho * Wo), make_float2(v.y, v.w));
        } else {
            // destination shape [C/4][2H][2W]; u indexes destination float4s
            const int Wn = W * 2, Hn = H * 2, w4 = Wn >> 2;
            const int64_t row = u / w4;               // (img, oc, yy)
            const int x = (int)(u - row * w4) * 4;
            const int yy = (int)(row % Hn);
            const int64_t ioc = row / Hn;             // img * C/4 + oc
            const int Cq = C >> 2;
            const int64_t img = ioc / Cq;
            const int oc = (int)(ioc - img * Cq);
            const int c0 = oc * 4 + 2 * (yy & 1);
            const float* s0 = in + ((img * (int64_t)C + c0) * H + (yy >> 1)) * W + (x >> 1);
            const float2 a = __ldcs(reinterpret_cast<const float2*>(s0));
            const float2 b = __ldcs(reinterpret_cast<const float2*>(s0 + (int64_t)H * W));
            __stcs(reinterpret_cast<float4*>(out) + u, make_float4(a.x, b.x, a.y, b.y));
        }
    }
}

cudaError_t launch_permute(const float* in, float* out, int64_t n, int C, int H, int W, int mode,
                           cudaStream_t s) {
    int64_t total = n * (int64_t)C * H * W;
    if (total == 0) return cudaSuccess;
    const bool aligned = (reinterpret_cast<uintptr_t>(in) % 16 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
    const bool vec = aligned && (mode == 2 ? (2 * W) % 4 == 0 && C % 4 == 0 : W % 4 == 0) &&
                     (mode != 1 || (H % 2 == 0));
    if (vec) {
        const int64_t units = total / 4;
        int64_t blocks = (units + 255) / 256;
        if (blocks > 148 * 16) blocks = 148 * 16;
        k_permute4<<<(unsigned)blocks, 256, 0, s>>>(in, out, units, C, H, W, mode);
        count_launch();
        return cudaGetLastError();
    }
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    k_permute<<<(unsigned)blocks, 256, 0, s>>>(in, out, total, C, H, W, mode);
    count_launch();
    return cudaGetLastError();
}

}  // namespace ci
