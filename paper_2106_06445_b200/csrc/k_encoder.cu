// Light learned encoder (Arch E, CI_ENC_LEARNED): the parts that are not the conv->ReLU->conv
// tail (which runs on tcgen05 through the fused stage kernel, umma_encoder_tail):
//   k_enc_e1_mean  : m[b] = (1/k) sum_i ReLU(conv3x3(E1, x_{b,i}))  -- weight-shared first layer
//                    on every input, averaged after it; fp32, ascending i.  One
//                    thread per output pixel computes all C1 channels (inputs read once per
//                    image, register-tiled).  Also writes psi(m) into the encoder-tail buffer.
//   k_unsqueeze_add: u = psi^-1(z) + m  (U-Net-style skip, SURVEY Arch E)
// E4 (c1 -> in_c, ~1% of the encoder FLOPs) uses the fp32 direct-convolution kernel.
#include "ci_internal.h"

namespace ci {

template <int CI, int C1>
__global__ void __launch_bounds__(128) k_enc_e1_mean(const float* __restrict__ x, int k, int64_t B, int H, int W,
                                                     const float* __restrict__ W1, const float* __restrict__ b1,
                                                     float* __restrict__ m, float* __restrict__ zpsi,
                                                     int64_t zstride) {
    __shared__ float sw[C1 * CI * 9 + C1];
    for (int i = threadIdx.x; i < C1 * CI * 9 + C1; i += blockDim.x)
        sw[i] = i < C1 * CI * 9 ? W1[i] : b1[i - C1 * CI * 9];
    __syncthreads();
    const int64_t HW = (int64_t)H * W;
    const int Ho = H / 2, Wo = W / 2;
    const float fk = (float)k;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < B * HW;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = idx / HW;
        const int rem = (int)(idx - b * HW);
        const int y = rem / W, xx = rem - (rem / W) * W;
        float sum[C1];
#pragma unroll
        for (int o = 0; o < C1; o++) sum[o] = 0.f;
        for (int q = 0; q < k; q++) {
            const float* xq = x + (b * k + q) * CI * HW;
            float in[CI * 9];
#pragma unroll
            for (int c = 0; c < CI; c++)
#pragma unroll
                for (int u = 0; u < 3; u++)
#pragma unroll
                    for (int v = 0; v < 3; v++) {
                        const int ii = y + u - 1, jj = xx + v - 1;
                        in[(c * 3 + u) * 3 + v] =
                            (ii >= 0 && ii < H && jj >= 0 && jj < W) ? __ldg(xq + c * HW + ii * W + jj) : 0.f;
                    }
#pragma unroll
            for (int o = 0; o < C1; o++) {
                float acc = 0.f;
#pragma unroll
                for (int t = 0; t < CI * 9; t++) acc = fmaf(sw[o * CI * 9 + t], in[t], acc);
                sum[o] = __fadd_rn(sum[o], fmaxf(acc + sw[C1 * CI * 9 + o], 0.f));
            }
        }
        float* zb = zpsi + b * zstride;
#pragma unroll
        for (int o = 0; o < C1; o++) {
            const float mv = __fdiv_rn(sum[o], fk);
            m[(b * C1 + o) * HW + rem] = mv;
            zb[((int64_t)(o * 4 + 2 * (y & 1) + (xx & 1)) * Ho + (y >> 1)) * Wo + (xx >> 1)] = mv;
        }
    }
}

// generic fallback (any CI <= 4, C1 <= 32)
__global__ void k_enc_e1_mean_generic(const float* __restrict__ x, int k, int64_t B, int CI, int H, int W,
                                      const float* __restrict__ W1, const float* __restrict__ b1, int C1,
                                      float* __restrict__ m, float* __restrict__ zpsi, int64_t zstride) {
    const int64_t HW = (int64_t)H * W;
    const int Ho = H / 2, Wo = W / 2;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < B * C1 * HW;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = idx / (C1 * HW);
        const int r = (int)(idx - b * C1 * HW);
        const int o = r / (int)HW, rem = r - o * (int)HW;
        const int y = rem / W, xx = rem - (rem / W) * W;
        float sum = 0.f;
        for (int q = 0; q < k; q++) {
            const float* xq = x + (b * k + q) * CI * HW;
            float acc = 0.f;
            for (int c = 0; c < CI; c++)
                for (int u = -1; u <= 1; u++)
                    for (int v = -1; v <= 1; v++) {
                        const int ii = y + u, jj = xx + v;
                        if (ii < 0 || ii >= H || jj < 0 || jj >= W) continue;
                        acc = fmaf(W1[((o * CI + c) * 3 + u + 1) * 3 + v + 1], xq[c * HW + ii * W + jj], acc);
                    }
            sum = __fadd_rn(sum, fmaxf(acc + b1[o], 0.f));
        }
        const float mv = __fdiv_rn(sum, (float)k);
        m[idx] = mv;
        zpsi[b * zstride + ((int64_t)(o * 4 + 2 * (y & 1) + (xx & 1)) * Ho + (y >> 1)) * Wo + (xx >> 1)] = mv;
    }
}

// u[b][c][y][x] = z[b][4c + 2(y&1) + (x&1)][y/2][x/2] + m[b][c][y][x]   (z rows at zstride)
__global__ void k_unsqueeze_add(const float* __restrict__ z, int64_t zstride, const float* __restrict__ m,
                                float* __restrict__ u, int64_t B, int C, int H, int W) {
    const int64_t HW = (int64_t)H * W, total = B * C * HW;
    const int Ho = H / 2, Wo = W / 2;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = idx / (C * HW);
        const int r = (int)(idx - b * C * HW);
        const int c = r / (int)HW;
        const int rem = r - c * (int)HW;
        const int y = rem / W, xx = rem - (rem / W) * W;
        const int zc = c * 4 + 2 * (y & 1) + (xx & 1);
        u[idx] = z[b * zstride + ((int64_t)zc * Ho + (y >> 1)) * Wo + (xx >> 1)] + m[idx];
    }
}

static int grid_of(int64_t total, int block) {
    int64_t g = (total + block - 1) / block;
    if (g > 148 * 32) g = 148 * 32;
    return (int)(g < 1 ? 1 : g);
}

cudaError_t launch_enc_e1_mean(const float* x, int k, int64_t B, int Ci, int H, int W, const float* W1,
                               const float* b1, int C1, float* m, float* zpsi, int64_t zstride, cudaStream_t s) {
    const int64_t npix = B * (int64_t)H * W;
    if (npix == 0) return cudaSuccess;
    if (Ci == 3 && C1 == 16)
        k_enc_e1_mean<3, 16><<<grid_of(npix, 128), 128, 0, s>>>(x, k, B, H, W, W1, b1, m, zpsi, zstride);
    else if (Ci == 3 && C1 == 4)
        k_enc_e1_mean<3, 4><<<grid_of(npix, 128), 128, 0, s>>>(x, k, B, H, W, W1, b1, m, zpsi, zstride);
    else
        k_enc_e1_mean_generic<<<grid_of(npix * C1, 256), 256, 0, s>>>(x, k, B, Ci, H, W, W1, b1, C1, m, zpsi,
                                                                      zstride);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_unsqueeze_add(const float* z, int64_t zstride, const float* m, float* u, int64_t B, int C,
                                 int H, int W, cudaStream_t s) {
    const int64_t total = B * C * (int64_t)H * W;
    if (total == 0) return cudaSuccess;
    k_unsqueeze_add<<<grid_of(total, 256), 256, 0, s>>>(z, zstride, m, u, B, C, H, W);
    count_launch();
    return cudaGetLastError();
}

}  // namespace ci
