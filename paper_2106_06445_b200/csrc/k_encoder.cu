// Light learned encoder (Arch E, CI_ENC_LEARNED): the parts that are not plain 3x3 convs.
//   k_enc_e1_mean  : m[b] = (1/k) sum_i ReLU(conv3x3(E1, x_{b,i}))  -- weight-shared first layer
//                    on every input, averaged after it; fp32, ascending i.
//   k_unsqueeze_add: u = psi^-1(z) + m  (U-Net-style skip, SURVEY Arch E)
// E2, E3, E4 run through the fp32 direct-convolution kernel (launch_conv_simt): the encoder
// is ~2% of the C4 FLOPs.
#include "ci_internal.h"

namespace ci {

__global__ void k_enc_e1_mean(const float* __restrict__ x, int k, int64_t B, int Ci, int H, int W,
                              const float* __restrict__ W1, const float* __restrict__ b1, int C1,
                              float* __restrict__ m) {
    const int64_t HW = (int64_t)H * W;
    const int64_t total = B * C1 * HW;
    const float fk = (float)k;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = idx / (C1 * HW);
        const int r = (int)(idx - b * C1 * HW);
        const int o = r / (int)HW;
        const int rem = r - o * (int)HW;
        const int i0 = rem / W, j0 = rem - (rem / W) * W;
        const float* wo = W1 + (int64_t)o * Ci * 9;
        float sum = 0.f;
        for (int q = 0; q < k; q++) {
            const float* xq = x + ((b * k + q) * Ci) * HW;
            float acc = 0.f;
            for (int c = 0; c < Ci; c++) {
                const float* xc = xq + c * HW;
                const float* wc = wo + c * 9;
#pragma unroll
                for (int u = -1; u <= 1; u++) {
                    const int ii = i0 + u;
                    if (ii < 0 || ii >= H) continue;
#pragma unroll
                    for (int v = -1; v <= 1; v++) {
                        const int jj = j0 + v;
                        if (jj < 0 || jj >= W) continue;
                        acc = fmaf(__ldg(wc + (u + 1) * 3 + (v + 1)), xc[ii * W + jj], acc);
                    }
                }
            }
            sum = __fadd_rn(sum, fmaxf(acc + __ldg(b1 + o), 0.f));
        }
        m[idx] = __fdiv_rn(sum, fk);
    }
}

// u[b][c][y][x] = z[b][4c + 2(y&1) + (x&1)][y/2][x/2] + m[b][c][y][x]
__global__ void k_unsqueeze_add(const float* __restrict__ z, const float* __restrict__ m,
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
        u[idx] = z[((b * 4 * C + zc) * Ho + (y >> 1)) * Wo + (xx >> 1)] + m[idx];
    }
}

static int grid_of(int64_t total) {
    int64_t g = (total + 255) / 256;
    if (g > 148 * 32) g = 148 * 32;
    return (int)(g < 1 ? 1 : g);
}

cudaError_t launch_enc_e1_mean(const float* x, int k, int64_t B, int Ci, int H, int W, const float* W1,
                               const float* b1, int C1, float* m, cudaStream_t s) {
    const int64_t total = B * C1 * (int64_t)H * W;
    if (total == 0) return cudaSuccess;
    k_enc_e1_mean<<<grid_of(total), 256, 0, s>>>(x, k, B, Ci, H, W, W1, b1, C1, m);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_unsqueeze_add(const float* z, const float* m, float* u, int64_t B, int C, int H, int W,
                                 cudaStream_t s) {
    const int64_t total = B * C * (int64_t)H * W;
    if (total == 0) return cudaSuccess;
    k_unsqueeze_add<<<grid_of(total), 256, 0, s>>>(z, m, u, B, C, H, W);
    count_launch();
    return cudaGetLastError();
}

}  // namespace ci
