// Light learned encoder (Arch E, CI_ENC_LEARNED): the CUDA-core parts around
// the conv->ReLU->conv tail (which runs on tcgen05 through the fused stage kernel,
// umma_encoder_tail):
//   k_enc_e1_mean : m[b] = (1/k) sum_i ReLU(conv3x3(E1, x_{b,i}))  -- weight-shared first layer on
//                   every input, averaged after it; also writes psi(m), the tail's
//                   input.  fp32, summation over i ascending.
//   k_enc_out     : x_p = conv3x3(E4, psi^-1(z) + m)  -- the U-Net-style skip fused into E4: the
//                   CTA of group b builds u = psi^-1(z) + m in shared memory, then every thread
//                   computes the in_c outputs of four pixels (no u round trip through HBM).
// Both hold their (small) weights in the kernel parameter space -- the constant bank, so every
// FFMA reads its weight as an immediate constant-bank operand: no load instruction per MAC.
#include "ci_internal.h"

namespace ci {

template <int CI, int C1>
struct E1Params {
    float w[C1 * CI * 9];   // [C1][CI][3][3]
    float b[C1];
};
template <int CI, int C1>
struct E4Params {
    float w[CI * C1 * 9];   // [CI][C1][3][3]
    float b[CI];
};

// thread -> 4 horizontally adjacent pixels of group b's image plane, all C1 channels
template <int CI, int C1>
__global__ void __launch_bounds__(256) k_enc_e1_mean(const float* __restrict__ x, int k, int64_t B, int H, int W,
                                                     const __grid_constant__ E1Params<CI, C1> p,
                                                     float* __restrict__ m, float* __restrict__ zpsi,
                                                     int64_t zstride) {
    constexpr int PX = 4;
    const int64_t HW = (int64_t)H * W;
    const int Ho = H / 2, Wo = W / 2, wq = W / PX;
    const float fk = (float)k;
    const int64_t units = B * (int64_t)H * wq;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < units; u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = u / ((int64_t)H * wq);
        const int r = (int)(u - b * H * wq);
        const int y = r / wq, x0 = (r - y * wq) * PX;
        float sum[C1][PX];
#pragma unroll
        for (int o = 0; o < C1; o++)
#pragma unroll
            for (int q = 0; q < PX; q++) sum[o][q] = 0.f;
        for (int i = 0; i < k; i++) {
            const float* xi = x + (b * k + i) * CI * HW;
            float in[CI][3][PX + 2];   // rows y-1..y+1, columns x0-1 .. x0+PX (zero outside)
#pragma unroll
            for (int c = 0; c < CI; c++)
#pragma unroll
                for (int uu = 0; uu < 3; uu++) {
                    const int yy = y + uu - 1;
                    const bool rowok = yy >= 0 && yy < H;
#pragma unroll
                    for (int j = 0; j < PX + 2; j++) {
                        const int xx = x0 + j - 1;
                        in[c][uu][j] = (rowok && xx >= 0 && xx < W) ? __ldg(xi + c * HW + yy * W + xx) : 0.f;
                    }
                }
#pragma unroll
            for (int o = 0; o < C1; o++) {
#pragma unroll
                for (int q = 0; q < PX; q++) {
                    float acc = 0.f;   // taps in (c, u, v) order, then the bias
#pragma unroll
                    for (int c = 0; c < CI; c++)
#pragma unroll
                        for (int uu = 0; uu < 3; uu++)
#pragma unroll
                            for (int v = 0; v < 3; v++) acc = fmaf(p.w[((o * CI + c) * 3 + uu) * 3 + v], in[c][uu][q + v], acc);
                    sum[o][q] = __fadd_rn(sum[o][q], fmaxf(acc + p.b[o], 0.f));
                }
            }
        }
        float* zb = zpsi + b * zstride;
#pragma unroll
        for (int o = 0; o < C1; o++) {
            float mv[PX];
#pragma unroll
            for (int q = 0; q < PX; q++) mv[q] = __fdiv_rn(sum[o][q], fk);
            *reinterpret_cast<float4*>(m + (b * C1 + o) * HW + y * W + x0) = make_float4(mv[0], mv[1], mv[2], mv[3]);
            // psi: pixel (y, x) -> channel 4o + 2(y&1) + (x&1) at (y/2, x/2); x0 is even
            float* z0 = zb + ((int64_t)(o * 4 + 2 * (y & 1)) * Ho + (y >> 1)) * Wo + (x0 >> 1);
            *reinterpret_cast<float2*>(z0) = make_float2(mv[0], mv[2]);
            *reinterpret_cast<float2*>(z0 + (int64_t)Ho * Wo) = make_float2(mv[1], mv[3]);
        }
    }
}

// one CTA per group (grid-stride): u = psi^-1(z) + m in shared memory [C1][H+2][W+2] (zero
// border), then x_p[o] = b[o] + sum_{c,u,v} E4[o][c][u][v] u[c][y+u-1][x+v-1]
template <int CI, int C1>
__global__ void __launch_bounds__(256) k_enc_out(const float* __restrict__ z, int64_t zstride,
                                                 const float* __restrict__ m, int64_t B, int H, int W,
                                                 const __grid_constant__ E4Params<CI, C1> p, float* __restrict__ xp) {
    constexpr int PX = 4;
    extern __shared__ float us[];
    const int Hp = H + 2, Wp = W + 2;
    const int64_t HW = (int64_t)H * W;
    const int Ho = H / 2, Wo = W / 2;
    for (int i = threadIdx.x; i < C1 * Hp * Wp; i += blockDim.x) us[i] = 0.f;
    for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
        __syncthreads();   // the previous group's reads are done
        const float* zb = z + b * zstride;
        const float* mb = m + b * C1 * HW;
        for (int i = threadIdx.x; i < C1 * (int)HW; i += blockDim.x) {   // m-order: coalesced m reads
            const int c = i / (int)HW, rem = i - c * (int)HW, y = rem / W, xx = rem - y * W;
            const float zv = zb[((int64_t)(c * 4 + 2 * (y & 1) + (xx & 1)) * Ho + (y >> 1)) * Wo + (xx >> 1)];
            us[(c * Hp + y + 1) * Wp + xx + 1] = zv + mb[i];
        }
        __syncthreads();
        const int wq = W / PX;
        for (int t = threadIdx.x; t < H * wq; t += blockDim.x) {
            const int y = t / wq, x0 = (t - y * wq) * PX;
            float acc[CI][PX];
#pragma unroll
            for (int o = 0; o < CI; o++)
#pragma unroll
                for (int q = 0; q < PX; q++) acc[o][q] = 0.f;
#pragma unroll 4
            for (int c = 0; c < C1; c++) {
                float win[3][PX + 2];
#pragma unroll
                for (int uu = 0; uu < 3; uu++)
#pragma unroll
                    for (int j = 0; j < PX + 2; j++) win[uu][j] = us[(c * Hp + y + uu) * Wp + x0 + j];
#pragma unroll
                for (int o = 0; o < CI; o++)
#pragma unroll
                    for (int q = 0; q < PX; q++)
#pragma unroll
                        for (int uu = 0; uu < 3; uu++)
#pragma unroll
                            for (int v = 0; v < 3; v++) acc[o][q] = fmaf(p.w[((o * C1 + c) * 3 + uu) * 3 + v], win[uu][q + v], acc[o][q]);
            }
            float* ob = xp + b * CI * HW + y * W + x0;
#pragma unroll
            for (int o = 0; o < CI; o++)   // identity activation on the encoder output
                *reinterpret_cast<float4*>(ob + o * HW) =
                    make_float4(acc[o][0] + p.b[o], acc[o][1] + p.b[o], acc[o][2] + p.b[o], acc[o][3] + p.b[o]);
        }
    }
}

static int grid_of(int64_t total, int block) {
    int64_t g = (total + block - 1) / block;
    if (g > 148 * 32) g = 148 * 32;
    return (int)(g < 1 ? 1 : g);
}

bool enc_supported(int Ci, int C1, int H, int W) {
    return Ci == 3 && (C1 == 4 || C1 == 8 || C1 == 16) && W % 4 == 0 && H % 2 == 0 &&
           (size_t)C1 * (H + 2) * (W + 2) * sizeof(float) <= 200 * 1024;
}

template <int CI, int C1>
static cudaError_t e1_t(const float* x, int k, int64_t B, int H, int W, const float* hw1, const float* hb1, float* m,
                        float* zpsi, int64_t zstride, cudaStream_t s) {
    E1Params<CI, C1> p;
    memcpy(p.w, hw1, sizeof(p.w));
    memcpy(p.b, hb1, sizeof(p.b));
    k_enc_e1_mean<CI, C1><<<grid_of(B * (int64_t)H * (W / 4), 256), 256, 0, s>>>(x, k, B, H, W, p, m, zpsi, zstride);
    return cudaGetLastError();
}

cudaError_t launch_enc_e1_mean(const float* x, int k, int64_t B, int Ci, int H, int W, const float* hw1,
                               const float* hb1, int C1, float* m, float* zpsi, int64_t zstride, cudaStream_t s) {
    if (B == 0) return cudaSuccess;
    cudaError_t e = cudaErrorInvalidValue;
    if (Ci == 3 && C1 == 16) e = e1_t<3, 16>(x, k, B, H, W, hw1, hb1, m, zpsi, zstride, s);
    else if (Ci == 3 && C1 == 8) e = e1_t<3, 8>(x, k, B, H, W, hw1, hb1, m, zpsi, zstride, s);
    else if (Ci == 3 && C1 == 4) e = e1_t<3, 4>(x, k, B, H, W, hw1, hb1, m, zpsi, zstride, s);
    count_launch();
    return e;
}

template <int CI, int C1>
static cudaError_t out_t(const float* z, int64_t zstride, const float* m, int64_t B, int H, int W, const float* hw4,
                         const float* hb4, float* xp, cudaStream_t s) {
    E4Params<CI, C1> p;
    memcpy(p.w, hw4, sizeof(p.w));
    memcpy(p.b, hb4, sizeof(p.b));
    const size_t smem = (size_t)C1 * (H + 2) * (W + 2) * sizeof(float);
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_enc_out<CI, C1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int grid = (int)std::min<int64_t>(B, 148 * 3);
    k_enc_out<CI, C1><<<grid, 256, smem, s>>>(z, zstride, m, B, H, W, p, xp);
    return cudaGetLastError();
}

cudaError_t launch_enc_out(const float* z, int64_t zstride, const float* m, int64_t B, int Ci, int C1, int H, int W,
                           const float* hw4, const float* hb4, float* xp, cudaStream_t s) {
    if (B == 0) return cudaSuccess;
    cudaError_t e = cudaErrorInvalidValue;
    if (Ci == 3 && C1 == 16) e = out_t<3, 16>(z, zstride, m, B, H, W, hw4, hb4, xp, s);
    else if (Ci == 3 && C1 == 8) e = out_t<3, 8>(z, zstride, m, B, H, W, hw4, hb4, xp, s);
    else if (Ci == 3 && C1 == 4) e = out_t<3, 4>(z, zstride, m, B, H, W, hw4, hb4, xp, s);
    count_launch();
    return e;
}

}  // namespace ci
