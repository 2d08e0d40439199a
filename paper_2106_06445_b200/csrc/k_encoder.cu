// Light learned encoder (Arch E, CI_ENC_LEARNED): the CUDA-core parts around
// the conv->ReLU->conv tail (which runs on tcgen05 through the fused stage kernel,
// umma_encoder_tail):
//   k_enc_e1_mean : m[b] = (1/k) sum_i ReLU(conv3x3(E1, x_{b,i}))  -- weight-shared first layer on
//                   every input, averaged after it; also writes psi(m), the tail's
//                   input.  fp32, summation over i ascending.
//   k_enc_out     : x_p = conv3x3(E4, psi^-1(z) + m)  -- the U-Net-style skip fused into E4.
// One CTA of 256 threads owns one group's whole image (H x W <= 1024 pixels); a thread computes
// PX = 4 horizontally adjacent output pixels, so each 3 x 6 input window it reads from shared
// memory feeds 4 x 9 taps.  The image sits in shared memory with a zero halo that is written
// once per CTA (the interior positions never change): E1 streams the k inputs through two
// buffers with 16-byte cp.async (input i+1 lands while input i is convolved); E4 builds
// u = psi^-1(z) + m there.  The weights live in the kernel parameter space (the constant bank):
// the inner loops are FFMA with constant operands + LDS.
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

constexpr int kEncThreads = 256, kEncPx = 4;

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Shared-memory image layout of one channel: (H + 2) rows of RS floats; the interior pixel (y, x)
// sits at row y + 1, column x + 4 (16-byte aligned rows for cp.async), columns 3 and W + 4 are
// the zero halo.  The 3x6 window of output pixels x0..x0+3 starts at column x0 + 3.
template <int W>
struct EncTile {
    static constexpr int RS = W + 8;
    __host__ __device__ static constexpr int plane(int H) { return (H + 2) * RS; }
};

template <int CI, int C1, int W>
__global__ void __launch_bounds__(kEncThreads, 2) k_enc_e1_mean(const float* __restrict__ x, int k, int64_t B,
                                                               int H, const __grid_constant__ E1Params<CI, C1> p,
                                                               float* __restrict__ m, float* __restrict__ zpsi,
                                                               int64_t zstride) {
    extern __shared__ __align__(16) float xs[];   // [2][CI][H + 2][RS]
    constexpr int RS = EncTile<W>::RS, WQ = W / kEncPx, W4 = W / 4;
    const int plane = EncTile<W>::plane(H), tileN = CI * plane;
    const int HW = H * W, Ho = H / 2, Wo = W / 2;
    const int r = threadIdx.x / WQ, x0 = (threadIdx.x % WQ) * kEncPx;
    const bool act = r < H;
    const float fk = (float)k;
    for (int e = threadIdx.x; e < 2 * tileN; e += kEncThreads) xs[e] = 0.f;   // halo (and interior)
    const int nvec = CI * H * W4;   // 16-byte interior chunks per input
    for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
        auto load = [&](int i, int buf) {
            const float* xi = x + (b * k + i) * (int64_t)CI * HW;
            float* dst = xs + buf * tileN;
            for (int v = threadIdx.x; v < nvec; v += kEncThreads) {
                const int c = v / (H * W4), rem = v - c * (H * W4), y = rem / W4, xq = rem - y * W4;
                cp_async16(dst + c * plane + (y + 1) * RS + 4 + xq * 4, xi + c * HW + y * W + xq * 4);
            }
            cp_async_commit();
        };
        __syncthreads();   // the previous group's readers are done with both buffers
        load(0, 0);
        float sum[C1][kEncPx];
#pragma unroll
        for (int o = 0; o < C1; o++)
#pragma unroll
            for (int q = 0; q < kEncPx; q++) sum[o][q] = 0.f;
        for (int i = 0; i < k; i++) {
            if (i + 1 < k) {
                load(i + 1, (i + 1) & 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            if (act) {
                const float* t = xs + (i & 1) * tileN + r * RS + x0 + 3;
                float in[CI][3][kEncPx + 2];
#pragma unroll
                for (int c = 0; c < CI; c++)
#pragma unroll
                    for (int u = 0; u < 3; u++)
#pragma unroll
                        for (int j = 0; j < kEncPx + 2; j++) in[c][u][j] = t[c * plane + u * RS + j];
#pragma unroll
                for (int o = 0; o < C1; o++) {
#pragma unroll
                    for (int q = 0; q < kEncPx; q++) {
                        float acc = 0.f;   // taps in (c, u, v) order, then the bias
#pragma unroll
                        for (int c = 0; c < CI; c++)
#pragma unroll
                            for (int u = 0; u < 3; u++)
#pragma unroll
                                for (int v = 0; v < 3; v++)
                                    acc = fmaf(p.w[((o * CI + c) * 3 + u) * 3 + v], in[c][u][q + v], acc);
                        sum[o][q] = __fadd_rn(sum[o][q], fmaxf(acc + p.b[o], 0.f));
                    }
                }
            }
            __syncthreads();   // buffer i & 1 is refilled by the next iteration's prefetch
        }
        if (act) {
            float* zb = zpsi + b * zstride;
#pragma unroll
            for (int o = 0; o < C1; o++) {
                float mv[kEncPx];
#pragma unroll
                for (int q = 0; q < kEncPx; q++) mv[q] = __fdiv_rn(sum[o][q], fk);
                *reinterpret_cast<float4*>(m + (b * C1 + o) * HW + r * W + x0) = make_float4(mv[0], mv[1], mv[2], mv[3]);
                // psi: pixel (y, x) -> channel 4o + 2(y&1) + (x&1) at (y/2, x/2); x0 is even
                float* z0 = zb + ((int64_t)(o * 4 + 2 * (r & 1)) * Ho + (r >> 1)) * Wo + (x0 >> 1);
                *reinterpret_cast<float2*>(z0) = make_float2(mv[0], mv[2]);
                *reinterpret_cast<float2*>(z0 + (int64_t)Ho * Wo) = make_float2(mv[1], mv[3]);
            }
        }
    }
}

// u = psi^-1(z) + m in shared memory [C1][H+2][RS] (zero halo), then
// x_p[o] = b[o] + sum_{c,u,v} E4[o][c][u][v] u[c][y+u-1][x+v-1]
template <int CI, int C1, int W>
__global__ void __launch_bounds__(kEncThreads, 2) k_enc_out(const float* __restrict__ z, int64_t zstride,
                                                           const float* __restrict__ m, int64_t B, int H,
                                                           const __grid_constant__ E4Params<CI, C1> p,
                                                           float* __restrict__ xp) {
    extern __shared__ __align__(16) float us[];
    constexpr int RS = EncTile<W>::RS, WQ = W / kEncPx;
    const int plane = EncTile<W>::plane(H), tileN = C1 * plane;
    const int HW = H * W, Ho = H / 2, Wo = W / 2;
    const int r = threadIdx.x / WQ, x0 = (threadIdx.x % WQ) * kEncPx;
    for (int e = threadIdx.x; e < tileN; e += kEncThreads) us[e] = 0.f;   // halo (and interior)
    constexpr int W4 = W / 4;
    const int nquad = C1 * H * W4;   // 4-pixel runs (x % 4 == 0): one float4 of m, one float2 of each z plane
    for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
        const float* zb = z + b * zstride;
        const float* mb = m + b * (int64_t)C1 * HW;
        __syncthreads();   // the previous group's readers are done
        constexpr int U = 8;   // runs in flight per thread (3 loads each)
        for (int v0 = threadIdx.x; v0 < nquad; v0 += U * kEncThreads) {
            float4 mv[U];
            float2 z0[U], z1[U];
#pragma unroll
            for (int j = 0; j < U; j++) {
                const int v = v0 + j * kEncThreads;
                if (v < nquad) {
                    const int c = v / (H * W4), rem = v - c * (H * W4), y = rem / W4, xq = rem - y * W4;
                    mv[j] = *reinterpret_cast<const float4*>(mb + c * HW + y * W + 4 * xq);
                    // psi^-1: pixel (y, x) of channel c is z[4c + 2(y&1) + (x&1)][y/2][x/2]
                    const float* zr = zb + ((int64_t)(c * 4 + 2 * (y & 1)) * Ho + (y >> 1)) * Wo + 2 * xq;
                    z0[j] = *reinterpret_cast<const float2*>(zr);                       // x even
                    z1[j] = *reinterpret_cast<const float2*>(zr + (int64_t)Ho * Wo);    // x odd
                }
            }
#pragma unroll
            for (int j = 0; j < U; j++) {
                const int v = v0 + j * kEncThreads;
                if (v < nquad) {
                    const int c = v / (H * W4), rem = v - c * (H * W4), y = rem / W4, xq = rem - y * W4;
                    float* d = us + c * plane + (y + 1) * RS + 4 + 4 * xq;
                    *reinterpret_cast<float4*>(d) =
                        make_float4(z0[j].x + mv[j].x, z1[j].x + mv[j].y, z0[j].y + mv[j].z, z1[j].y + mv[j].w);
                }
            }
        }
        __syncthreads();
        if (r < H) {
            float acc[CI][kEncPx];
#pragma unroll
            for (int o = 0; o < CI; o++)
#pragma unroll
                for (int q = 0; q < kEncPx; q++) acc[o][q] = 0.f;
            const float* t = us + r * RS + x0 + 3;
#pragma unroll
            for (int c = 0; c < C1; c++) {
                float win[3][kEncPx + 2];
#pragma unroll
                for (int u = 0; u < 3; u++)
#pragma unroll
                    for (int j = 0; j < kEncPx + 2; j++) win[u][j] = t[c * plane + u * RS + j];
#pragma unroll
                for (int o = 0; o < CI; o++)
#pragma unroll
                    for (int q = 0; q < kEncPx; q++)
#pragma unroll
                        for (int u = 0; u < 3; u++)
#pragma unroll
                            for (int v = 0; v < 3; v++)
                                acc[o][q] = fmaf(p.w[((o * C1 + c) * 3 + u) * 3 + v], win[u][q + v], acc[o][q]);
            }
            float* ob = xp + b * (int64_t)CI * HW + r * W + x0;
#pragma unroll
            for (int o = 0; o < CI; o++)   // identity activation on the encoder output
                *reinterpret_cast<float4*>(ob + o * HW) =
                    make_float4(acc[o][0] + p.b[o], acc[o][1] + p.b[o], acc[o][2] + p.b[o], acc[o][3] + p.b[o]);
        }
    }
}

bool enc_supported(int Ci, int C1, int H, int W) {
    return Ci == 3 && (C1 == 4 || C1 == 8 || C1 == 16) && (W == 8 || W == 16 || W == 32) && H % 2 == 0 && H >= 2 &&
           H * W <= kEncThreads * kEncPx;
}

static int enc_grid(int64_t B) { return (int)std::max<int64_t>(1, std::min<int64_t>(B, 148 * 4)); }

template <int CI, int C1, int W>
static cudaError_t e1_t(const float* x, int k, int64_t B, int H, const float* hw1, const float* hb1, float* m,
                        float* zpsi, int64_t zstride, cudaStream_t s) {
    E1Params<CI, C1> p;
    memcpy(p.w, hw1, sizeof(p.w));
    memcpy(p.b, hb1, sizeof(p.b));
    const size_t smem = sizeof(float) * 2 * CI * EncTile<W>::plane(H);
    k_enc_e1_mean<CI, C1, W><<<enc_grid(B), kEncThreads, smem, s>>>(x, k, B, H, p, m, zpsi, zstride);
    return cudaGetLastError();
}

template <int CI, int C1>
static cudaError_t e1_w(const float* x, int k, int64_t B, int H, int W, const float* hw1, const float* hb1, float* m,
                        float* zpsi, int64_t zstride, cudaStream_t s) {
    if (W == 32) return e1_t<CI, C1, 32>(x, k, B, H, hw1, hb1, m, zpsi, zstride, s);
    if (W == 16) return e1_t<CI, C1, 16>(x, k, B, H, hw1, hb1, m, zpsi, zstride, s);
    if (W == 8) return e1_t<CI, C1, 8>(x, k, B, H, hw1, hb1, m, zpsi, zstride, s);
    return cudaErrorInvalidValue;
}

cudaError_t launch_enc_e1_mean(const float* x, int k, int64_t B, int Ci, int H, int W, const float* hw1,
                               const float* hb1, int C1, float* m, float* zpsi, int64_t zstride, cudaStream_t s) {
    if (B == 0) return cudaSuccess;
    cudaError_t e = cudaErrorInvalidValue;
    if (Ci == 3 && C1 == 16) e = e1_w<3, 16>(x, k, B, H, W, hw1, hb1, m, zpsi, zstride, s);
    else if (Ci == 3 && C1 == 8) e = e1_w<3, 8>(x, k, B, H, W, hw1, hb1, m, zpsi, zstride, s);
    else if (Ci == 3 && C1 == 4) e = e1_w<3, 4>(x, k, B, H, W, hw1, hb1, m, zpsi, zstride, s);
    count_launch();
    return e;
}

template <int CI, int C1, int W>
static cudaError_t out_t(const float* z, int64_t zstride, const float* m, int64_t B, int H, const float* hw4,
                         const float* hb4, float* xp, cudaStream_t s) {
    E4Params<CI, C1> p;
    memcpy(p.w, hw4, sizeof(p.w));
    memcpy(p.b, hb4, sizeof(p.b));
    const size_t smem = sizeof(float) * C1 * EncTile<W>::plane(H);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_enc_out<CI, C1, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    k_enc_out<CI, C1, W><<<enc_grid(B), kEncThreads, smem, s>>>(z, zstride, m, B, H, p, xp);
    return cudaGetLastError();
}

template <int CI, int C1>
static cudaError_t out_w(const float* z, int64_t zstride, const float* m, int64_t B, int H, int W, const float* hw4,
                         const float* hb4, float* xp, cudaStream_t s) {
    if (W == 32) return out_t<CI, C1, 32>(z, zstride, m, B, H, hw4, hb4, xp, s);
    if (W == 16) return out_t<CI, C1, 16>(z, zstride, m, B, H, hw4, hb4, xp, s);
    if (W == 8) return out_t<CI, C1, 8>(z, zstride, m, B, H, hw4, hb4, xp, s);
    return cudaErrorInvalidValue;
}

cudaError_t launch_enc_out(const float* z, int64_t zstride, const float* m, int64_t B, int Ci, int C1, int H, int W,
                           const float* hw4, const float* hb4, float* xp, cudaStream_t s) {
    if (B == 0) return cudaSuccess;
    cudaError_t e = cudaErrorInvalidValue;
    if (Ci == 3 && C1 == 16) e = out_w<3, 16>(z, zstride, m, B, H, W, hw4, hb4, xp, s);
    else if (Ci == 3 && C1 == 8) e = out_w<3, 8>(z, zstride, m, B, H, W, hw4, hb4, xp, s);
    else if (Ci == 3 && C1 == 4) e = out_w<3, 4>(z, zstride, m, B, H, W, hw4, hb4, xp, s);
    count_launch();
    return e;
}

}  // namespace ci
