// Light learned encoder (Arch E, CI_ENC_LEARNED): the CUDA-core parts around
// the conv->ReLU->conv tail (which runs on tcgen05 through the fused stage kernel,
// umma_encoder_tail):
//   k_enc_e1_mean : m[b] = (1/k) sum_i ReLU(conv3x3(E1, x_{b,i}))  -- weight-shared first layer on
//                   every input, averaged after it; also writes psi(m), the tail's
//                   input.  fp32, summation over i ascending.
//   k_enc_out     : x_p = conv3x3(E4, psi^-1(z) + m)  -- the U-Net-style skip fused into E4.
// Both are band-tiled: a CTA of 256 threads owns one band of BR = 256 / W image rows of one group
// (one output pixel per thread).  The band's input window (BR + 2 rows incl. the 3x3 halo, zero
// padded) is staged in shared memory -- E1 double-buffers the k inputs with cp.async so input
// i+1 streams in while input i is convolved; E4 builds u = psi^-1(z) + m there.  The weights
// live in the kernel parameter space (the constant bank): every FFMA reads its weight as an
// immediate constant-bank operand, so the inner loops are FFMA + LDS only.
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

constexpr int kEncThreads = 256;

__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool ok) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(ok ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// rows per band: one pixel per thread
__host__ __device__ inline int enc_band_rows(int H, int W) { return min(kEncThreads / W, H); }

template <int CI, int C1>
__global__ void __launch_bounds__(kEncThreads, 4) k_enc_e1_mean(const float* __restrict__ x, int k, int64_t B, int H,
                                                            int W, const __grid_constant__ E1Params<CI, C1> p,
                                                            float* __restrict__ m, float* __restrict__ zpsi,
                                                            int64_t zstride) {
    extern __shared__ float xs[];   // [2][CI][BR + 2][W + 2]
    const int BR = enc_band_rows(H, W), nb = (H + BR - 1) / BR;
    const int Wp = W + 2, plane = (BR + 2) * Wp, tileN = CI * plane;
    const int64_t HW = (int64_t)H * W;
    const int Ho = H / 2, Wo = W / 2;
    const int r = threadIdx.x / W, xx = threadIdx.x - r * W;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float fk = (float)k;
    for (int64_t unit = blockIdx.x; unit < B * nb; unit += gridDim.x) {
        const int64_t b = unit / nb;
        const int y0 = (int)(unit - b * nb) * BR, y = y0 + r;
        const bool act = r < BR && y < H;
        auto load = [&](int i, int buf) {   // input i's band window, zero outside the image
            const float* xi = x + (b * k + i) * CI * HW;
            float* dst = xs + buf * tileN;
            // warp w fills window rows w, w + 8, ...; lanes walk the columns
            for (int row = warp; row < CI * (BR + 2); row += kEncThreads / 32) {
                const int c = row / (BR + 2), yy = y0 + row - c * (BR + 2) - 1;
                const bool rok = yy >= 0 && yy < H;
                const float* src = xi + c * HW + (int64_t)yy * W - 1;
                for (int cc = lane; cc < Wp; cc += 32) {
                    const bool ok = rok && cc >= 1 && cc <= W;
                    cp_async4(dst + row * Wp + cc, ok ? src + cc : xi, ok);
                }
            }
            cp_async_commit();
        };
        __syncthreads();   // the previous unit's readers are done with both buffers
        load(0, 0);
        float sum[C1];
#pragma unroll
        for (int o = 0; o < C1; o++) sum[o] = 0.f;
        for (int i = 0; i < k; i++) {
            if (i + 1 < k) {
                load(i + 1, (i + 1) & 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            if (act) {
                const float* t = xs + (i & 1) * tileN + r * Wp + xx;
                float in[CI][3][3];
#pragma unroll
                for (int c = 0; c < CI; c++)
#pragma unroll
                    for (int u = 0; u < 3; u++)
#pragma unroll
                        for (int v = 0; v < 3; v++) in[c][u][v] = t[c * plane + u * Wp + v];
#pragma unroll
                for (int o = 0; o < C1; o++) {
                    float acc = 0.f;   // taps in (c, u, v) order, then the bias
#pragma unroll
                    for (int c = 0; c < CI; c++)
#pragma unroll
                        for (int u = 0; u < 3; u++)
#pragma unroll
                            for (int v = 0; v < 3; v++) acc = fmaf(p.w[((o * CI + c) * 3 + u) * 3 + v], in[c][u][v], acc);
                    sum[o] = __fadd_rn(sum[o], fmaxf(acc + p.b[o], 0.f));
                }
            }
            __syncthreads();   // buffer i & 1 is refilled by the next iteration's prefetch
        }
        if (act) {
            float* zb = zpsi + b * zstride;
            // psi: pixel (y, x) -> channel 4o + 2(y&1) + (x&1) at (y/2, x/2)
            const int64_t zoff = ((int64_t)(2 * (y & 1) + (xx & 1)) * Ho + (y >> 1)) * Wo + (xx >> 1);
#pragma unroll
            for (int o = 0; o < C1; o++) {
                const float mv = __fdiv_rn(sum[o], fk);
                m[(b * C1 + o) * HW + y * W + xx] = mv;
                zb[(int64_t)o * 4 * Ho * Wo + zoff] = mv;
            }
        }
    }
}

// u = psi^-1(z) + m in shared memory [C1][BR+2][W+2] (zero border), then
// x_p[o] = b[o] + sum_{c,u,v} E4[o][c][u][v] u[c][y+u-1][x+v-1].  The z gather and the m rows
// stream in with cp.async (all of a thread's copies in flight at once: the fill is latency-,
// not bandwidth-bound), then one pass adds them in place.
template <int CI, int C1>
__global__ void __launch_bounds__(kEncThreads, 4) k_enc_out(const float* __restrict__ z, int64_t zstride,
                                                           const float* __restrict__ m, int64_t B, int H, int W,
                                                           const __grid_constant__ E4Params<CI, C1> p,
                                                           float* __restrict__ xp) {
    extern __shared__ float us[];   // [2][C1][BR + 2][W + 2]: psi^-1(z) window, m window
    const int BR = enc_band_rows(H, W), nb = (H + BR - 1) / BR;
    const int Wp = W + 2, plane = (BR + 2) * Wp, tileN = C1 * plane;
    float* ms = us + tileN;
    const int64_t HW = (int64_t)H * W;
    const int Ho = H / 2, Wo = W / 2;
    const int r = threadIdx.x / W, xx = threadIdx.x - r * W;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t unit = blockIdx.x; unit < B * nb; unit += gridDim.x) {
        const int64_t b = unit / nb;
        const int y0 = (int)(unit - b * nb) * BR, y = y0 + r;
        const float* zb = z + b * zstride;
        const float* mb = m + b * C1 * HW;
        __syncthreads();   // the previous unit's readers are done
        // warp w fills window rows w, w + 8, ...; lanes walk the columns (zero outside the image)
        for (int row = warp; row < C1 * (BR + 2); row += kEncThreads / 32) {
            const int c = row / (BR + 2), yy = y0 + row - c * (BR + 2) - 1;
            const bool rok = yy >= 0 && yy < H;
            const float* zr = zb + ((int64_t)(c * 4 + 2 * (yy & 1)) * Ho + (yy >> 1)) * Wo;   // + (x&1) plane
            const float* mr = mb + c * HW + (int64_t)yy * W;
            for (int cc = lane; cc < Wp; cc += 32) {
                const int xc = cc - 1;
                const bool ok = rok && xc >= 0 && xc < W;
                cp_async4(us + row * Wp + cc, ok ? zr + (int64_t)(xc & 1) * Ho * Wo + (xc >> 1) : zb, ok);
                cp_async4(ms + row * Wp + cc, ok ? mr + xc : mb, ok);
            }
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        for (int e = threadIdx.x; e < tileN; e += kEncThreads) us[e] += ms[e];
        __syncthreads();
        if (r < BR && y < H) {
            float acc[CI];
#pragma unroll
            for (int o = 0; o < CI; o++) acc[o] = 0.f;
            const float* t = us + r * Wp + xx;
#pragma unroll
            for (int c = 0; c < C1; c++) {
                float win[3][3];
#pragma unroll
                for (int u = 0; u < 3; u++)
#pragma unroll
                    for (int v = 0; v < 3; v++) win[u][v] = t[c * plane + u * Wp + v];
#pragma unroll
                for (int o = 0; o < CI; o++)
#pragma unroll
                    for (int u = 0; u < 3; u++)
#pragma unroll
                        for (int v = 0; v < 3; v++) acc[o] = fmaf(p.w[((o * C1 + c) * 3 + u) * 3 + v], win[u][v], acc[o]);
            }
#pragma unroll
            for (int o = 0; o < CI; o++)   // identity activation on the encoder output
                xp[(b * CI + o) * HW + y * W + xx] = acc[o] + p.b[o];
        }
    }
}

bool enc_supported(int Ci, int C1, int H, int W) {
    return Ci == 3 && (C1 == 4 || C1 == 8 || C1 == 16) && W >= 2 && W <= kEncThreads && kEncThreads % W == 0 &&
           H % 2 == 0 && W % 2 == 0;
}

// resident units: a few waves of 148 SMs, grid-stride beyond
static int enc_grid(int64_t units) { return (int)std::max<int64_t>(1, std::min<int64_t>(units, 148 * 16)); }

template <int CI, int C1>
static cudaError_t e1_t(const float* x, int k, int64_t B, int H, int W, const float* hw1, const float* hb1, float* m,
                        float* zpsi, int64_t zstride, cudaStream_t s) {
    E1Params<CI, C1> p;
    memcpy(p.w, hw1, sizeof(p.w));
    memcpy(p.b, hb1, sizeof(p.b));
    const int BR = enc_band_rows(H, W), nb = (H + BR - 1) / BR;
    const size_t smem = sizeof(float) * 2 * CI * (BR + 2) * (W + 2);
    k_enc_e1_mean<CI, C1><<<enc_grid(B * nb), kEncThreads, smem, s>>>(x, k, B, H, W, p, m, zpsi, zstride);
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
    const int BR = enc_band_rows(H, W), nb = (H + BR - 1) / BR;
    const size_t smem = sizeof(float) * 2 * C1 * (BR + 2) * (W + 2);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_enc_out<CI, C1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    k_enc_out<CI, C1><<<enc_grid(B * nb), kEncThreads, smem, s>>>(z, zstride, m, B, H, W, p, xp);
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
