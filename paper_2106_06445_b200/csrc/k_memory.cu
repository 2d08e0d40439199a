#include <stdlib.h>
// HBM-bound kernels of the coded path: encode-mean (K7), decode (K8), linear heads +
// argmax (K9) and the device drop-index generator (K12).
//
// Roofline: mean reads k*d*4 B and writes d*4 B per group; decode reads
// (k-1)*d*4 + d*4 + 4 B and writes d*4 B per group.  Both are pure streams: float4
// loads, one thread per (group, 4 features), grid sized to 148 SMs x resident blocks.
#include "ci_internal.h"

namespace ci {

__device__ __forceinline__ float4 ld_stream(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

// m[b][e] = (sum_{i=0}^{k-1} h[b][i][e]) / k ; fp32 sum in ascending i, then one division
// (SURVEY Q7 reading; c_{1,j} = 1/k).
template <int KMAX>
__global__ void __launch_bounds__(256) k_mean(const float4* __restrict__ h, float4* __restrict__ m,
                                              int k, int64_t B, int64_t d4, const float4* __restrict__ eps) {
    const int64_t total = B * d4;
    const float fk = (float)k;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t b = idx / d4, e = idx - b * d4;
        const float4* src = h + b * k * d4 + e;
        float4 v[KMAX > 0 ? KMAX : 1];
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        if (KMAX > 0) {
#pragma unroll
            for (int i = 0; i < KMAX; i++)
                if (i < k) v[i] = ld_stream(src + i * d4);
#pragma unroll
            for (int i = 0; i < KMAX; i++)
                if (i < k) {
                    acc.x = __fadd_rn(acc.x, v[i].x); acc.y = __fadd_rn(acc.y, v[i].y);
                    acc.z = __fadd_rn(acc.z, v[i].z); acc.w = __fadd_rn(acc.w, v[i].w);
                }
        } else {
            for (int i = 0; i < k; i++) {
                float4 t = ld_stream(src + i * d4);
                acc.x = __fadd_rn(acc.x, t.x); acc.y = __fadd_rn(acc.y, t.y);
                acc.z = __fadd_rn(acc.z, t.z); acc.w = __fadd_rn(acc.w, t.w);
            }
        }
        float4 r = make_float4(__fdiv_rn(acc.x, fk), __fdiv_rn(acc.y, fk), __fdiv_rn(acc.z, fk),
                               __fdiv_rn(acc.w, fk));
        if (eps) {   // perturbed encode (f4): mean + eps
            const float4 e4 = ld_stream(eps + idx);
            r.x = __fadd_rn(r.x, e4.x); r.y = __fadd_rn(r.y, e4.y); r.z = __fadd_rn(r.z, e4.z); r.w = __fadd_rn(r.w, e4.w);
        }
        m[idx] = r;
    }
}

static int grid_for(int64_t total, int block) {
    int64_t g = (total + block - 1) / block;
    int64_t cap = 148 * (2048 / block) * 4;  // 4 waves of fully resident blocks
    if (g > cap) g = cap;
    return (int)(g < 1 ? 1 : g);
}

// scalar variants (d % 4 != 0, e.g. the 2-D rotation pin)
__global__ void k_mean_scalar(const float* __restrict__ h, float* __restrict__ m, int k, int64_t B, int64_t d,
                              const float* __restrict__ eps) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < B * d;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t b = idx / d, e = idx - b * d;
        float acc = 0.f;
        for (int i = 0; i < k; i++) acc = __fadd_rn(acc, h[(b * k + i) * d + e]);
        const float r = __fdiv_rn(acc, (float)k);
        m[idx] = eps ? __fadd_rn(r, eps[idx]) : r;
    }
}
__global__ void k_decode_scalar(float* __restrict__ h, const float* __restrict__ p, const int32_t* __restrict__ drop,
                                int k, int64_t B, int64_t d, int* __restrict__ flag) {
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < B * d;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t b = idx / d, e = idx - b * d;
        int j = drop[b];
        if (j == -1) continue;                                    // no loss in this group
        if (j < 0 || j >= k) { if (e == 0) atomicAdd(flag, 1); continue; }
        float acc = 0.f;
        for (int i = 0; i < k; i++)
            if (i != j) acc = __fadd_rn(acc, h[(b * k + i) * d + e]);
        h[(b * k + j) * d + e] = __fmaf_rn((float)k, p[b * d + e], -acc);
    }
}

cudaError_t launch_mean(const float* h, float* m, int k, int64_t B, int64_t d, cudaStream_t s, const float* eps) {
    if (d % 4) {
        if (B * d == 0) return cudaSuccess;
        k_mean_scalar<<<grid_for(B * d, 256), 256, 0, s>>>(h, m, k, B, d, eps);
        count_launch();
        return cudaGetLastError();
    }
    int64_t d4 = d / 4, total = B * d4;
    if (total == 0) return cudaSuccess;
    int g = grid_for(total, 256);
    auto H = reinterpret_cast<const float4*>(h);
    auto M = reinterpret_cast<float4*>(m);
    auto E = reinterpret_cast<const float4*>(eps);
    if (k <= 4) k_mean<4><<<g, 256, 0, s>>>(H, M, k, B, d4, E);
    else if (k <= 10) k_mean<10><<<g, 256, 0, s>>>(H, M, k, B, d4, E);
    else if (k <= 16) k_mean<16><<<g, 256, 0, s>>>(H, M, k, B, d4, E);
    else k_mean<0><<<g, 256, 0, s>>>(H, M, k, B, d4, E);
    count_launch();
    return cudaGetLastError();
}

// h[b][j] = k * p[b] - sum_{i != j, ascending} h[b][i]   for j = drop[b] in [0,k)
// (App. C).  In place; only slot j is written.
template <int KMAX>
__global__ void __launch_bounds__(256) k_decode(float4* __restrict__ h, const float4* __restrict__ p,
                                                const int32_t* __restrict__ drop, int k, int64_t B,
                                                int64_t d4, int* __restrict__ flag) {
    const int64_t total = B * d4, stride = (int64_t)gridDim.x * blockDim.x;
    const float fk = (float)k;
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    // the next iteration's drop index is loaded one iteration ahead: the k-1 row loads depend on
    // it (slot j is skipped), so a just-in-time load would serialise an L2 round trip before
    // every batch of DRAM loads (measured 69% vs 82% DRAM throughput of k_mean under ncu)
    int jn = idx < total ? __ldg(drop + idx / d4) : -1;
    for (; idx < total; idx += stride) {
        int64_t b = idx / d4, e = idx - b * d4;
        const int j = jn;
        if (idx + stride < total) jn = __ldg(drop + (idx + stride) / d4);
        if (j == -1) continue;                                    // no loss in this group
        if (j < 0 || j >= k) {
            if (e == 0) atomicAdd(flag, 1);
            continue;
        }
        float4* g = h + b * k * d4 + e;
        float4 pv = ld_stream(p + b * d4 + e);
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        if (KMAX > 0) {
            float4 v[KMAX > 0 ? KMAX : 1];
#pragma unroll
            for (int i = 0; i < KMAX; i++)
                if (i < k && i != j) v[i] = ld_stream(g + i * d4);
#pragma unroll
            for (int i = 0; i < KMAX; i++)
                if (i < k && i != j) {
                    acc.x = __fadd_rn(acc.x, v[i].x); acc.y = __fadd_rn(acc.y, v[i].y);
                    acc.z = __fadd_rn(acc.z, v[i].z); acc.w = __fadd_rn(acc.w, v[i].w);
                }
        } else {
            for (int i = 0; i < k; i++) {
                if (i == j) continue;
                float4 t = ld_stream(g + i * d4);
                acc.x = __fadd_rn(acc.x, t.x); acc.y = __fadd_rn(acc.y, t.y);
                acc.z = __fadd_rn(acc.z, t.z); acc.w = __fadd_rn(acc.w, t.w);
            }
        }
        g[j * d4] = make_float4(__fmaf_rn(fk, pv.x, -acc.x), __fmaf_rn(fk, pv.y, -acc.y),
                                __fmaf_rn(fk, pv.z, -acc.z), __fmaf_rn(fk, pv.w, -acc.w));
    }
}

cudaError_t launch_decode(float* h, const float* p, const int32_t* drop, int k, int64_t B,
                          int64_t d, int* flag, cudaStream_t s) {
    if (d % 4) {
        if (B * d == 0) return cudaSuccess;
        k_decode_scalar<<<grid_for(B * d, 256), 256, 0, s>>>(h, p, drop, k, B, d, flag);
        count_launch();
        return cudaGetLastError();
    }
    int64_t d4 = d / 4, total = B * d4;
    if (total == 0) return cudaSuccess;
    int g = grid_for(total, 256);
    auto H = reinterpret_cast<float4*>(h);
    auto P = reinterpret_cast<const float4*>(p);
    if (k <= 4) k_decode<4><<<g, 256, 0, s>>>(H, P, drop, k, B, d4, flag);
    else if (k <= 10) k_decode<10><<<g, 256, 0, s>>>(H, P, drop, k, B, d4, flag);
    else if (k <= 16) k_decode<16><<<g, 256, 0, s>>>(H, P, drop, k, B, d4, flag);
    else k_decode<0><<<g, 256, 0, s>>>(H, P, drop, k, B, d4, flag);
    count_launch();
    return cudaGetLastError();
}

// logits[r][c] = sum_e W[c][e] z[r][e] + b[c]; label = first argmax.
// One warp handles ROWS rows; lanes stride the feature axis with float4 loads; W (C x d)
// is read through L1 once per ROWS rows.  Fixed reduction tree -> deterministic.
constexpr int CLS_ROWS = 4;
constexpr int CLS_CMAX = 16;
// Linear heads + first argmax.  A warp owns 4 rows;
// lane l accumulates float4 columns l, l+32, ... in order (fixed order: deterministic), then a
// butterfly reduction.  The head weights are staged per 512-column chunk in shared memory and
// shared by the CTA's 8 warps (32 rows per CTA): 8x less weight traffic than one L1 pass of W
// per warp.
constexpr int CLS_CH4 = 128;   // float4 columns per chunk
__global__ void __launch_bounds__(256) k_classify_smem(const float* __restrict__ z, int64_t n, int64_t d,
                                                       const float* __restrict__ W, const float* __restrict__ bias,
                                                       int C, float* __restrict__ logits,
                                                       int32_t* __restrict__ labels) {
    extern __shared__ float4 wsm[];   // [C][CLS_CH4]
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t d4 = d >> 2;
    const float4* W4 = reinterpret_cast<const float4*>(W);
    for (int64_t rb = (int64_t)blockIdx.x * 32; rb < n; rb += (int64_t)gridDim.x * 32) {
        const int64_t r0 = rb + wid * CLS_ROWS;
        float acc[CLS_ROWS][CLS_CMAX];
#pragma unroll
        for (int r = 0; r < CLS_ROWS; r++)
#pragma unroll
            for (int c = 0; c < CLS_CMAX; c++) acc[r][c] = 0.f;
        for (int64_t c0 = 0; c0 < d4; c0 += CLS_CH4) {
            const int cnt = (int)(d4 - c0 < CLS_CH4 ? d4 - c0 : CLS_CH4);
            __syncthreads();
            for (int i = threadIdx.x; i < C * CLS_CH4; i += blockDim.x) {
                const int c = i / CLS_CH4, e = i - c * CLS_CH4;
                if (e < cnt) wsm[i] = __ldg(W4 + (int64_t)c * d4 + c0 + e);
            }
            __syncthreads();
            for (int e = lane; e < cnt; e += 32) {
                float4 zv[CLS_ROWS];
#pragma unroll
                for (int r = 0; r < CLS_ROWS; r++)
                    zv[r] = (r0 + r < n) ? ld_stream(reinterpret_cast<const float4*>(z + (r0 + r) * d) + c0 + e)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int c = 0; c < CLS_CMAX; c++) {
                    if (c >= C) break;
                    const float4 w = wsm[c * CLS_CH4 + e];
#pragma unroll
                    for (int r = 0; r < CLS_ROWS; r++) {
                        float a = acc[r][c];
                        a = fmaf(w.x, zv[r].x, a);
                        a = fmaf(w.y, zv[r].y, a);
                        a = fmaf(w.z, zv[r].z, a);
                        a = fmaf(w.w, zv[r].w, a);
                        acc[r][c] = a;
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < CLS_ROWS; r++)
#pragma unroll
            for (int c = 0; c < CLS_CMAX; c++) {
                if (c >= C) break;
                float v = acc[r][c];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                acc[r][c] = v;
            }
        if (lane == 0) {
#pragma unroll
            for (int r = 0; r < CLS_ROWS; r++) {
                const int64_t row = r0 + r;
                if (row >= n) break;
                int best = 0;
                float bv = 0.f;
#pragma unroll
                for (int c = 0; c < CLS_CMAX; c++) {
                    if (c >= C) break;
                    const float v = acc[r][c] + __ldg(bias + c);
                    if (logits) logits[row * C + c] = v;
                    if (c == 0 || v > bv) { bv = v; best = c; }
                }
                if (labels) labels[row] = best;
            }
        }
    }
}

// Heads with the whole weight matrix resident in shared memory (C d floats <= kClsResident): one
// persistent CTA of 16 warps per SM, loaded once; each warp streams 4 rows of z (float4, two
// iterations in flight per row) and keeps their C partial dot products in registers, then one
// warp reduction per logit.  No per-chunk barriers, so the z stream is never interrupted.
constexpr int kClsResident = 160 * 1024;
__global__ void __launch_bounds__(512) k_classify_resident(const float* __restrict__ z, int64_t n, int64_t d,
                                                           const float* __restrict__ W, const float* __restrict__ bias,
                                                           int C, float* __restrict__ logits, int32_t* __restrict__ labels) {
    extern __shared__ float4 wres[];   // [C][d/4]
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t d4 = d >> 2;
    const float4* W4 = reinterpret_cast<const float4*>(W);
    {   // W -> shared memory with 8 loads in flight per thread (a serial load / store loop pays the
        // memory latency once per element)
        const int64_t nw = (int64_t)C * d4;
        for (int64_t i0 = threadIdx.x; i0 < nw; i0 += 8 * (int64_t)blockDim.x) {
            float4 t[8];
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int64_t i = i0 + (int64_t)j * blockDim.x;
                if (i < nw) t[j] = __ldg(W4 + i);
            }
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int64_t i = i0 + (int64_t)j * blockDim.x;
                if (i < nw) wres[i] = t[j];
            }
        }
    }
    __syncthreads();
    for (int64_t rb = ((int64_t)blockIdx.x * nw + wid) * CLS_ROWS; rb < n; rb += (int64_t)gridDim.x * nw * CLS_ROWS) {
        float acc[CLS_ROWS][CLS_CMAX];
#pragma unroll
        for (int r = 0; r < CLS_ROWS; r++)
#pragma unroll
            for (int c = 0; c < CLS_CMAX; c++) acc[r][c] = 0.f;
        const float4* zr[CLS_ROWS];
#pragma unroll
        for (int r = 0; r < CLS_ROWS; r++) zr[r] = reinterpret_cast<const float4*>(z + (rb + r < n ? rb + r : rb) * d);
#pragma unroll 4
        for (int64_t e = lane; e < d4; e += 32) {
            float4 zv[CLS_ROWS];
#pragma unroll
            for (int r = 0; r < CLS_ROWS; r++) zv[r] = ld_stream(zr[r] + e);
#pragma unroll
            for (int c = 0; c < CLS_CMAX; c++) {
                if (c >= C) break;
                const float4 w = wres[(int64_t)c * d4 + e];
#pragma unroll
                for (int r = 0; r < CLS_ROWS; r++) {
                    float a = acc[r][c];
                    a = fmaf(w.x, zv[r].x, a);
                    a = fmaf(w.y, zv[r].y, a);
                    a = fmaf(w.z, zv[r].z, a);
                    a = fmaf(w.w, zv[r].w, a);
                    acc[r][c] = a;
                }
            }
        }
#pragma unroll
        for (int r = 0; r < CLS_ROWS; r++)
#pragma unroll
            for (int c = 0; c < CLS_CMAX; c++) {
                if (c >= C) break;
                float v = acc[r][c];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                acc[r][c] = v;
            }
        if (lane == 0) {
#pragma unroll
            for (int r = 0; r < CLS_ROWS; r++) {
                const int64_t row = rb + r;
                if (row >= n) break;
                int best = 0;
                float bv = 0.f;
#pragma unroll
                for (int c = 0; c < CLS_CMAX; c++) {
                    if (c >= C) break;
                    const float v = acc[r][c] + __ldg(bias + c);
                    if (logits) logits[row * C + c] = v;
                    if (c == 0 || v > bv) { bv = v; best = c; }
                }
                if (labels) labels[row] = best;
            }
        }
    }
}

__global__ void k_classify_scalar(const float* __restrict__ z, int64_t n, int64_t d, const float* __restrict__ W,
                                  const float* __restrict__ bias, int C, float* __restrict__ logits,
                                  int32_t* __restrict__ labels) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        int best = 0;
        float bv = 0.f;
        for (int c = 0; c < C; c++) {
            float acc = 0.f;
            for (int64_t e = 0; e < d; e++) acc = fmaf(W[c * d + e], z[r * d + e], acc);
            float v = acc + bias[c];
            if (logits) logits[r * C + c] = v;
            if (c == 0 || v > bv) { bv = v; best = c; }
        }
        if (labels) labels[r] = best;
    }
}

cudaError_t launch_classify(const float* z, int64_t n, int64_t d, const float* W, const float* b,
                            int C, float* logits, int32_t* labels, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (d % 4) {
        k_classify_scalar<<<grid_for(n, 128), 128, 0, s>>>(z, n, d, W, b, C, logits, labels);
        count_launch();
        return cudaGetLastError();
    }
    const size_t wbytes = (size_t)C * d * sizeof(float);
    static const bool no_resident = getenv("CI_NO_CLS_RESIDENT") != nullptr;   // A/B switch
    if (!no_resident && C <= CLS_CMAX && wbytes <= (size_t)kClsResident) {
        static bool attr = false;
        if (!attr) {
            cudaError_t e = cudaFuncSetAttribute(k_classify_resident, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 kClsResident);
            if (e != cudaSuccess) return e;
            attr = true;
        }
        const int64_t need = (n + 16 * CLS_ROWS - 1) / (16 * CLS_ROWS);
        k_classify_resident<<<(unsigned)(need < 148 ? need : 148), 512, wbytes, s>>>(z, n, d, W, b, C, logits, labels);
        count_launch();
        return cudaGetLastError();
    }
    int64_t blocks = (n + 31) / 32;
    if (blocks > 148 * 4) blocks = 148 * 4;
    k_classify_smem<<<(unsigned)blocks, 256, (size_t)C * CLS_CH4 * sizeof(float4), s>>>(z, n, d, W, b, C, logits,
                                                                                     labels);
    count_launch();
    return cudaGetLastError();
}

// drop[b] = (uint32)(splitmix64_at(seed, b) >> 32) % k   (bit-identical to fixtures.make_drops)
__global__ void k_make_drops(int k, int64_t B, uint64_t seed, int32_t* __restrict__ drop) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < B;
         b += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = seed + (uint64_t)(b + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z = z ^ (z >> 31);
        drop[b] = (int32_t)((uint32_t)(z >> 32) % (uint32_t)k);
    }
}

cudaError_t launch_make_drops(int k, int64_t B, uint64_t seed, int32_t* drop, cudaStream_t s) {
    if (B == 0) return cudaSuccess;
    k_make_drops<<<grid_for(B, 256), 256, 0, s>>>(k, B, seed, drop);
    count_launch();
    return cudaGetLastError();
}

// Worker coefficients of the masked-reduction decode / mean (codedinv.h CI_COEF_*)

}  // namespace ci
