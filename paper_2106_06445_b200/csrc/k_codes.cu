// General (n, k) codes: the r = n - k parity combinations and the subset
// decode.  Both are HBM-bound streams over [B][*][d] fp32 features.
//
//  * k_combine_general: comb[b][i][:] = sum_j c_{i,j} h[b][j][:]  (Eq. 3; the
//    systematic generator's parity rows).  fp32 FMA, ascending j.  One thread per float4.
//  * k_decode_general: one CTA per group.  S = the k smallest available tasks; the missing main
//    tasks M (|M| = p) are the unknowns of the p parity rows in S:
//        sum_{j in M} c_{i,j} f_j = P_i - sum_{j avail main} c_{i,j} f_j
//    so f_M = A^-1 (P - C_avail f_avail) with A = c[P_S][M] (p x p).  Thread 0 inverts A in
//    fp64 (Gauss-Jordan, partial pivoting) and folds it into a p x k weight table W over the
//    rows actually read; then the CTA streams out[m][:] = sum_s W[m][s] row_s[:]
//    (Eq. 2 "multiply the inverse of the coefficient matrix").
#include <algorithm>

#include "ci_internal.h"

namespace ci {

namespace {
constexpr int kMaxN = 32;

constexpr double kSingTol = 1e-9;   // SPEC.md:24 singular-subset threshold (scaled determinant)

__global__ void __launch_bounds__(256) k_combine_general(const float* __restrict__ h, const float* __restrict__ coef,
                                                         float* __restrict__ out, int k, int r, int64_t B,
                                                         int64_t d) {
    const bool vec = (d % 4) == 0;
    const int64_t dv = vec ? d / 4 : d;
    const int64_t total = B * r * dv;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = idx % dv, bi = idx / dv;
        const int i = (int)(bi % r);
        const int64_t b = bi / r;
        const float* c = coef + (int64_t)i * k;
        if (vec) {
            const float4* src = reinterpret_cast<const float4*>(h + b * k * d) + e;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int j = 0; j < k; j++) {
                const float cj = __ldg(c + j);
                const float4 v = __ldcs(src + j * dv);
                acc.x = fmaf(cj, v.x, acc.x); acc.y = fmaf(cj, v.y, acc.y);
                acc.z = fmaf(cj, v.z, acc.z); acc.w = fmaf(cj, v.w, acc.w);
            }
            reinterpret_cast<float4*>(out + (b * r + i) * d)[e] = acc;
        } else {
            float acc = 0.f;
            for (int j = 0; j < k; j++) acc = fmaf(__ldg(c + j), h[(b * k + j) * d + e], acc);
            out[(b * r + i) * d + e] = acc;
        }
    }
}

__global__ void __launch_bounds__(256) k_decode_general(float* __restrict__ h, const float* __restrict__ hp,
                                                        const float* __restrict__ coef,
                                                        const uint32_t* __restrict__ avail, int k, int r,
                                                        int64_t B, int64_t d, int* __restrict__ flag) {
    __shared__ int s_p, s_nsrc;
    __shared__ int s_miss[kMaxN];            // missing main task of unknown m
    __shared__ const float* s_src[kMaxN];    // rows read: available mains in S, then parities in S
    __shared__ float s_w[kMaxN][kMaxN];      // W[m][s]
    __shared__ double s_a[kMaxN][2 * kMaxN]; // [A | I] for Gauss-Jordan
    const int n = k + r;
    for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
        if (threadIdx.x == 0) {
            const uint32_t av = __ldg(avail + b) & (n >= 32 ? 0xFFFFFFFFu : ((1u << n) - 1u));
            int S[kMaxN], ns = 0;
            for (int t = 0; t < n && ns < k; t++)
                if ((av >> t) & 1u) S[ns++] = t;
            int p = 0, nsrc = 0;
            if (ns < k) {
                atomicAdd(flag + 1, 1);   // fewer than k results: undecodable (ci_check)
            } else {
                int par[kMaxN], np = 0;
                // missing mains = main tasks not in S (mains have the smallest indices, so every
                // available main is in S)
                int inS[kMaxN] = {0};
                for (int q = 0; q < k; q++) inS[S[q]] = 1;
                for (int j = 0; j < k; j++)
                    if (!inS[j]) s_miss[p++] = j;
                for (int q = 0; q < k; q++) {
                    if (S[q] < k) s_src[nsrc++] = h + (b * k + S[q]) * d;
                    else par[np++] = S[q] - k;
                }
                const int nmain = nsrc;
                for (int a = 0; a < np; a++) s_src[nsrc++] = hp + (b * r + par[a]) * d;
                // A[a][m] = c[par[a]][miss[m]];  Gauss-Jordan on [A | I]
                for (int a = 0; a < p; a++)
                    for (int c2 = 0; c2 < 2 * p; c2++)
                        s_a[a][c2] = c2 < p ? (double)__ldg(coef + par[a] * k + s_miss[c2])
                                            : (c2 - p == a ? 1.0 : 0.0);
                // singular test of SPEC.md:24: |det G_S| with every row of G_S scaled to unit 2-norm.  G_S's main rows are unit vectors, so this
                // is |det A| / prod_a ||c[par[a]]||_2 (full k-length parity rows), det A = the
                // product of the Gauss-Jordan pivots: scale invariant, unlike an absolute pivot floor.
                double sdet = 1.0;
                for (int a = 0; a < p; a++) {
                    double nrm = 0.0;
                    for (int j = 0; j < k; j++) {
                        const double c = (double)__ldg(coef + par[a] * k + j);
                        nrm += c * c;
                    }
                    sdet /= sqrt(nrm);
                }
                bool singular = false;
                for (int col = 0; col < p && !singular; col++) {
                    int piv = col;
                    for (int a = col + 1; a < p; a++)
                        if (fabs(s_a[a][col]) > fabs(s_a[piv][col])) piv = a;
                    sdet *= fabs(s_a[piv][col]);
                    if (s_a[piv][col] == 0.0 || !(sdet > kSingTol)) { singular = true; break; }
                    if (piv != col)
                        for (int c2 = 0; c2 < 2 * p; c2++) {
                            double t = s_a[col][c2]; s_a[col][c2] = s_a[piv][c2]; s_a[piv][c2] = t;
                        }
                    const double inv = 1.0 / s_a[col][col];
                    for (int c2 = 0; c2 < 2 * p; c2++) s_a[col][c2] *= inv;
                    for (int a = 0; a < p; a++) {
                        if (a == col) continue;
                        const double f = s_a[a][col];
                        if (f != 0.0)
                            for (int c2 = 0; c2 < 2 * p; c2++) s_a[a][c2] -= f * s_a[col][c2];
                    }
                }
                if (singular) {
                    atomicAdd(flag + 1, 1);   // singular subset: undecodable (ci_check)
                    p = 0;
                } else {
                    // f_M = Ainv P_S - Ainv C[P_S][avail mains] f_avail
                    for (int m = 0; m < p; m++) {
                        for (int q = 0; q < nmain; q++) {
                            const int j = S[q];
                            double acc = 0.0;
                            for (int a = 0; a < p; a++) acc += s_a[m][p + a] * (double)__ldg(coef + par[a] * k + j);
                            s_w[m][q] = (float)(-acc);
                        }
                        for (int a = 0; a < np; a++) s_w[m][nmain + a] = (float)s_a[m][p + a];
                    }
                }
            }
            s_p = p;
            s_nsrc = nsrc;
        }
        __syncthreads();
        const int p = s_p, nsrc = s_nsrc;
        if (p > 0) {
            for (int64_t e = threadIdx.x; e < d; e += blockDim.x)
                for (int m = 0; m < p; m++) {   // p is usually 1: one pass over the k rows read
                    float acc = 0.f;
                    for (int s = 0; s < nsrc; s++) acc = fmaf(s_w[m][s], s_src[s][e], acc);
                    h[(b * k + s_miss[m]) * d + e] = acc;
                }
        }
        __syncthreads();
    }
}
}  // namespace

cudaError_t launch_combine_general(const float* h, const float* coef, float* out, int k, int r, int64_t B,
                                   int64_t d, cudaStream_t s) {
    const int64_t total = B * r * ((d % 4) == 0 ? d / 4 : d);
    if (total == 0) return cudaSuccess;
    int64_t g = (total + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    k_combine_general<<<(unsigned)g, 256, 0, s>>>(h, coef, out, k, r, B, d);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_decode_general(float* h, const float* hp, const float* coef, const uint32_t* avail, int k, int r,
                                  int64_t B, int64_t d, int* flag, cudaStream_t s) {
    if (B == 0) return cudaSuccess;
    const int g = (int)std::min<int64_t>(B, 148 * 8);
    k_decode_general<<<g, 256, 0, s>>>(h, hp, coef, avail, k, r, B, d, flag);
    count_launch();
    return cudaGetLastError();
}

}  // namespace ci
