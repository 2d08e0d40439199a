// Stage 2 of Arch C (8x8 images, c = 24 coupling channels, m = 128 hidden) as a TS-mode kernel.
// DESIGN.md 7.2c.  Same block as k_stage / k_stage_ts (Eq. 1):
//   s_out <- s_out (+|-) F(s_in),  F = conv3x3(W2) o ReLU o conv3x3(W1).
//
//  * Two images per 128-row M-tile with no pad rows or columns (100% of the MMA rows are
//    pixels; k_stage's padded raster held 3 images in 2 tiles = 75%).  A row shift would cross
//    image and row borders, so conv1's input is kept as nine masked VIEWS, one per tap:
//    V_{u,v}[p] = X[y+u][x+v] (0 outside the image).  conv1 is then a plain K-major GEMM over
//    27 planes of 8 channels (+ the constant-1 plane that carries the folded conv1 bias): 14
//    K = 16 steps, the two K halves of a step two adjacent planes (LBO = one plane).
//  * The hidden (128 channels, ReLU, fp16 hi + lo) is written back into TMEM over acc1 and read
//    by conv2 in TS mode (A from TMEM).  conv2 stacks all 9 taps in N: two passes over the
//    outputs (channels 0-11 then 12-23; N = 108 -> 112 each: column 54 half + 6 tap + o), so a
//    slot needs 128 + 112 TMEM columns.  The epilogue forms out[p] = sum_{u,v} Z_{u,v}[p + 8u + v]:
//    horizontal neighbours are lanes +-1 (image rows are 8-aligned in a warp), vertical ones lanes
//    +-8, except across the two warps of an image (one 32-B exchange per border row).
//  * Two slots (tiles) per CTA, each served by its own group of 8 epilogue warps; per block the
//    MMA thread issues conv1(A) conv1(B) conv2a(A) conv2a(B) conv2b(A) conv2b(B).  The views are
//    ONE shared buffer (112 KB): group A writes its views for block k+1 once conv1(B, k) has
//    completed, group B once conv1(A, k+1) has completed.  Weight segments are streamed per
//    slot (the ring cannot hold a whole 112 KB conv1 segment).
//  * The fp32 state of the slot's two images stays in shared memory for the whole stage.
#include <stdio.h>

#include "ci_internal.h"
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "umma.cuh"

namespace ci {
using namespace umma;

namespace ts2 {
constexpr int kThreads = 576;      // warp 0 producer, warp 1 MMA, warps 2..17 epilogue (2 groups)
constexpr int kEpi = 256;
constexpr int H = 8, W = 8, HW = 64, C = 48, c = 24, M = 128;
constexpr int NP1 = 28;                     // conv1 K planes: 9 taps x 3 + the constant-1 plane
constexpr int PB = 128 * 16;                // plane bytes (one tile, no guards)
constexpr int N1 = 128, N2 = 112;           // conv1 / conv2-pass MMA widths
constexpr int K1 = 14, K2 = 8;              // k-steps
constexpr int NSLOT = 3, SLOTB = 16384;     // weight ring
constexpr int ST_BYTES = 2 * C * HW * 4;    // fp32 state of the slot's two images
constexpr int XCH_BYTES = 2 * 2 * 32 * 32;  // vertical exchange [pass][half][32 border rows][8] fp32
__host__ __device__ constexpr int kstep(int N, int pm) { return N * 32 * (pm == 2 ? 2 : 1); }
__host__ __device__ constexpr int per_slot(int N, int pm) { return SLOTB / kstep(N, pm); }
__host__ __device__ constexpr int view_bytes(int pm) { return (pm ? 2 : 1) * NP1 * PB; }
__host__ __device__ constexpr int smem_bytes(int pm) {
    return NSLOT * SLOTB + view_bytes(pm) + 2 * (ST_BYTES + XCH_BYTES) + 512;
}
}  // namespace ts2

namespace {
__device__ __forceinline__ void t2_ld16(uint32_t taddr, float (&v)[16]) { tmem_ld16(taddr, v); }
__device__ __forceinline__ void t2_ld4(uint32_t taddr, float (&v)[4]) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 4; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void t2_ld2(uint32_t taddr, float (&v)[2]) {
    uint32_t r[2];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(taddr));
    v[0] = __uint_as_float(r[0]);
    v[1] = __uint_as_float(r[1]);
}
__device__ __forceinline__ void t2_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ float2 t2_add2(float2 a, float2 b) {
    float2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&r))
        : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
    return r;
}
__device__ __forceinline__ float2 t2_sub2(float2 a, float2 b) {
    float2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&r))
        : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
    return r;
}
__device__ __forceinline__ float2 t2_fma2(float2 a, float2 b, float2 c) {
    float2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(*reinterpret_cast<unsigned long long*>(&r))
        : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
          "l"(*reinterpret_cast<unsigned long long*>(&c)));
    return r;
}
// two fp32 -> packed 16-bit pair (a in the low half): fp16 hi / lo split, or bf16
__device__ __forceinline__ void t2_split(float a, float b, uint32_t& hi, uint32_t& lo) {
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(b), "f"(a));
    const float2 d = t2_sub2(make_float2(a, b), __half22float2(*reinterpret_cast<const __half2*>(&hi)));
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(d.y), "f"(d.x));
}
__device__ __forceinline__ uint32_t t2_bf16x2(float a, float b) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
    return r;
}
}  // namespace

template <int PM>
__global__ void __launch_bounds__(ts2::kThreads, 1) k_stage_ts2(TsArgs a) {
    using namespace ts2;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint8_t* ring = smem;
    uint8_t* views = ring + NSLOT * SLOTB;                 // [hi: 28 planes][lo: 28 planes]
    uint8_t* gbase = views + view_bytes(PM);               // [2] x { state, xch }
    auto sstate = [&](int s) { return reinterpret_cast<float*>(gbase + (size_t)s * (ST_BYTES + XCH_BYTES)); };
    auto sxch = [&](int s) { return reinterpret_cast<float*>(gbase + (size_t)s * (ST_BYTES + XCH_BYTES) + ST_BYTES); };
    uint64_t* bars = reinterpret_cast<uint64_t*>(gbase + 2 * (ST_BYTES + XCH_BYTES));
    uint64_t* full = bars;            // [3]
    uint64_t* empty = bars + 4;       // [3]
    uint64_t* bqf = bars + 8;         // [4]
    uint64_t* bqe = bars + 12;        // [4]
    uint64_t* x_rdy = bars + 16;      // [2] the shared views hold slot s's input for its next conv1
    uint64_t* a1t = bars + 18;        // [2] conv1 of slot s done (commit; also frees the views)
    uint64_t* hdt = bars + 20;        // [2] hidden of slot s in TMEM
    uint64_t* a2t = bars + 22;        // [2] conv2 pass of slot s done (commit; twice per block)
    uint64_t* a2r = bars + 24;        // [2] pass-a accumulator of slot s read (pass b may overwrite)
    volatile int64_t* bq = reinterpret_cast<volatile int64_t*>(bars + 26);   // [4]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 30);

    {   // views: zero (masked taps, never written later); constant-1 plane: channel 0 = 1.0 (hi)
        uint4 z = make_uint4(0, 0, 0, 0);
        for (int i = tid; i < view_bytes(PM) / 16; i += kThreads) reinterpret_cast<uint4*>(views)[i] = z;
        __syncthreads();
        const uint32_t one = PM ? 0x3C00u : 0x3F80u;   // fp16 / bf16 1.0 in the low half
        for (int r = tid; r < 128; r += kThreads)
            *reinterpret_cast<uint4*>(views + (size_t)27 * PB + r * 16) = make_uint4(one, 0, 0, 0);
    }
    fence_proxy_async();
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    if (tid == 0) {
        for (int i = 0; i < NSLOT; i++) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        for (int i = 0; i < 4; i++) { mbar_init(&bqf[i], 1); mbar_init(&bqe[i], 1 + kEpi); }
        for (int i = 0; i < 2; i++) {
            mbar_init(&x_rdy[i], kEpi); mbar_init(&a1t[i], 1); mbar_init(&hdt[i], kEpi);
            mbar_init(&a2t[i], 1); mbar_init(&a2r[i], kEpi);
        }
        fence_mbar_init();
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    const int64_t nbatch = (a.n + 1) / 2;   // two images per slot batch
    auto bq_read = [&](int i) -> int64_t {
        mbar_wait(&bqf[i & 3], (uint32_t)((i >> 2) & 1));
        return bq[i & 3];
    };
    const int SEG1 = K1 * kstep(N1, PM), SEG2 = K2 * kstep(N2, PM);
    constexpr int G1 = per_slot(N1, PM), G2 = per_slot(N2, PM);   // k-steps per ring slot

    if (warp == 0) {
        // ================= producer ==========================================================
        if (lane == 0) {
            int slot = 0;
            uint32_t phase = 0;
            int64_t claimed = 0;
            auto next = [&]() -> int64_t {
                const int64_t k = claimed++;
                if (k == 0) return blockIdx.x;
                return a.ctr ? (int64_t)gridDim.x + atomicAdd(a.ctr, 1) : (int64_t)blockIdx.x + k * gridDim.x;
            };
            auto publish = [&](int i, int64_t v) {
                mbar_wait(&bqe[i & 3], (uint32_t)(((i >> 2) & 1) ^ 1));
                bq[i & 3] = v;
                mbar_arrive(&bqf[i & 3]);
            };
            auto stream = [&](const uint8_t* src, int K, int G, int kb) {
                for (int s0 = 0; s0 < K; s0 += G) {
                    const uint32_t bytes = (uint32_t)(min(G, K - s0) * kb);
                    mbar_wait(&empty[slot], phase ^ 1);
                    mbar_arrive_expect_tx(&full[slot], bytes);
                    bulk_g2s(ring + (size_t)slot * SLOTB, src + (size_t)s0 * kb, bytes, &full[slot]);
                    if (++slot == NSLOT) { slot = 0; phase ^= 1; }
                }
            };
            for (int pi = 0;; pi++) {
                const int64_t b0 = next();
                const int64_t b1 = b0 < nbatch ? next() : nbatch;
                publish(2 * pi, b0);
                publish(2 * pi + 1, b1);
                if (b0 >= nbatch) break;
                const int ns = b1 < nbatch ? 2 : 1;
                for (int tt = 0; tt < a.nb; tt++) {
                    const int t = a.inverse ? a.nb - 1 - tt : tt;
                    const uint8_t* src = a.wpack + (int64_t)t * a.blk_bytes;
                    for (int s = 0; s < ns; s++) stream(src, K1, G1, kstep(N1, PM));
                    for (int pass = 0; pass < 2; pass++)
                        for (int s = 0; s < ns; s++) stream(src + SEG1 + pass * SEG2, K2, G2, kstep(N2, PM));
                }
                if (b1 >= nbatch) {
                    publish(2 * pi + 2, nbatch);
                    break;
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ================= MMA issuer ========================================================
        if (elect_one()) {
            int slot = 0;
            uint32_t phase = 0, kb = 0;
            const uint32_t rb = smem_u32(ring), vb = smem_u32(views);
            const uint32_t id1 = idesc_of(128, N1, PM != 0);
            const uint32_t id2 = idesc_of(128, N2, PM != 0);
            constexpr uint32_t LOA = (uint32_t)(NP1 * PB / 16);   // lo planes, descriptor units
            auto acquire = [&]() -> uint32_t {
                mbar_wait(&full[slot], phase);
                fence_after();
                return rb + (uint32_t)slot * SLOTB;
            };
            auto release = [&]() {
                commit(&empty[slot]);
                if (++slot == NSLOT) { slot = 0; phase ^= 1; }
            };
            for (int pi = 0;; pi++) {
                const int64_t b0 = bq_read(2 * pi);
                mbar_arrive(&bqe[(2 * pi) & 3]);
                if (b0 >= nbatch) break;
                const int64_t b1 = bq_read(2 * pi + 1);
                mbar_arrive(&bqe[(2 * pi + 1) & 3]);
                const int ns = b1 < nbatch ? 2 : 1;
                for (int tt = 0; tt < a.nb; tt++, kb++) {
                    const uint32_t par = kb & 1;
                    // conv1 (SS: A = the nine views, one K-major operand of 28 planes)
                    for (int s = 0; s < 2; s++) {
                        if (s >= ns) { commit(&a1t[s]); continue; }   // keeps the views hand-off regular
                        mbar_wait(&x_rdy[s], par);
                        fence_after();
                        const uint32_t d = tmem + (uint32_t)(s * 256);
                        for (int s0 = 0; s0 < K1; s0 += G1) {
                            const uint32_t w = acquire();
#pragma unroll
                            for (int q = 0; q < G1; q++) {
                                const int ks = s0 + q;
                                if (ks >= K1) break;
                                const uint64_t ad = smem_desc(vb + (uint32_t)(2 * ks * PB), PB, 128);
                                const uint64_t bd = smem_desc(w + (uint32_t)(q * kstep(N1, PM)), N1 * 16, 128);
                                const uint32_t acc = ks > 0 ? 1u : 0u;
                                mma_bf16(d, ad, bd, id1, acc);
                                if (PM >= 1) mma_bf16(d, ad + LOA, bd, id1, 1u);
                                if (PM == 2) mma_bf16(d, ad, bd + (uint64_t)(N1 * 32 / 16), id1, 1u);
                            }
                            release();
                        }
                        commit(&a1t[s]);
                    }
                    // conv2, two passes over the outputs (TS: A = the hidden in TMEM)
                    for (int pass = 0; pass < 2; pass++)
                        for (int s = 0; s < ns; s++) {
                            if (pass == 0) mbar_wait(&hdt[s], par);
                            else mbar_wait(&a2r[s], par);
                            fence_after();
                            const uint32_t tb = tmem + (uint32_t)(s * 256);
                            for (int s0 = 0; s0 < K2; s0 += G2) {
                                const uint32_t w = acquire();
#pragma unroll
                                for (int q = 0; q < G2; q++) {
                                    const int ks = s0 + q;
                                    if (ks >= K2) break;
                                    const uint32_t ahi = tb + (uint32_t)(16 * ks);   // hidden 16 ks..+15: hi | lo
                                    const uint64_t bd = smem_desc(w + (uint32_t)(q * kstep(N2, PM)), N2 * 16, 128);
                                    const uint32_t acc = ks > 0 ? 1u : 0u;
                                    mma_ts(tb + 128, ahi, bd, id2, acc);
                                    if (PM >= 1) mma_ts(tb + 128, ahi + 8, bd, id2, 1u);
                                    if (PM == 2) mma_ts(tb + 128, ahi, bd + (uint64_t)(N2 * 32 / 16), id2, 1u);
                                }
                                release();
                            }
                            commit(&a2t[s]);
                        }
                }
                if (ns == 1) break;
            }
        }
        __syncwarp();
    } else {
        // ================= epilogue: group g = slot g (8 warps) ================================
        // row p = 32 quarter + lane of the tile: image p / 64, y = (p % 64) / 8, x = p % 8.  Warps w
        // and w+4 share a lane quarter: conv1 epilogue half h = hidden 64h..64h+63; conv2 epilogue
        // half h = outputs 12 pass + 6h..+5; view writes half 0 = taps 0-4, half 1 = taps 5-8.
        const int g = (warp - 2) >> 3, ew = (warp - 2) & 7, quarter = warp & 3, half = ew >> 2, et = ew * 32 + lane;
        const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
        const int p = quarter * 32 + lane, img = p >> 6, pp = p & 63, y = pp >> 3, x = pp & 7;
        const uint32_t bar_id = 1 + g;
        auto gsync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(kEpi) : "memory"); };
        float* st = sstate(g);
        float* xch0 = sxch(g);
        const float2 ml = make_float2(x > 0 ? 1.f : 0.f, x > 0 ? 1.f : 0.f);
        const float2 mr = make_float2(x < W - 1 ? 1.f : 0.f, x < W - 1 ? 1.f : 0.f);
        // cross-warp vertical neighbours: the second warp of an image (odd quarter) lanes 0-7 need
        // H_-1 of the first warp's lanes 24-31 and vice versa (H_+1)
        const bool xtop = (quarter & 1) && lane < 8, xbot = !(quarter & 1) && lane >= 24;
        auto in_half = [&](int t) { return ((a.first_orient + t) & 1) == 0 ? 0 : c; };
        // views <- this pixel's 24 channels at offset ch0 of the state (the next conv1's input)
        auto write_views = [&](int ch0, int nimg) {
            const bool present = img < nimg;
            float v[c];
#pragma unroll
            for (int o = 0; o < c; o++) v[o] = present ? st[(img * C + ch0 + o) * HW + pp] : 0.f;
            uint32_t hi[12], lo[12];
#pragma unroll
            for (int e = 0; e < 12; e++) {
                if (PM) t2_split(v[2 * e], v[2 * e + 1], hi[e], lo[e]);
                else { hi[e] = t2_bf16x2(v[2 * e], v[2 * e + 1]); lo[e] = 0; }
            }
#pragma unroll
            for (int tap = 0; tap < 9; tap++) {
                if ((tap < 5) != (half == 0)) continue;
                const int u = tap / 3 - 1, vv = tap % 3 - 1;
                // V_{u,v}[q] = X[q + 8u + v]: this pixel feeds row q = p - 8u - v when that pixel exists
                if (y - u < 0 || y - u > H - 1 || x - vv < 0 || x - vv > W - 1) continue;
                const int q = p - 8 * u - vv;
#pragma unroll
                for (int pl = 0; pl < 3; pl++) {
                    const size_t off = (size_t)(tap * 3 + pl) * PB + (size_t)q * 16;
                    *reinterpret_cast<uint4*>(views + off) = make_uint4(hi[4 * pl], hi[4 * pl + 1], hi[4 * pl + 2], hi[4 * pl + 3]);
                    if (PM)
                        *reinterpret_cast<uint4*>(views + (size_t)NP1 * PB + off) =
                            make_uint4(lo[4 * pl], lo[4 * pl + 1], lo[4 * pl + 2], lo[4 * pl + 3]);
                }
            }
        };
        uint32_t kb = 0;
        for (int i = 0;; i++) {
            const int qe = 2 * i + g;
            const int64_t b = bq_read(qe);
            mbar_arrive(&bqe[qe & 3]);
            if (b >= nbatch) break;
            const int64_t img0 = 2 * b;
            const int nimg = a.n - img0 < 2 ? 1 : 2;
            float* gst = a.state + img0 * (int64_t)C * HW;
            {   // the slot's state -> shared memory
                const float4* src = reinterpret_cast<const float4*>(gst);
                float4* dst = reinterpret_cast<float4*>(st);
                for (int q = et; q < nimg * C * HW / 4; q += kEpi) dst[q] = __ldcg(src + q);
            }
            gsync();
            // first block's views: A after conv1(B) of the previous block, B after conv1(A) of this one
            if (g == 0) { if (kb > 0) mbar_wait(&a1t[1], (kb - 1) & 1); }
            else mbar_wait(&a1t[0], kb & 1);
            write_views(in_half(a.inverse ? a.nb - 1 : 0), nimg);
            fence_proxy_async();
            mbar_arrive(&x_rdy[g]);
            for (int tt = 0; tt < a.nb; tt++, kb++) {
                const uint32_t par = kb & 1;
                const int t = a.inverse ? a.nb - 1 - tt : tt;
                const int out_off = c - in_half(t);
                const bool write_next = tt + 1 < a.nb;
                const float* b2 = a.bias + (int64_t)t * a.bias_stride + M;
                // ---- conv1 epilogue: acc1 -> ReLU -> fp16 hi | lo words over the columns just read
                mbar_wait(&a1t[g], par);
                fence_after();
#pragma unroll
                for (int rd = 0; rd < 4; rd++) {
                    const uint32_t col = tmem + lane_addr + (uint32_t)(g * 256 + 64 * half + 16 * rd);
                    float v[16];
                    t2_ld16(col, v);
                    tmem_wait_ld();
                    uint32_t hw[8], lw[8];
#pragma unroll
                    for (int e = 0; e < 8; e++) {
                        const float p0 = fmaxf(v[2 * e], 0.f), p1 = fmaxf(v[2 * e + 1], 0.f);
                        if (PM) t2_split(p0, p1, hw[e], lw[e]);
                        else hw[e] = t2_bf16x2(p0, p1);
                    }
                    t2_st8(col, hw);
                    if (PM) t2_st8(col + 8, lw);
                }
                tmem_wait_st();
                fence_before();
                mbar_arrive(&hdt[g]);
                // ---- conv2 epilogue, two passes: col2im of the 9 tap groups, s_out (+|-)= F + b2
#pragma unroll 1
                for (int pass = 0; pass < 2; pass++) {
                    const int ch0 = 12 * pass + 6 * half;   // this thread's 6 outputs
                    float2 bb[3];
#pragma unroll
                    for (int o = 0; o < 3; o++) bb[o] = make_float2(__ldg(b2 + ch0 + 2 * o), __ldg(b2 + ch0 + 2 * o + 1));
                    mbar_wait(&a2t[g], (uint32_t)pass);
                    fence_after();
                    float2 z[9][3];   // column 54 half + 6 tap + o
                    {
                        const uint32_t col = tmem + lane_addr + (uint32_t)(g * 256 + 128 + 54 * half);
                        float za[16], zb[16], zc[16], zd[4], ze[2];
                        t2_ld16(col, za);
                        t2_ld16(col + 16, zb);
                        t2_ld16(col + 32, zc);
                        t2_ld4(col + 48, zd);
                        t2_ld2(col + 52, ze);
                        tmem_wait_ld();
                        auto zq = [&](int q) -> float {
                            return q < 16 ? za[q] : q < 32 ? zb[q - 16] : q < 48 ? zc[q - 32] : q < 52 ? zd[q - 48] : ze[q - 52];
                        };
#pragma unroll
                        for (int q = 0; q < 27; q++) z[q / 3][q % 3] = make_float2(zq(2 * q), zq(2 * q + 1));
                    }
                    fence_before();
                    if (pass == 0) mbar_arrive(&a2r[g]);   // pass b may overwrite the accumulator
                    // horizontal: H_u[r] = Z_{u,-1}[r-1] + Z_{u,0}[r] + Z_{u,+1}[r+1] (masked at x = 0 / W-1)
                    float2 hs[3][3];
#pragma unroll
                    for (int u = 0; u < 3; u++)
#pragma unroll
                        for (int o = 0; o < 3; o++) {
                            const float2 zl = z[u * 3 + 0][o], zr = z[u * 3 + 2][o];
                            const float2 l = make_float2(__shfl_up_sync(0xffffffffu, zl.x, 1), __shfl_up_sync(0xffffffffu, zl.y, 1));
                            const float2 r = make_float2(__shfl_down_sync(0xffffffffu, zr.x, 1), __shfl_down_sync(0xffffffffu, zr.y, 1));
                            hs[u][o] = t2_fma2(l, ml, t2_fma2(r, mr, z[u * 3 + 1][o]));
                        }
                    // vertical: out[p] = H_-1[p-8] + H_0[p] + H_+1[p+8]; rows +-8 are lanes +-8 except
                    // across the two warps of an image (exchange); image borders = warp borders
                    float* xch = xch0 + (pass * 2 + half) * (32 * 8);   // 32 border rows per tile
                    float2 mid[3];
#pragma unroll
                    for (int o = 0; o < 3; o++) {
                        const float2 up = make_float2(__shfl_up_sync(0xffffffffu, hs[0][o].x, 8), __shfl_up_sync(0xffffffffu, hs[0][o].y, 8));
                        const float2 dn = make_float2(__shfl_down_sync(0xffffffffu, hs[2][o].x, 8), __shfl_down_sync(0xffffffffu, hs[2][o].y, 8));
                        const float2 mu = make_float2(lane >= 8 ? 1.f : 0.f, lane >= 8 ? 1.f : 0.f);
                        const float2 md = make_float2(lane < 24 ? 1.f : 0.f, lane < 24 ? 1.f : 0.f);
                        mid[o] = t2_add2(t2_fma2(up, mu, t2_fma2(dn, md, hs[1][o])), bb[o]);
                    }
                    if (xbot || xtop) {   // publish H_-1 (first warp, lanes 24-31) / H_+1 (second warp, lanes 0-7)
                        const int u = xbot ? 0 : 2;
                        const int e = img * 16 + (xbot ? lane - 24 : 8 + lane);
                        reinterpret_cast<float4*>(xch)[2 * e] = make_float4(hs[u][0].x, hs[u][0].y, hs[u][1].x, hs[u][1].y);
                        reinterpret_cast<float2*>(xch)[4 * e + 2] = hs[u][2];
                    }
                    gsync();
                    if (xbot || xtop) {   // the row 8 above (xtop) / below (xbot), published by the other warp
                        const int q = img * 16 + (xtop ? lane : 8 + lane - 24);
                        const float4 o0 = reinterpret_cast<const float4*>(xch)[2 * q];
                        const float2 o1 = reinterpret_cast<const float2*>(xch)[4 * q + 2];
                        mid[0] = t2_add2(mid[0], make_float2(o0.x, o0.y));
                        mid[1] = t2_add2(mid[1], make_float2(o0.z, o0.w));
                        mid[2] = t2_add2(mid[2], o1);
                    }
#pragma unroll
                    for (int o = 0; o < 3; o++) {
                        float* sp = st + (img * C + out_off + ch0 + 2 * o) * HW + pp;
                        const float2 old = make_float2(sp[0], sp[HW]);
                        const float2 nv = a.inverse ? t2_sub2(old, mid[o]) : t2_add2(old, mid[o]);
                        sp[0] = nv.x;
                        sp[HW] = nv.y;
                    }
                }
                if (write_next) {
                    gsync();   // the pixel's 24 updated channels come from both halves and both passes
                    // the shared views are free once the other slot's conv1 has completed
                    if (g == 0) mbar_wait(&a1t[1], par);
                    else mbar_wait(&a1t[0], (kb + 1) & 1);
                    write_views(out_off, nimg);
                    fence_proxy_async();
                    mbar_arrive(&x_rdy[g]);
                }
            }
            // ---- state back to global memory
            gsync();
            {
                float4* dst = reinterpret_cast<float4*>(gst);
                const float4* src = reinterpret_cast<const float4*>(st);
                for (int q = et; q < nimg * C * HW / 4; q += kEpi) __stcg(dst + q, src[q]);
            }
            gsync();
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

bool stage_ts2_shape(int H, int W, int C, int c, int m, int residual, int act) {
    return H == ts2::H && W == ts2::W && C == ts2::C && c == ts2::c && m == ts2::M && !residual && act == 0 &&
           !getenv("CI_NO_TS2");
}
int64_t stage_ts2_block_bytes(int pm) {
    return (int64_t)ts2::K1 * ts2::kstep(ts2::N1, pm) + 2 * (int64_t)ts2::K2 * ts2::kstep(ts2::N2, pm);
}

typedef void (*Ts2Kernel)(TsArgs);
static Ts2Kernel ts2_kernel(int pm) { return pm == 2 ? k_stage_ts2<2> : (pm == 1 ? k_stage_ts2<1> : k_stage_ts2<0>); }

cudaError_t stage_ts2_prepare() {
    cudaError_t e = cudaSuccess;
    for (int pm = 0; pm < 3 && e == cudaSuccess; pm++)
        e = cudaFuncSetAttribute(ts2_kernel(pm), cudaFuncAttributeMaxDynamicSharedMemorySize, ts2::smem_bytes(pm));
    return e;
}

cudaError_t launch_stage_ts2(const TsArgs& a, int pm, cudaStream_t st) {
    if (a.n <= 0) return cudaSuccess;
    const int64_t nbatch = (a.n + 1) / 2;
    const int grid = (int)std::min<int64_t>((nbatch + 1) / 2, 148);
    ts2_kernel(pm)<<<grid, ts2::kThreads, ts2::smem_bytes(pm), st>>>(a);
    return cudaGetLastError();
}

}  // namespace ci
