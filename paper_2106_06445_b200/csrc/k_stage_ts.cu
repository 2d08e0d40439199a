// Stage 1 of Arch C (16x16 images, c = 6 coupling channels, m = 64 hidden) as a TS-mode kernel:
// the hidden activation never leaves tensor memory.  DESIGN.md 7.2b.
//
// One additive-coupling block (i-RevNet style; reading Q1 of DESIGN.md 2):
//   s_out <- s_out (+|-) F(s_in),
//   F = conv3x3(W2) o ReLU o conv3x3(W1)   (cross-correlation, zero padding).
//
//  * Raster WITHOUT pad column or pad band: one image = 256 rows = exactly two 128-row M-tiles
//    (100% of the MMA rows are pixels; the padded raster of k_stage holds 2 images in 5 tiles).
//    Horizontal taps can no longer be row shifts (they would wrap into the next image row), so
//    the conv1 input is kept in three views: Xc (the input), Xl[p] = X[p-1] (0 at x = 0) and
//    Xr[p] = X[p+1] (0 at x = W-1).  Tap (u, v) of row p is row p + u W of view v: vertical
//    shifts only, and the pair-mode k-step order of k_stage is kept (9 taps x 8 channels in 5
//    K = 16 steps, the two 8-channel K halves of a step LBO bytes apart: l|c views, or two
//    rows of Xr 16 rows apart).
//  * conv1 (SS mode, A = X views in shared memory, B = W1 streamed by the TMA engine) writes
//    acc1[row][h]; the epilogue applies ReLU, splits into fp16 hi + lo and stores the result
//    back into TMEM (tcgen05.st) as the A operand of conv2: lane = pixel row, two 16-bit
//    channels per 32-bit column (tests/test_gpu_umma.py pins the layout).
//  * conv2 (TS mode: A from TMEM, only B crosses the 128 B/clk shared-memory port; measured at
//    the compute floor N/2 cycles) computes all 9 taps at once: N = 64 columns = 9 taps x 6
//    outputs (column 6 tap + o) + padding, K = the 64 hidden channels.  The epilogue forms
//    out[p] = sum_{u,v} Z_{u,v}[p + u W + v]: the horizontal part with lane shuffles (image rows
//    are 16-aligned inside a warp), the vertical part with one xor-16 shuffle (two image rows per
//    warp) plus one 32-B shared-memory exchange with the neighbouring warp row.
//  * Two images ("slots") per CTA in flight: TMEM columns [0,256) and [256,512), each served by
//    its own group of 8 epilogue warps.  The MMA issue order per block, conv1(A) conv1(B)
//    conv2(A) conv2(B), lets the tensor core run one image's convolutions while the other
//    image's group is in its epilogue; the groups are otherwise independent (own barriers,
//    own batch-queue entries, own state load / store).
//  * The image's fp32 state lives in shared memory for the whole stage; the group prefetches its
//    next image with cp.async into a second buffer.  Images are read / written in the layout the
//    caller names (stage_io.cuh), so the squeeze psi / psi^-1 at the stage boundaries costs no pass.
// Precisions as k_stage (PM: 0 bf16, 1 f16x2, 2 f16x3 with the stacked conv1).
#include <stdio.h>

#include "ci_internal.h"
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "stage_io.cuh"
#include "umma.cuh"

namespace ci {
using namespace umma;

namespace ts {
constexpr int kThreads = 576;      // warp 0 producer, warp 1 MMA, warps 2..17 epilogue (2 groups)
constexpr int kEpi = 256;          // threads of one epilogue group (one image slot)
constexpr int H = 16, W = 16, HW = 256, C = 12, c = 6, M = 64;
constexpr int G = 16;                       // guard rows above the image (one image row)
constexpr int RT = G + HW + 32;             // rows per view plane (32 guard rows below)
constexpr int PB = RT * 16;                 // plane bytes
constexpr int N1 = 64, N2 = 64;             // conv1 / conv2 MMA widths
constexpr int K1 = 5, K2 = 4;               // k-steps
constexpr int NSLOT = 4, SLOTB = 20480;     // weight ring
constexpr int ST_BYTES = C * HW * 4;        // fp32 state of one image (two buffers per slot: cp.async prefetch)
constexpr int XCH_BYTES = 2 * HW * 32;      // vertical exchange [block parity][row][8] fp32
__host__ __device__ constexpr int kstep(int N, int pm) { return N * 32 * (pm == 2 ? 2 : 1); }
__host__ __device__ constexpr int nplanes(int pm) { return pm ? 6 : 3; }
__host__ __device__ constexpr int slot_bytes(int pm) { return nplanes(pm) * PB + 2 * ST_BYTES + XCH_BYTES; }
__host__ __device__ constexpr int smem_bytes(int pm) { return NSLOT * SLOTB + 2 * slot_bytes(pm) + 512; }
}  // namespace ts

__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float (&v)[4]) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 4; i++) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, float (&v)[2]) {
    uint32_t r[2];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(taddr));
    v[0] = __uint_as_float(r[0]);
    v[1] = __uint_as_float(r[1]);
}
__device__ __forceinline__ void tmem_st16u(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

// f32x2 arithmetic (sm_100 FADD2 / FFMA2): two lanes of a float2 per instruction
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    float2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&r))
        : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
    return r;
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    float2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&r))
        : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
    return r;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    float2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(*reinterpret_cast<unsigned long long*>(&r))
        : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
          "l"(*reinterpret_cast<unsigned long long*>(&c)));
    return r;
}

__device__ __forceinline__ void tmem_st8u(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
// two fp32 -> packed 16-bit pair (a in the low half): fp16 hi / lo split, or bf16
__device__ __forceinline__ void ts_split(float a, float b, uint32_t& hi, uint32_t& lo) {
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(b), "f"(a));
    const float2 d = sub2(make_float2(a, b), __half22float2(*reinterpret_cast<const __half2*>(&hi)));
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(d.y), "f"(d.x));
}
__device__ __forceinline__ uint32_t ts_bf16x2(float a, float b) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
    return r;
}

// PM: precision; STK (PM == 2 only): stacked conv1, hi(x) [W_hi | W_lo] as one 2N-wide MMA
#define TS_WAIT(acc, call)                                             \
    do {                                                               \
        const long long t0_ = a.dbg ? clock64() : 0;                   \
        call;                                                          \
        if (a.dbg) acc += (unsigned long long)(clock64() - t0_);       \
    } while (0)

template <int PM, int STK>
__global__ void __launch_bounds__(ts::kThreads, 1) k_stage_ts(TsArgs a) {
    using namespace ts;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint8_t* ring = smem;
    uint8_t* slots = ring + NSLOT * SLOTB;   // [2] x { X planes [hi l c r][lo l c r], state, xch }
    auto xplanes = [&](int s) { return slots + (size_t)s * slot_bytes(PM); };
    auto sstate = [&](int s) { return reinterpret_cast<float*>(slots + (size_t)s * slot_bytes(PM) + nplanes(PM) * PB); };
    auto sxch = [&](int s) {
        return reinterpret_cast<float4*>(slots + (size_t)s * slot_bytes(PM) + nplanes(PM) * PB + 2 * ST_BYTES);
    };
    uint64_t* bars = reinterpret_cast<uint64_t*>(slots + 2 * slot_bytes(PM));
    uint64_t* full = bars;            // [4]
    uint64_t* empty = bars + 4;       // [4]
    uint64_t* bqf = bars + 8;         // [4] batch queue entry published
    uint64_t* bqe = bars + 12;        // [4] entry consumed (MMA thread + every epilogue thread)
    uint64_t* x_rdy = bars + 16;      // [2] X views of slot s final for the next conv1 (epilogue)
    uint64_t* a1t = bars + 18;        // [2][2] conv1 of (slot, tile) done (commit)
    uint64_t* hdt = bars + 22;        // [2][2] hidden of (slot, tile) in TMEM (epilogue)
    uint64_t* a2t = bars + 26;        // [2][2] conv2 of (slot, tile) done (commit)
    volatile int64_t* bq = reinterpret_cast<volatile int64_t*>(bars + 30);   // [4]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 34);

    {   // X views: zero guards, x = 0 column of Xl, x = W-1 column of Xr (never written later)
        uint4 z = make_uint4(0, 0, 0, 0);
        for (int s = 0; s < 2; s++)
            for (int i = tid; i < nplanes(PM) * PB / 16; i += kThreads) reinterpret_cast<uint4*>(xplanes(s))[i] = z;
    }
    fence_proxy_async();
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    if (tid == 0) {
        for (int i = 0; i < 4; i++) {
            mbar_init(&full[i], 1); mbar_init(&empty[i], 1);
            mbar_init(&bqf[i], 1); mbar_init(&bqe[i], 1 + kEpi);
        }
        for (int i = 0; i < 2; i++) mbar_init(&x_rdy[i], kEpi);   // one epilogue group each
        for (int i = 0; i < 4; i++) { mbar_init(&a1t[i], 1); mbar_init(&hdt[i], kEpi); mbar_init(&a2t[i], 1); }
        fence_mbar_init();
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    const int64_t nbatch = a.n;   // one image per batch
    auto bq_read = [&](int i) -> int64_t {
        mbar_wait(&bqf[i & 3], (uint32_t)((i >> 2) & 1));
        return bq[i & 3];
    };
    const int SEG1 = K1 * kstep(N1, PM), SEG2 = K2 * kstep(N2, PM);

    if (warp == 0) {
        // ================= producer: claims batches in pairs, streams packed weights =========
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
            for (int pi = 0;; pi++) {
                const int64_t b0 = next();
                const int64_t b1 = b0 < nbatch ? next() : nbatch;
                publish(2 * pi, b0);
                publish(2 * pi + 1, b1);   // group B reads its entry even when the queue is done
                if (b0 >= nbatch) break;
                for (int tt = 0; tt < a.nb; tt++) {
                    const int t = a.inverse ? a.nb - 1 - tt : tt;
                    const uint8_t* src = a.wpack + (int64_t)t * a.blk_bytes;
                    for (int sg = 0; sg < 2; sg++) {
                        const uint32_t bytes = sg == 0 ? SEG1 : SEG2;
                        mbar_wait(&empty[slot], phase ^ 1);
                        mbar_arrive_expect_tx(&full[slot], bytes);
                        bulk_g2s(ring + (size_t)slot * SLOTB, src, bytes, &full[slot]);
                        src += bytes;
                        if (++slot == NSLOT) { slot = 0; phase ^= 1; }
                    }
                }
                if (b1 >= nbatch) {   // group A's next entry: terminator
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
            unsigned long long c_x = 0, c_h = 0, c_f = 0;   // CI_DEBUG_CYCLES: MMA-thread waits
            const long long c_t0 = clock64();
            const uint32_t rb = smem_u32(ring);
            const uint32_t id1w = idesc_of(128, STK ? 2 * N1 : N1, PM != 0);
            const uint32_t id1 = idesc_of(128, N1, PM != 0);
            const uint32_t id2 = idesc_of(128, N2, PM != 0);
            constexpr uint32_t LOA = (uint32_t)(3 * PB / 16);     // lo views, descriptor units
            constexpr uint32_t B1LBO = (uint32_t)((STK ? 2 : 1) * N1 * 16);
            for (int pi = 0;; pi++) {
                const int64_t b0 = bq_read(2 * pi);
                mbar_arrive(&bqe[(2 * pi) & 3]);
                if (b0 >= nbatch) break;
                const int64_t b1 = bq_read(2 * pi + 1);
                mbar_arrive(&bqe[(2 * pi + 1) & 3]);
                const int ns = b1 < nbatch ? 2 : 1;
                for (int tt = 0; tt < a.nb; tt++, kb++) {
                    const uint32_t par = kb & 1;
                    // conv1 of both slots: one weight segment
                    TS_WAIT(c_f, mbar_wait(&full[slot], phase));
                    fence_after();
                    const uint32_t w1 = rb + (uint32_t)slot * SLOTB;
                    for (int s = 0; s < ns; s++) {
                        TS_WAIT(c_x, mbar_wait(&x_rdy[s], par));
                        fence_after();
                        const uint32_t xs = smem_u32(xplanes(s));
#pragma unroll
                        for (int t = 0; t < 2; t++) {
                            const uint32_t d = tmem + (uint32_t)(s * 256 + t * 128);
#pragma unroll
                            for (int ks = 0; ks < K1; ks++) {
                                // k-step ks (pair order): views l|c at row shift (ks-1) W, or two rows
                                // of Xr 16 apart (taps (-1,+1)|(0,+1), then (+1,+1)|zero weights)
                                const uint32_t base = ks < 3 ? xs : xs + 2 * PB;
                                const int row = G + t * 128 + (ks < 3 ? (ks - 1) * W : (ks == 3 ? -W : W));
                                const uint32_t lbo = ks < 3 ? (uint32_t)PB : (uint32_t)(W * 16);
                                const uint64_t ad = smem_desc(base + (uint32_t)row * 16u, lbo, 128);
                                const uint64_t bd = smem_desc(w1 + (uint32_t)(ks * kstep(N1, PM)), B1LBO, 128);
                                const uint32_t acc = ks > 0 ? 1u : 0u;
                                if (STK) {   // hi(x) [W_hi | W_lo] (2N wide), then lo(x) W_hi
                                    mma_bf16(d, ad, bd, id1w, acc);
                                    mma_bf16(d, ad + LOA, bd, id1, 1u);
                                } else if (PM == 2) {   // hi(x) W_hi + lo(x) W_hi + hi(x) W_lo
                                    mma_bf16(d, ad, bd, id1, acc);
                                    mma_bf16(d, ad + LOA, bd, id1, 1u);
                                    mma_bf16(d, ad, bd + (uint64_t)(N1 * 32 / 16), id1, 1u);
                                } else {
                                    mma_bf16(d, ad, bd, id1, acc);
                                    if (PM == 1) mma_bf16(d, ad + LOA, bd, id1, 1u);
                                }
                            }
                            commit(&a1t[s * 2 + t]);
                        }
                    }
                    commit(&empty[slot]);
                    if (++slot == NSLOT) { slot = 0; phase ^= 1; }
                    // conv2 of both slots (TS mode: A = the hidden in TMEM)
                    TS_WAIT(c_f, mbar_wait(&full[slot], phase));
                    fence_after();
                    const uint32_t w2 = rb + (uint32_t)slot * SLOTB;
                    for (int s = 0; s < ns; s++) {
#pragma unroll
                        for (int t = 0; t < 2; t++) {
                            TS_WAIT(c_h, mbar_wait(&hdt[s * 2 + t], par));
                            fence_after();
                            const uint32_t tb = tmem + (uint32_t)(s * 256 + t * 128);
#pragma unroll
                            for (int ks = 0; ks < K2; ks++) {
                                // hidden channels 16 ks..16 ks+15: hi words at column 16 ks, lo at 16 ks + 8
                                const uint32_t ahi = tb + (uint32_t)(16 * ks);
                                const uint64_t bd = smem_desc(w2 + (uint32_t)(ks * kstep(N2, PM)), N2 * 16, 128);
                                const uint32_t acc = ks > 0 ? 1u : 0u;
                                mma_ts(tb + 64, ahi, bd, id2, acc);
                                if (PM >= 1) mma_ts(tb + 64, ahi + 8, bd, id2, 1u);                        // lo(h) W
                                if (PM == 2) mma_ts(tb + 64, ahi, bd + (uint64_t)(N2 * 32 / 16), id2, 1u);  // hi(h) W_lo
                            }
                            commit(&a2t[s * 2 + t]);
                        }
                    }
                    commit(&empty[slot]);
                    if (++slot == NSLOT) { slot = 0; phase ^= 1; }
                }
                if (ns == 1) break;
            }
            if (a.dbg) {
                unsigned long long* o = a.dbg + blockIdx.x * 16;
                o[0] = clock64() - c_t0; o[1] = c_x; o[2] = c_h; o[3] = c_f;
            }
        }
        __syncwarp();
    } else {
        // ================= epilogue: two independent groups of 8 warps, group g = image slot g ==
        // warp w reads TMEM lanes 32 (w % 4)..+31; in a group, warps w and w+4 share a lane quarter:
        // conv1 epilogue: half 0 takes hidden channels 0-31, half 1 hidden 32-63 (both tiles);
        // conv2 epilogue: half h takes M-tile h (all 6 outputs of its pixel rows)
        const int g = (warp - 2) >> 3, ew = (warp - 2) & 7, quarter = warp & 3, half = ew >> 2, et = ew * 32 + lane;
        const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
        const int x = lane & 15;
        const uint32_t bar_id = 1 + g;
        auto gsync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(kEpi) : "memory"); };
        uint8_t* xs = xplanes(g);
        float* xch0 = reinterpret_cast<float*>(sxch(g));
        const float2 ml = make_float2(x > 0 ? 1.f : 0.f, x > 0 ? 1.f : 0.f);          // left tap inside the image
        const float2 mr = make_float2(x < W - 1 ? 1.f : 0.f, x < W - 1 ? 1.f : 0.f);  // right tap inside the image
        // X views at row p: 8 channels (one 16-byte row per view and precision plane).  Branch-free:
        // the Xl / Xr rows a border pixel would feed are written as zeros (they must stay zero).
        auto write_x = [&](int p, const float (&v)[8]) {
            uint4 hi, lo;
            if (PM) {
                ts_split(v[0], v[1], hi.x, lo.x);
                ts_split(v[2], v[3], hi.y, lo.y);
                ts_split(v[4], v[5], hi.z, lo.z);
                ts_split(v[6], v[7], hi.w, lo.w);
            } else {
                hi = make_uint4(ts_bf16x2(v[0], v[1]), ts_bf16x2(v[2], v[3]), ts_bf16x2(v[4], v[5]), ts_bf16x2(v[6], v[7]));
                lo = hi;
            }
            const int xx = p & 15;
            const uint4 z4 = make_uint4(0, 0, 0, 0);
            const size_t off = (size_t)(G + p) * 16;
            auto put = [&](int view, int row_delta, bool keep) {
                *reinterpret_cast<uint4*>(xs + (size_t)view * PB + off + row_delta * 16) = keep ? hi : z4;
                if (PM) *reinterpret_cast<uint4*>(xs + (size_t)(3 + view) * PB + off + row_delta * 16) = keep ? lo : z4;
            };
            put(1, 0, true);         // Xc[p]
            put(0, 1, xx < W - 1);   // Xl[p+1] = X[p]
            put(2, -1, xx > 0);      // Xr[p-1] = X[p]
        };
        // image state (src, layout in_mode) -> shared-memory buffer (cp.async, completes on wait_all)
        auto fetch_state = [&](int64_t bb, float* dst) {
            io_fetch_async<C, H, W>(a.src + bb * (int64_t)C * HW, a.in_mode, dst, et, kEpi);
        };
        auto in_half = [&](int t) { return ((a.first_orient + t) & 1) == 0 ? 0 : c; };
        uint32_t kb = 0;
        bool prefetched = false;
        for (int i = 0;; i++) {
            const int qe = 2 * i + g;
            const int64_t b = bq_read(qe);
            mbar_arrive(&bqe[qe & 3]);
            if (b >= nbatch) break;
            float* gst = a.dst + b * (int64_t)C * HW;
            float* st = sstate(g) + (i & 1) * (C * HW);
            // ---- image state -> shared memory (prefetched during the previous image's last blocks)
            if (!prefetched) fetch_state(b, st);
            asm volatile("cp.async.wait_all;" ::: "memory");
            prefetched = false;
            gsync();
            {   // first block's input half -> X views
                const int ioff = in_half(a.inverse ? a.nb - 1 : 0);
                const int p = half * 128 + quarter * 32 + lane;
                float v[8];
#pragma unroll
                for (int o = 0; o < 8; o++) v[o] = o < c ? st[(ioff + o) * HW + p] : (o == c ? 1.f : 0.f);
                write_x(p, v);
                fence_proxy_async();
                mbar_arrive(&x_rdy[g]);
            }
            for (int tt = 0; tt < a.nb; tt++, kb++) {
                const uint32_t par = kb & 1;
                const int t = a.inverse ? a.nb - 1 - tt : tt;
                const int out_off = c - in_half(t);
                const bool write_next = tt + 1 < a.nb;
                float bb[c];   // conv2 bias of this block (loads in flight during the conv1 epilogue)
                {
                    const float* b2 = a.bias + (int64_t)t * a.bias_stride + M;
#pragma unroll
                    for (int o = 0; o < c; o++) bb[o] = __ldg(b2 + o);
                }
                if (tt == a.nb - 2 || (a.nb == 1 && tt == 0)) {   // prefetch the group's next image state
                    const int64_t bn = bq_read(qe + 2);
                    if (bn < nbatch) {
                        fetch_state(bn, sstate(g) + ((i + 1) & 1) * (C * HW));
                        prefetched = true;
                    }
                }
                // ---- conv1 epilogue: acc1 -> ReLU -> fp16 hi / lo (or bf16) words back into TMEM,
                // into the same columns this thread read (half h: columns [32h, 32h+32))
#pragma unroll
                for (int tl = 0; tl < 2; tl++) {
                    mbar_wait(&a1t[g * 2 + tl], par);
                    fence_after();
                    const uint32_t col = tmem + lane_addr + (uint32_t)(g * 256 + tl * 128 + 32 * half);
                    // two rounds of 16 hidden channels; round 1's loads are in flight while round 0 is
                    // converted (round 0 only writes columns it read, round 1 reads other columns)
                    float v[2][16], w[2][STK ? 16 : 1];
                    tmem_ld16(col, v[0]);
                    if constexpr (STK != 0) tmem_ld16(col + 64, *reinterpret_cast<float (*)[16]>(&w[0][0]));
                    tmem_wait_ld();
                    tmem_ld16(col + 16, v[1]);
                    if constexpr (STK != 0) tmem_ld16(col + 80, *reinterpret_cast<float (*)[16]>(&w[1][0]));
#pragma unroll
                    for (int rd = 0; rd < 2; rd++) {
                        if (rd == 1) tmem_wait_ld();
                        if constexpr (STK != 0) {   // stacked: hi(x) W_lo columns at +64
#pragma unroll
                            for (int e = 0; e < 8; e++) {
                                const float2 r = add2(make_float2(v[rd][2 * e], v[rd][2 * e + 1]),
                                                      make_float2(w[rd][2 * e], w[rd][2 * e + 1]));
                                v[rd][2 * e] = r.x;
                                v[rd][2 * e + 1] = r.y;
                            }
                        }
                        uint32_t hw[8], lw[8];
#pragma unroll
                        for (int e = 0; e < 8; e++) {
                            const float p0 = fmaxf(v[rd][2 * e], 0.f), p1 = fmaxf(v[rd][2 * e + 1], 0.f);
                            if (PM) ts_split(p0, p1, hw[e], lw[e]);
                            else hw[e] = ts_bf16x2(p0, p1);
                        }
                        // hidden channels 16 k..16 k+15 (k = 2 half + rd): hi words at column 16 k, lo
                        // words at 16 k + 8 -- only columns this round has already read
                        tmem_st8u(col + 16 * rd, hw);
                        if (PM) tmem_st8u(col + 16 * rd + 8, lw);
                    }
                    tmem_wait_st();
                    fence_before();
                    mbar_arrive(&hdt[g * 2 + tl]);
                }
                // ---- conv2 epilogue (tile `half`): col2im of the 9 tap groups, s_out (+|-)= F + b2
                const int p = half * 128 + quarter * 32 + lane, y = p >> 4;
                float* xch = xch0 + (par ? HW * 8 : 0);   // double-buffered by block parity
                float2 mid[c / 2];
                {
                    mbar_wait(&a2t[g * 2 + half], par);
                    fence_after();
                    const uint32_t col = tmem + lane_addr + (uint32_t)(g * 256 + half * 128 + 64);
                    float2 z[9][c / 2];   // column tap * 6 + o
                    {
                        float za[16], zb[16], zc[16], zd[4], ze[2];
                        tmem_ld16(col, za);
                        tmem_ld16(col + 16, zb);
                        tmem_ld16(col + 32, zc);
                        tmem_ld4(col + 48, zd);
                        tmem_ld2(col + 52, ze);
                        tmem_wait_ld();
                        auto zq = [&](int q) -> float {
                            return q < 16 ? za[q] : q < 32 ? zb[q - 16] : q < 48 ? zc[q - 32] : q < 52 ? zd[q - 48] : ze[q - 52];
                        };
#pragma unroll
                        for (int q = 0; q < 27; q++) z[q / 3][q % 3] = make_float2(zq(2 * q), zq(2 * q + 1));
                    }
                    fence_before();
                    // horizontal: H_u[r] = Z_{u,-1}[r-1] + Z_{u,0}[r] + Z_{u,+1}[r+1] (masked at x = 0 / W-1)
                    float2 hsum[3][c / 2];
#pragma unroll
                    for (int u = 0; u < 3; u++)
#pragma unroll
                        for (int o = 0; o < c / 2; o++) {
                            const float2 zl = z[u * 3 + 0][o], zr = z[u * 3 + 2][o];
                            const float2 l = make_float2(__shfl_up_sync(0xffffffffu, zl.x, 1), __shfl_up_sync(0xffffffffu, zl.y, 1));
                            const float2 r = make_float2(__shfl_down_sync(0xffffffffu, zr.x, 1), __shfl_down_sync(0xffffffffu, zr.y, 1));
                            hsum[u][o] = fma2(l, ml, fma2(r, mr, z[u * 3 + 1][o]));
                        }
                    // vertical: out[p] = H_-1[p-W] + H_0[p] + H_+1[p+W].  Lanes l < 16 (even y) take
                    // H_+1 of lane l+16 and publish their H_+1 for the warp row above; lanes >= 16
                    // take H_-1 of lane l-16 and publish their H_-1 for the warp row below.
                    float2 pub[c / 2];
#pragma unroll
                    for (int o = 0; o < c / 2; o++) {
                        const float2 send = lane < 16 ? hsum[0][o] : hsum[2][o];
                        const float2 recv = make_float2(__shfl_xor_sync(0xffffffffu, send.x, 16), __shfl_xor_sync(0xffffffffu, send.y, 16));
                        mid[o] = add2(add2(hsum[1][o], recv), make_float2(bb[2 * o], bb[2 * o + 1]));
                        pub[o] = lane < 16 ? hsum[2][o] : hsum[0][o];
                    }
                    reinterpret_cast<float4*>(xch)[p] = make_float4(pub[0].x, pub[0].y, pub[1].x, pub[1].y);
                    reinterpret_cast<float2*>(xch + 4 * HW)[p] = pub[2];
                }
                gsync();
                {
                    float* st = sstate(g) + (i & 1) * (C * HW);
                    const int q = lane < 16 ? (y > 0 ? p - W : -1) : (y < H - 1 ? p + W : -1);
                    float4 o0 = make_float4(0.f, 0.f, 0.f, 0.f);
                    float2 o1 = make_float2(0.f, 0.f);
                    if (q >= 0) { o0 = reinterpret_cast<const float4*>(xch)[q]; o1 = reinterpret_cast<const float2*>(xch + 4 * HW)[q]; }
                    const float2 ov[3] = {make_float2(o0.x, o0.y), make_float2(o0.z, o0.w), o1};
                    float nv[8];
#pragma unroll
                    for (int o2 = 0; o2 < c / 2; o2++) {
                        const float2 f = add2(mid[o2], ov[o2]);
                        float* sp = st + (out_off + 2 * o2) * HW + p;
                        const float2 old = make_float2(sp[0], sp[HW]);
                        const float2 n2 = a.inverse ? sub2(old, f) : add2(old, f);
                        sp[0] = n2.x;
                        sp[HW] = n2.y;
                        nv[2 * o2] = n2.x;
                        nv[2 * o2 + 1] = n2.y;
                    }
                    nv[6] = 1.f;   // constant-1 channel (folded conv1 bias)
                    nv[7] = 0.f;
                    if (write_next) {
                        write_x(p, nv);
                        fence_proxy_async();
                        mbar_arrive(&x_rdy[g]);
                    }
                }
            }
            // ---- state back to global memory
            gsync();
            io_store<C, H, W>(gst, a.out_mode, sstate(g) + (i & 1) * (C * HW), et, kEpi);   // layout out_mode
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

bool stage_ts_shape(int H, int W, int C, int c, int m, int residual, int act) {
    return H == ts::H && W == ts::W && C == ts::C && c == ts::c && m == ts::M && !residual && act == 0 &&
           !getenv("CI_NO_TS");
}
int64_t stage_ts_block_bytes(int pm) { return (int64_t)ts::K1 * ts::kstep(ts::N1, pm) + ts::K2 * ts::kstep(ts::N2, pm); }
int stage_ts_n2() { return ts::N2; }
int stage_ts_smem(int pm) { return ts::smem_bytes(pm); }

// conv2 column n of the TS layout -> (tap, output channel), or tap = -1 for padding columns
void stage_ts_col(int n, int& tap, int& o) {
    if (n < 9 * ts::c) { tap = n / ts::c; o = n % ts::c; return; }
    tap = -1; o = -1;
}

typedef void (*TsKernel)(TsArgs);
static TsKernel ts_kernel(int pm, int stk) {
    return pm == 2 ? (stk ? k_stage_ts<2, 1> : k_stage_ts<2, 0>) : (pm == 1 ? k_stage_ts<1, 0> : k_stage_ts<0, 0>);
}

cudaError_t stage_ts_prepare() {
    cudaError_t e = cudaSuccess;
    for (int pm = 0; pm < 3 && e == cudaSuccess; pm++)
        for (int stk = 0; stk < (pm == 2 ? 2 : 1) && e == cudaSuccess; stk++)
            e = cudaFuncSetAttribute(ts_kernel(pm, stk), cudaFuncAttributeMaxDynamicSharedMemorySize, ts::smem_bytes(pm));
    return e;
}

bool stage_ts_stacked(int pm) { return pm == 2 && !getenv("CI_TS_UNSTK"); }

cudaError_t launch_stage_ts(const TsArgs& a, int pm, int stk, cudaStream_t st) {
    const int grid = (int)std::min<int64_t>((a.n + 1) / 2, 148);
    if (a.n <= 0) return cudaSuccess;
    ts_kernel(pm, stk)<<<grid, ts::kThreads, ts::smem_bytes(pm), st>>>(a);
    return cudaGetLastError();
}

}  // namespace ci
