// Stage 2 of Arch C (8x8 images, c = 24 coupling channels, m = 128 hidden) as a TS-mode kernel.
// DESIGN.md 7.2c.  Same block as k_stage / k_stage_ts (i-RevNet-style additive coupling, PAPER.md:168;
// reading Q1 of DESIGN.md 2):
//   s_out <- s_out (+|-) F(s_in),  F = conv3x3(W2) o ReLU o conv3x3(W1).
//
//  * Two images per 128-row M-tile with no pad rows or columns (100% of the MMA rows are
//    pixels; k_stage's padded raster held 3 images in 2 tiles = 75%), rows interleaved by image
//    row: r = 16 y + 8 img + x.  A vertical tap is then a row shift of 16 that stays inside the
//    image (rows beyond the tile are zero guard rows), and a horizontal tap uses one of three
//    views of the input, Xc, Xl[r] = X[r-1] (0 at x = 0), Xr[r] = X[r+1] (0 at x = 7).  conv1 runs
//    14 K = 16 steps over (vertical shift, view, 8-channel plane) pairs + the constant-1 plane
//    (folded conv1 bias), the two K halves of a step LBO bytes apart.
//  * The hidden (128 channels, ReLU, fp16 hi + lo) is written back into TMEM over acc1 and read
//    by conv2 in TS mode (A from TMEM).  conv2 stacks all 9 taps in N: two passes over the
//    outputs (channels 0-11 then 12-23; N = 108 -> 112 each: column 54 half + 6 tap + o), so a
//    slot needs 128 + 112 TMEM columns.  The epilogue forms out[r] = sum_{u,v} Z_{u,v}[r + 16u + v]:
//    horizontal neighbours are lanes +-1 (masked at x = 0 / 7), vertical ones lanes +-16 (one
//    xor-16 shuffle) or the neighbouring warp's rows (one exchange through shared memory).
//  * Two slots (tiles) per CTA with their own views, state and group of 8 epilogue warps.  The
//    MMA thread runs slot B half a block behind slot A: conv1(A,k) conv2(B,k-1) conv2(A,k)
//    conv1(B,k), so every hand-off between a slot's epilogue and its next MMA step is covered by
//    at least one conv1 or two conv2 passes of the other slot.
//  * The fp32 state of the slot's two images stays in shared memory for the whole stage; it is read
//    and written in the layouts the caller names (stage_io.cuh: the squeeze psi / psi^-1 at the
//    stage boundaries fused into the load / store).
//  * Weights stream through a 3 x 24 KB ring per slot-block; the ring's depth (per-piece latency,
//    not the chip's L2 -> SM bytes: halving those with cluster multicast, MC below, did not help)
//    is this kernel's bound.
#include <stdio.h>

#include "ci_internal.h"
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "stage_io.cuh"
#include "umma.cuh"

namespace ci {
using namespace umma;

namespace ts2 {
constexpr int kThreads = 576;      // warp 0 producer, warp 1 MMA, warps 2..17 epilogue (2 groups)
constexpr int kEpi = 256;
constexpr int H = 8, W = 8, HW = 64, C = 48, c = 24, M = 128;
constexpr int NPL = 10;                     // view planes: 3 views x 3 planes of 8 channels + constant-1
constexpr int G = 16;                       // guard rows above / below the 128 tile rows (one row shift)
constexpr int PB = (128 + G) * 16;          // plane stride: 128 rows + 16 guard rows shared with the next plane
constexpr int LOB = (G + NPL * (128 + G)) * 16;   // one precision's planes (leading guard + 10 strides)
constexpr int N1 = 128, N2 = 112;           // conv1 / conv2-pass MMA widths
constexpr int K1 = 14, K2 = 8;              // k-steps
// weight ring: three k-steps per slot in f16x3 (conv1 24 KB, conv2 21 KB).  Measured: the stream is
// bound by the per-copy latency, not the bytes in flight (8 x 8 KB slots: s1 +30%, 4 x 16 KB: 0.69 ms)
constexpr int NSLOT = 3, SLOTB = 24576;
constexpr int ST_BYTES = 2 * C * HW * 4;    // fp32 state of the slot's two images
constexpr int XCH_BYTES = 2 * 128 * 24;     // vertical exchange [half][row][6] fp32 (both passes)
__host__ __device__ constexpr int kstep(int N, int pm) { return N * 32 * (pm == 2 ? 2 : 1); }
__host__ __device__ constexpr int per_slot(int N, int pm) { return SLOTB / kstep(N, pm); }
__host__ __device__ constexpr int view_bytes(int pm) { return (pm ? 2 : 1) * LOB; }
__host__ __device__ constexpr int slot_bytes(int pm) { return view_bytes(pm) + ST_BYTES + XCH_BYTES; }
__host__ __device__ constexpr int smem_bytes(int pm) { return NSLOT * SLOTB + 2 * slot_bytes(pm) + 512; }
// conv1 k-step s: A start (bytes from the plane base of the views) and LBO (bytes)
__host__ __device__ constexpr int k1_start(int s) {
    return s < 12 ? 2 * (s % 4) * PB + (G + 16 * (s / 4 - 1)) * 16 : 8 * PB + (G + (s == 12 ? -16 : 16)) * 16;
}
__host__ __device__ constexpr int k1_lbo(int s) { return s < 12 ? PB : (s == 12 ? 256 : PB - 256); }
}  // namespace ts2

namespace {
// cycle counters (CI_DEBUG_CYCLES): time spent in `call` added to acc when a.dbg is set.  The MMA
// thread's are always compiled in; the epilogue's only with -DCI_TS_EPI_CYCLES (they cost registers).
#ifdef CI_TS_EPI_CYCLES
constexpr bool kEpiCycles = true;
#else
constexpr bool kEpiCycles = false;
#endif
#define T2_WAIT(acc, call)                                             \
    do {                                                               \
        const long long t0_ = a.dbg ? clock64() : 0;                   \
        call;                                                          \
        if (a.dbg) acc += (unsigned long long)(clock64() - t0_);       \
    } while (0)
#define T2_EWAIT(acc, call)                                                        \
    do {                                                                           \
        const long long t0_ = (kEpiCycles && a.dbg) ? clock64() : 0;               \
        call;                                                                      \
        if (kEpiCycles && a.dbg) acc += (unsigned long long)(clock64() - t0_);     \
    } while (0)
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

// MC: launched as clusters of two CTAs that stream the same weight sequence; each CTA copies half
// of every ring piece and multicasts it to both (one L2 read per pair: half the per-SM L2 -> SM
// bytes), and a piece is refilled only after both CTAs' MMAs released it (empty count 2, commits
// multicast to the pair).  Batches are assigned statically, four per cluster and iteration.
template <int PM, bool MC>
__global__ void __launch_bounds__(ts2::kThreads, 1) k_stage_ts2(TsArgs a) {
    using namespace ts2;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint8_t* ring = smem;
    uint8_t* slots = ring + NSLOT * SLOTB;   // [2] x { views [hi: 10 planes][lo: 10 planes], state, xch }
    auto sviews = [&](int s) { return slots + (size_t)s * slot_bytes(PM); };
    auto sstate = [&](int s) { return reinterpret_cast<float*>(slots + (size_t)s * slot_bytes(PM) + view_bytes(PM)); };
    auto sxch = [&](int s) {
        return reinterpret_cast<float*>(slots + (size_t)s * slot_bytes(PM) + view_bytes(PM) + ST_BYTES);
    };
    uint64_t* bars = reinterpret_cast<uint64_t*>(slots + 2 * slot_bytes(PM));
    uint64_t* full = bars;            // [NSLOT]
    uint64_t* empty = bars + 8;       // [NSLOT]
    uint64_t* bqf = bars + 16;        // [4]
    uint64_t* bqe = bars + 20;        // [4]
    uint64_t* x_rdy = bars + 24;      // [2] views of slot s final for its next conv1
    uint64_t* a1t = bars + 26;        // [2] conv1 of slot s done (commit)
    uint64_t* hdt = bars + 28;        // [2] hidden of slot s in TMEM
    uint64_t* a2t = bars + 30;        // [2] conv2 pass of slot s done (commit; twice per block)
    uint64_t* a2r = bars + 32;        // [2] pass-a accumulator of slot s read (pass b may overwrite)
    volatile int64_t* bq = reinterpret_cast<volatile int64_t*>(bars + 34);   // [4]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 38);

    {   // views: zero (guards, x borders of Xl / Xr); constant-1 plane: channel 0 = 1.0 on the tile rows
        uint4 z = make_uint4(0, 0, 0, 0);
        for (int s = 0; s < 2; s++)
            for (int i = tid; i < view_bytes(PM) / 16; i += kThreads) reinterpret_cast<uint4*>(sviews(s))[i] = z;
        __syncthreads();
        const uint32_t one = PM ? 0x3C00u : 0x3F80u;   // fp16 / bf16 1.0 in the low half
        for (int i = tid; i < 2 * 128; i += kThreads)
            *reinterpret_cast<uint4*>(sviews(i >> 7) + (size_t)9 * PB + (size_t)(G + (i & 127)) * 16) = make_uint4(one, 0, 0, 0);
    }
    fence_proxy_async();
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    if (tid == 0) {
        for (int i = 0; i < NSLOT; i++) { mbar_init(&full[i], 1); mbar_init(&empty[i], MC ? 2 : 1); }
        for (int i = 0; i < 4; i++) { mbar_init(&bqf[i], 1); mbar_init(&bqe[i], 1 + kEpi); }
        for (int i = 0; i < 2; i++) {
            mbar_init(&x_rdy[i], kEpi); mbar_init(&a1t[i], 1); mbar_init(&hdt[i], kEpi);
            mbar_init(&a2t[i], 1); mbar_init(&a2r[i], kEpi);
        }
        fence_mbar_init();
    }
    fence_before();
    __syncthreads();
    if (MC) cluster_sync();   // the peer's barriers are initialised before any multicast reaches them
    fence_after();
    const uint32_t tmem = *tmem_slot;
    const int crank = MC ? (int)cluster_rank() : 0;
    const int64_t ncl = gridDim.x >> 1, cid = blockIdx.x >> 1;
    auto mc_base = [&](int pi) -> int64_t { return 4 * (cid + (int64_t)pi * ncl); };   // MC: the cluster's first batch
    const int64_t nbatch = (a.n + 1) / 2;   // two images per slot batch
    auto bq_read = [&](int i) -> int64_t {
        mbar_wait(&bqf[i & 3], (uint32_t)((i >> 2) & 1));
        return bq[i & 3];
    };
    const int SEG1 = K1 * kstep(N1, PM), SEG2 = K2 * kstep(N2, PM);
    constexpr int G1 = per_slot(N1, PM), G2 = per_slot(N2, PM);   // k-steps per ring slot
    // MMA order of one image pair as (segment, block, slot); segment 0 = conv1, 1 = conv2 pass a,
    // 2 = pass b.  Default (a.sched == 1): slot B half a block behind slot A, each segment streamed
    // per slot: conv1(A,k) conv2a/b(B,k-1) conv2a/b(A,k) conv1(B,k).  a.sched == 0 (CI_TS2_LOCKSTEP):
    // per block conv1, conv2a, conv2b for both slots with their k-steps interleaved per ring piece
    // (slot -1), every weight byte streamed once per pair -- measured 12% slower: the ring waits
    // drop (0.90M -> 0.31M cycles) but each slot's epilogue is no longer covered by the other's MMAs.
    auto for_each_step = [&](int ns, auto&& f) {
        if (a.sched == 0) {
            for (int k = 0; k < a.nb; k++) { f(0, k, -1); f(1, k, -1); f(2, k, -1); }
            return;
        }
        for (int k = 0; k <= a.nb; k++) {
            if (k < a.nb) f(0, k, 0);
            if (ns == 2 && k >= 1) { f(1, k - 1, 1); f(2, k - 1, 1); }
            if (k < a.nb) { f(1, k, 0); f(2, k, 0); }
            if (ns == 2 && k < a.nb) f(0, k, 1);
        }
    };

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
            for (int pi = 0; MC; pi++) {
                const int64_t base = mc_base(pi), b0 = base + 2 * crank, b1 = b0 + 1;
                publish(2 * pi, b0 < nbatch ? b0 : nbatch);
                publish(2 * pi + 1, b1 < nbatch ? b1 : nbatch);
                if (base >= nbatch) break;
                for_each_step(2, [&](int seg, int k, int) {
                    const int t = a.inverse ? a.nb - 1 - k : k;
                    const uint8_t* src = a.wpack + (int64_t)t * a.blk_bytes + (seg == 0 ? 0 : SEG1 + (seg - 1) * SEG2);
                    const int K = seg == 0 ? K1 : K2, Gs = seg == 0 ? G1 : G2, kb = seg == 0 ? kstep(N1, PM) : kstep(N2, PM);
                    for (int s0 = 0; s0 < K; s0 += Gs) {
                        const uint32_t bytes = (uint32_t)(min(Gs, K - s0) * kb), hb = bytes / 2;
                        mbar_wait(&empty[slot], phase ^ 1);   // both CTAs released the piece
                        mbar_arrive_expect_tx(&full[slot], bytes);
                        bulk_g2s_mc(ring + (size_t)slot * SLOTB + crank * hb, src + (size_t)s0 * kb + crank * hb, hb,
                                    &full[slot], (uint16_t)3);
                        if (++slot == NSLOT) { slot = 0; phase ^= 1; }
                    }
                });
            }
            if (MC)   // every release (ours and the peer's) has arrived before the CTA may exit
                for (int i = 0; i < NSLOT; i++) {
                    mbar_wait(&empty[slot], phase ^ 1);
                    if (++slot == NSLOT) { slot = 0; phase ^= 1; }
                }
            for (int pi = 0; !MC; pi++) {
                const int64_t b0 = next();
                const int64_t b1 = b0 < nbatch ? next() : nbatch;
                publish(2 * pi, b0);
                publish(2 * pi + 1, b1);
                if (b0 >= nbatch) break;
                for_each_step(b1 < nbatch ? 2 : 1, [&](int seg, int k, int) {
                    const int t = a.inverse ? a.nb - 1 - k : k;
                    const uint8_t* src = a.wpack + (int64_t)t * a.blk_bytes + (seg == 0 ? 0 : SEG1 + (seg - 1) * SEG2);
                    const int K = seg == 0 ? K1 : K2, Gs = seg == 0 ? G1 : G2, kb = seg == 0 ? kstep(N1, PM) : kstep(N2, PM);
                    for (int s0 = 0; s0 < K; s0 += Gs) {
                        const uint32_t bytes = (uint32_t)(min(Gs, K - s0) * kb);
                        mbar_wait(&empty[slot], phase ^ 1);
                        mbar_arrive_expect_tx(&full[slot], bytes);
                        bulk_g2s(ring + (size_t)slot * SLOTB, src + (size_t)s0 * kb, bytes, &full[slot]);
                        if (++slot == NSLOT) { slot = 0; phase ^= 1; }
                    }
                });
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
            uint32_t phase = 0;
            uint32_t kbs[2] = {0, 0};   // blocks completed per slot (barrier phases)
            const uint32_t rb = smem_u32(ring);
            const uint32_t id1 = idesc_of(128, N1, PM != 0);
            const uint32_t id2 = idesc_of(128, N2, PM != 0);
            constexpr uint32_t LOA = (uint32_t)(LOB / 16);   // lo planes, descriptor units
            unsigned long long c_x = 0, c_h = 0, c_f = 0;
            const long long c_t0 = clock64();
            auto acquire = [&]() -> uint32_t {
                T2_WAIT(c_f, mbar_wait(&full[slot], phase));
                fence_after();
                return rb + (uint32_t)slot * SLOTB;
            };
            auto release = [&]() {
                if (MC) commit_mc(&empty[slot], (uint16_t)3);
                else commit(&empty[slot]);
                if (++slot == NSLOT) { slot = 0; phase ^= 1; }
            };
            for (int pi = 0;; pi++) {
                const int64_t b0 = bq_read(2 * pi);
                mbar_arrive(&bqe[(2 * pi) & 3]);
                if (!MC && b0 >= nbatch) break;
                const int64_t b1 = bq_read(2 * pi + 1);
                mbar_arrive(&bqe[(2 * pi + 1) & 3]);
                if (MC && mc_base(pi) >= nbatch) break;
                // MC: the pair streams both slots' weights whether or not this CTA has the batches
                const int ns = (MC || b1 < nbatch) ? 2 : 1;
                const bool valid[2] = {b0 < nbatch, b1 < nbatch};
                for_each_step(ns, [&](int seg, int, int sl) {
                    // slots this step runs (sl = -1: both, k-steps interleaved per ring piece)
                    const int s_lo = sl < 0 ? 0 : sl, s_hi = sl < 0 ? ns : sl + 1;
                    const int K = seg == 0 ? K1 : K2, Gs = seg == 0 ? G1 : G2;
                    for (int s0 = 0; s0 < K; s0 += Gs) {
                        const uint32_t w = acquire();
                        for (int s = s_lo; s < s_hi; s++) {
                            if (MC && !valid[s]) continue;
                            const uint32_t par = kbs[s] & 1;
                            const uint32_t tb = tmem + (uint32_t)(s * 256);
                            if (s0 == 0) {   // the slot's operand is ready: views (conv1), hidden (pass a), pass a read (b)
                                if (seg == 0) T2_WAIT(c_x, mbar_wait(&x_rdy[s], par));
                                else T2_WAIT(c_h, mbar_wait(seg == 1 ? &hdt[s] : &a2r[s], par));
                                fence_after();
                            }
                            if (seg == 0) {   // conv1 (SS: A = the views, vertical taps as row shifts of 16)
                                const uint32_t vb = smem_u32(sviews(s));
#pragma unroll
                                for (int q = 0; q < G1; q++) {
                                    const int ks = s0 + q;
                                    if (ks >= K1) break;
                                    const uint64_t ad = smem_desc(vb + (uint32_t)k1_start(ks), (uint32_t)k1_lbo(ks), 128);
                                    const uint64_t bd = smem_desc(w + (uint32_t)(q * kstep(N1, PM)), N1 * 16, 128);
                                    const uint32_t acc = ks > 0 ? 1u : 0u;
                                    mma_bf16(tb, ad, bd, id1, acc);
                                    if (PM >= 1) mma_bf16(tb, ad + LOA, bd, id1, 1u);
                                    if (PM == 2) mma_bf16(tb, ad, bd + (uint64_t)(N1 * 32 / 16), id1, 1u);
                                }
                            } else {          // conv2 pass (TS: A = the hidden in TMEM)
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
                            }
                        }
                        release();
                    }
                    for (int s = s_lo; s < s_hi; s++) {
                        if (MC && !valid[s]) continue;
                        commit(seg == 0 ? &a1t[s] : &a2t[s]);
                        if (seg == 2) kbs[s]++;
                    }
                });
                if (!MC && ns == 1) break;
            }
            if (a.dbg) {
                unsigned long long* o = a.dbg + blockIdx.x * 16;
                o[0] = clock64() - c_t0; o[1] = c_x; o[2] = c_h; o[3] = c_f;
            }
        }
        __syncwarp();
    } else {
        // ================= epilogue: group g = slot g (8 warps) ================================
        // row r = 32 quarter + lane: y = r / 16, image (r / 8) % 2, x = r % 8.  Warps w and w+4 share
        // a lane quarter: conv1 epilogue half h = hidden 64h..64h+63; conv2 epilogue half h =
        // outputs 12 pass + 6h..+5; view writes: half 0 = (view, plane) combos 0-4, half 1 = 5-8.
        const int g = (warp - 2) >> 3, ew = (warp - 2) & 7, quarter = warp & 3, half = ew >> 2, et = ew * 32 + lane;
        const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
        const int r = quarter * 32 + lane, y = r >> 4, img = (r >> 3) & 1, x = r & 7, pp = 8 * y + x;
        const uint32_t bar_id = 1 + g;
        auto gsync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(kEpi) : "memory"); };
        uint8_t* views = sviews(g);
        float* st = sstate(g);
        float* xch0 = sxch(g);
        const float2 ml = make_float2(x > 0 ? 1.f : 0.f, x > 0 ? 1.f : 0.f);
        const float2 mr = make_float2(x < W - 1 ? 1.f : 0.f, x < W - 1 ? 1.f : 0.f);
        auto in_half = [&](int t) { return ((a.first_orient + t) & 1) == 0 ? 0 : c; };
        // views <- this pixel's 24 channels at offset ch0 of the state (the next conv1's input).
        // Branch-free: a border pixel writes zeros into the Xl / Xr rows it would otherwise feed.
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
            const uint4 z4 = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int cb = 0; cb < 9; cb++) {
                if ((cb < 5) != (half == 0)) continue;
                const int view = cb / 3, pl = cb % 3;   // view 0 = l (row r+1), 1 = c (row r), 2 = r (row r-1)
                const int row = r + 1 - view;
                const bool keep = view == 1 || (view == 0 ? x < W - 1 : x > 0);
                const size_t off = (size_t)(view * 3 + pl) * PB + (size_t)(G + row) * 16;
                const uint4 h4 = make_uint4(hi[4 * pl], hi[4 * pl + 1], hi[4 * pl + 2], hi[4 * pl + 3]);
                *reinterpret_cast<uint4*>(views + off) = keep ? h4 : z4;
                if (PM) {
                    const uint4 l4 = make_uint4(lo[4 * pl], lo[4 * pl + 1], lo[4 * pl + 2], lo[4 * pl + 3]);
                    *reinterpret_cast<uint4*>(views + (size_t)LOB + off) = keep ? l4 : z4;
                }
            }
        };
        uint32_t kb = 0;
        unsigned long long c_a1 = 0, c_a2 = 0, c_e1 = 0, c_e2 = 0, c_v = 0, c_io = 0;
        const long long c_t0 = clock64();
        for (int i = 0;; i++) {
            const int qe = 2 * i + g;
            const int64_t b = bq_read(qe);
            mbar_arrive(&bqe[qe & 3]);
            if (b >= nbatch) break;
            const int64_t img0 = 2 * b;
            const int nimg = a.n - img0 < 2 ? 1 : 2;
            float* gst = a.dst + img0 * (int64_t)C * HW;
            const long long c_ios = (kEpiCycles && a.dbg) ? clock64() : 0;
            // the slot's state (src, layout in_mode) -> shared memory
            for (int ii = 0; ii < nimg; ii++)
                io_load<C, H, W>(a.src + (img0 + ii) * (int64_t)C * HW, a.in_mode, st + ii * C * HW, et, kEpi);
            gsync();
            write_views(in_half(a.inverse ? a.nb - 1 : 0), nimg);
            fence_proxy_async();
            mbar_arrive(&x_rdy[g]);
            if (kEpiCycles && a.dbg) c_io += (unsigned long long)(clock64() - c_ios);
            for (int tt = 0; tt < a.nb; tt++, kb++) {
                const uint32_t par = kb & 1;
                if (tt == a.nb - 3) {   // L2 prefetch of the group's next batch, if the producer has published it
                    const int qn = qe + 2;
                    if (mbar_test(&bqf[qn & 3], (uint32_t)((qn >> 2) & 1))) {
                        const int64_t bn = bq[qn & 3];
                        if (bn < nbatch) {
                            const int64_t in0 = 2 * bn, nb_img = a.n - in0 < 2 ? 1 : 2;
                            const char* pf = reinterpret_cast<const char*>(a.src + in0 * (int64_t)C * HW);
                            for (int off = et * 128; off < nb_img * C * HW * 4; off += kEpi * 128)
                                asm volatile("prefetch.global.L2 [%0];" ::"l"(pf + off));
                        }
                    }
                }
                const int t = a.inverse ? a.nb - 1 - tt : tt;
                const int out_off = c - in_half(t);
                const bool write_next = tt + 1 < a.nb;
                const float* b2 = a.bias + (int64_t)t * a.bias_stride + M;
                // ---- conv1 epilogue: acc1 -> ReLU -> fp16 hi | lo words over the columns just read
                T2_EWAIT(c_a1, mbar_wait(&a1t[g], par));
                fence_after();
                const long long c_e1s = (kEpiCycles && a.dbg) ? clock64() : 0;
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
                if (kEpiCycles && a.dbg) c_e1 += (unsigned long long)(clock64() - c_e1s);
                const long long c_e2s = (kEpiCycles && a.dbg) ? clock64() : 0;
                unsigned long long c_a2b = 0;
                // ---- conv2 epilogue, two passes: col2im of the 9 tap groups, s_out (+|-)= F + b2
#pragma unroll 1
                for (int pass = 0; pass < 2; pass++) {
                    const int ch0 = 12 * pass + 6 * half;   // this thread's 6 outputs
                    float2 bb[3];
#pragma unroll
                    for (int o = 0; o < 3; o++) bb[o] = make_float2(__ldg(b2 + ch0 + 2 * o), __ldg(b2 + ch0 + 2 * o + 1));
                    T2_EWAIT(c_a2b, mbar_wait(&a2t[g], (uint32_t)pass));
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
                            const float2 rr = make_float2(__shfl_down_sync(0xffffffffu, zr.x, 1), __shfl_down_sync(0xffffffffu, zr.y, 1));
                            hs[u][o] = t2_fma2(l, ml, t2_fma2(rr, mr, z[u * 3 + 1][o]));
                        }
                    // vertical: out[r] = H_-1[r-16] + H_0[r] + H_+1[r+16].  Lanes < 16 (even y) take H_+1 of
                    // lane +16 and publish their H_+1 for the warp above; lanes >= 16 take H_-1 of lane
                    // -16 and publish their H_-1 for the warp below.
                    float* xch = xch0 + half * (128 * 6);
                    if (pass == 1) gsync();   // every thread has read pass a's exchange values
                    float2 mid[3], pub[3];
#pragma unroll
                    for (int o = 0; o < 3; o++) {
                        const float2 send = lane < 16 ? hs[0][o] : hs[2][o];
                        const float2 recv = make_float2(__shfl_xor_sync(0xffffffffu, send.x, 16), __shfl_xor_sync(0xffffffffu, send.y, 16));
                        mid[o] = t2_add2(t2_add2(hs[1][o], recv), bb[o]);
                        pub[o] = lane < 16 ? hs[2][o] : hs[0][o];
                    }
#pragma unroll
                    for (int o = 0; o < 3; o++) reinterpret_cast<float2*>(xch)[3 * r + o] = pub[o];
                    gsync();
                    const int q = lane < 16 ? (y > 0 ? r - 16 : -1) : (y < H - 1 ? r + 16 : -1);
                    if (q >= 0) {
#pragma unroll
                        for (int o = 0; o < 3; o++) mid[o] = t2_add2(mid[o], reinterpret_cast<const float2*>(xch)[3 * q + o]);
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
                if (kEpiCycles && a.dbg) { c_a2 += c_a2b; c_e2 += (unsigned long long)(clock64() - c_e2s) - c_a2b; }
                if (write_next) {
                    const long long c_vs = (kEpiCycles && a.dbg) ? clock64() : 0;
                    gsync();   // the pixel's 24 updated channels come from both halves and both passes
                    write_views(out_off, nimg);
                    fence_proxy_async();
                    mbar_arrive(&x_rdy[g]);
                    if (kEpiCycles && a.dbg) c_v += (unsigned long long)(clock64() - c_vs);
                }
            }
            // ---- state back to global memory
            gsync();
            for (int ii = 0; ii < nimg; ii++)   // layout out_mode
                io_store<C, H, W>(gst + ii * C * HW, a.out_mode, st + ii * C * HW, et, kEpi);
            gsync();
        }
        if (kEpiCycles && a.dbg && g == 0 && et == 0) {
            unsigned long long* o = a.dbg + blockIdx.x * 16;
            o[6] = clock64() - c_t0; o[7] = c_a1; o[8] = c_a2; o[9] = c_e1; o[10] = c_e2; o[11] = c_v; o[12] = c_io;
        }
    }
    fence_before();
    __syncthreads();
    if (MC) cluster_sync();   // no multicast or remote arrival still in flight towards either CTA
    if (warp == 1) tmem_dealloc(tmem, 512);
}

bool stage_ts2_shape(int H, int W, int C, int c, int m, int residual, int act) {
    return H == ts2::H && W == ts2::W && C == ts2::C && c == ts2::c && m == ts2::M && !residual && act == 0 &&
           !getenv("CI_NO_TS2");
}
int64_t stage_ts2_block_bytes(int pm) {
    return (int64_t)ts2::K1 * ts2::kstep(ts2::N1, pm) + 2 * (int64_t)ts2::K2 * ts2::kstep(ts2::N2, pm);
}

int stage_ts2_smem(int pm) { return ts2::smem_bytes(pm); }

typedef void (*Ts2Kernel)(TsArgs);
static Ts2Kernel ts2_kernel(int pm, bool mc) {
    if (mc) return pm == 2 ? k_stage_ts2<2, true> : (pm == 1 ? k_stage_ts2<1, true> : k_stage_ts2<0, true>);
    return pm == 2 ? k_stage_ts2<2, false> : (pm == 1 ? k_stage_ts2<1, false> : k_stage_ts2<0, false>);
}
static bool ts2_mc() { static const bool on = getenv("CI_TS2_MC") != nullptr; return on; }   // A/B switch
static int ts2_max_clusters[3] = {0, 0, 0};

static cudaLaunchConfig_t ts2_config(int pm, int grid, cudaStream_t st, cudaLaunchAttribute* attr) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(ts2::kThreads);
    cfg.dynamicSmemBytes = ts2::smem_bytes(pm);
    cfg.stream = st;
    attr->id = cudaLaunchAttributeClusterDimension;
    attr->val.clusterDim.x = 2;
    attr->val.clusterDim.y = 1;
    attr->val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cfg;
}

cudaError_t stage_ts2_prepare() {
    cudaError_t e = cudaSuccess;
    for (int pm = 0; pm < 3 && e == cudaSuccess; pm++)
        for (int mc = 0; mc < 2 && e == cudaSuccess; mc++)
            e = cudaFuncSetAttribute(ts2_kernel(pm, mc), cudaFuncAttributeMaxDynamicSharedMemorySize, ts2::smem_bytes(pm));
    for (int pm = 0; pm < 3 && e == cudaSuccess; pm++) {   // pairs of SMs the cluster launch can hold at once
        cudaLaunchAttribute attr;
        cudaLaunchConfig_t cfg = ts2_config(pm, 2, nullptr, &attr);
        if (cudaOccupancyMaxActiveClusters(&ts2_max_clusters[pm], (const void*)ts2_kernel(pm, true), &cfg) != cudaSuccess) {
            ts2_max_clusters[pm] = 0;   // no cluster launch: the single-CTA kernel runs
            (void)cudaGetLastError();
        }
    }
    if (getenv("CI_DEBUG_PLAN"))
        fprintf(stderr, "[ci plan] ts2 cluster pairs resident: %d %d %d\n", ts2_max_clusters[0], ts2_max_clusters[1],
                ts2_max_clusters[2]);
    return e;
}

cudaError_t launch_stage_ts2(const TsArgs& a, int pm, cudaStream_t st) {
    if (a.n <= 0) return cudaSuccess;
    const int64_t nbatch = (a.n + 1) / 2;
    if (ts2_mc() && ts2_max_clusters[pm] > 0) {
        const int grid = 2 * (int)std::min<int64_t>((nbatch + 3) / 4, ts2_max_clusters[pm]);
        cudaLaunchAttribute attr;
        cudaLaunchConfig_t cfg = ts2_config(pm, grid, st, &attr);
        return cudaLaunchKernelEx(&cfg, ts2_kernel(pm, true), a);
    }
    const int grid = (int)std::min<int64_t>((nbatch + 1) / 2, 148);
    ts2_kernel(pm, false)<<<grid, ts2::kThreads, ts2::smem_bytes(pm), st>>>(a);
    return cudaGetLastError();
}

}  // namespace ci
