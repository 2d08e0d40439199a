// Test-only probes of the tcgen05 building blocks (include/codedinv_probe.h), built as their own
// library (libcodedinv_probe.so) so that none of this code ships in libcodedinv.so:
//  * ci_test_umma_gemm: one 128 x N x (16*nk) UMMA with the descriptor tricks the conv
//    kernel relies on (row-shifted start address; LBO = 16 B pairing adjacent rows; any
//    LBO, e.g. Wp rows for vertical tap pairs or across planes for the tri mode),
//    checked against a host reference by tests/test_gpu_umma.py;
//  * ci_test_umma_rate: back-to-back MMA issue rate per SM for a given N.
#include <stdarg.h>
#include <stdio.h>

#include "codedinv_probe.h"
#include "umma.cuh"

namespace ci {
using namespace umma;

static thread_local char g_probe_err[256] = "no error";
static void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_probe_err, sizeof(g_probe_err), fmt, ap);
    va_end(ap);
}
static ci_status_t cuda_status(cudaError_t e, const char* what) {
    set_error("CUDA error %d (%s) in %s", (int)e, cudaGetErrorString(e), what);
    return CI_ERR_CUDA;
}
#define CI_CUDA(call)                                              \
    do {                                                           \
        cudaError_t e_ = (call);                                   \
        if (e_ != cudaSuccess) return ::ci::cuda_status(e_, #call); \
    } while (0)
#define CI_CHECK_LAUNCH(what)                                      \
    do {                                                           \
        cudaError_t e_ = cudaGetLastError();                       \
        if (e_ != cudaSuccess) return ::ci::cuda_status(e_, what); \
    } while (0)

// A: [RA][KA] bf16 row-major in global; B: [N][KB] bf16 row-major.  SMEM planes of 8 channels:
// plane p holds rows 0..R-1 at 16-B stride (uniform, SBO = 128).
__global__ void __launch_bounds__(128) k_umma_gemm(const uint16_t* __restrict__ A, int RA, int KA,
                                                   const uint16_t* __restrict__ B, int N, int KB,
                                                   int shift, int mode, int nk, float* __restrict__ D) {
    const bool f16 = (mode >> 30) & 1;   // operands are fp16 (the f16x2 precision's instruction descriptor)
    mode &= ~(1 << 30);
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int pa = KA / 8, pb = KB / 8;
    uint8_t* sA = smem;
    uint8_t* sB = smem + (size_t)pa * RA * 16;
    // fill planes (generic proxy)
    for (int i = tid; i < RA * pa; i += 128) {
        int r = i / pa, p = i % pa;
        *reinterpret_cast<uint4*>(sA + ((size_t)p * RA + r) * 16) =
            *reinterpret_cast<const uint4*>(A + (size_t)r * KA + p * 8);
    }
    for (int i = tid; i < N * pb; i += 128) {
        int r = i / pb, p = i % pb;
        *reinterpret_cast<uint4*>(sB + ((size_t)p * N + r) * 16) =
            *reinterpret_cast<const uint4*>(B + (size_t)r * KB + p * 8);
    }
    fence_proxy_async();
    if (warp == 0) tmem_alloc(&tmem_base, 256);
    if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base;
    if (warp == 0 && elect_one()) {
        const uint32_t idesc = idesc_of(128, N, f16);
        for (int j = 0; j < nk; j++) {
            uint64_t ad, bd;
            if (mode == 0) {  // K-halves = planes 2j, 2j+1
                ad = smem_desc(smem_u32(sA) + (uint32_t)(2 * j * RA + shift) * 16, RA * 16, 128);
            } else if ((mode & 0xFF) == 1) {   // K-halves = rows r and r+1 of plane 0 (LBO = 16 B); step j moves 2 rows
                ad = smem_desc(smem_u32(sA) + (uint32_t)(shift + 2 * j) * 16, 16, 128);
            } else {   // mode 2: K-half 1 = LBO (mode >> 8) 16-B rows after K-half 0 (across planes); step j moves 1 row
                ad = smem_desc(smem_u32(sA) + (uint32_t)(shift + j) * 16, (uint32_t)(mode >> 8) * 16u, 128);
            }
            bd = smem_desc(smem_u32(sB) + (uint32_t)(2 * j * N) * 16, N * 16, 128);
            mma_bf16(tmem, ad, bd, idesc, j > 0);
        }
        commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    fence_after();
    for (int c = 0; c < N; c += 8) {
        float v[8];
        tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
        tmem_wait_ld();
        for (int q = 0; q < 8; q++) D[(size_t)(warp * 32 + (tid & 31)) * N + c + q] = v[q];
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 256);
}

// Issue-loop cost probe.  One elected thread issues `iters` k-steps of `ntile` MMAs each.
// variant bits: 1 = A/B start addresses carried across iterations (add + wrap),
// 2 = mbarrier try_wait on an already-completed barrier every k-step,
// 4 = tcgen05.commit every k-step, 8 = B advances per k-step, 16 = fully static addresses
__global__ void __launch_bounds__(128) k_umma_rate(int N, int iters, int ntile, int variant,
                                                   long long* __restrict__ cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar, slot_bar, done_bar, slot_bar2;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int ARows = 1088;
    uint8_t* sA = smem;
    uint8_t* sB = smem + 3 * ARows * 16;
    for (int i = tid; i < (3 * ARows * 16 + 65536) / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    fence_proxy_async();
    if (warp == 0) tmem_alloc(&tmem_base, 512);
    if (tid == 0) { mbar_init(&bar, 1); mbar_init(&slot_bar, 1); mbar_init(&done_bar, 1); mbar_init(&slot_bar2, 1); fence_mbar_init(); }
    fence_before();
    __syncthreads();
    if (tid == 0) mbar_arrive(&done_bar);   // phase 0 completed
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base;
    if (warp == 0) {
        const uint32_t idesc = idesc_bf16(128, N);
        const uint64_t a_desc0 = smem_desc(smem_u32(sA), ARows * 16, 128);
        const uint64_t b_desc0 = smem_desc(smem_u32(sB), N * 16, 128);
        const uint32_t dstride = 512u / (uint32_t)ntile;
        if (elect_one()) {
            long long t0 = clock64();
            uint64_t ac = a_desc0, bc = b_desc0;
            if (variant & 32) {   // v1-style loop. 64: A LBO 4320 B; 128: all MMAs into D=0;
                                  // 256: B advances per MMA; 512: A alternates tiles (+2048 B)
                const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
                const uint32_t albo = (variant & 64) ? 4320u : 192u * 16u;
                for (int j = 0; j < iters; j++) {
                    uint32_t aadr = a0 + (uint32_t)(j & 63) * 16 + ((variant & 512) ? (uint32_t)(j & 1) * 2048u : 0u);
                    uint64_t ad = smem_desc(aadr, albo, 128);
                    uint64_t bd = smem_desc(b0 + ((variant & 256) ? (uint32_t)(j & 7) * (uint32_t)N * 32u : 0u), (uint32_t)N * 16, 128);
                    mma_bf16(tmem + (uint32_t)((j & 1) * ((variant & 128) ? 0 : 256)), ad, bd, idesc, 1);
                    if ((j & 7) == 7) {
                        if (variant & 8192) { mbar_wait(&done_bar, 0); }
                        if (variant & 16384) { fence_after(); }
                        if (variant & 32768) { commit(&slot_bar); }
                    }
                }
                iters = 0;
            }
            for (int j = 0; j < iters; j++) {
                uint64_t ad, bd;
                if (variant & 16) { ad = a_desc0; bd = b_desc0; }
                else if (variant & 1) { ad = ac; bd = bc; }
                else { ad = a_desc0 + (uint64_t)((j * 7) & 63); bd = b_desc0 + ((variant & 8) ? (uint64_t)((j & 7) * N * 2) : 0); }
                for (int t = 0; t < ntile; t++)
                    mma_bf16(tmem + (uint32_t)t * dstride, ad + (uint64_t)(t * 128), bd, idesc, 1);
                if (variant & 2) mbar_wait(&done_bar, 0);
                if (variant & 4) commit(&slot_bar);
                if (variant & 1) {
                    ac += 7; if ((uint32_t)ac - (uint32_t)a_desc0 >= 64u) ac -= 64;
                    if (variant & 8) { bc += (uint64_t)N * 2; if ((uint32_t)bc - (uint32_t)b_desc0 >= (uint32_t)(16 * N)) bc = b_desc0; }
                }
            }
            commit(&bar);
            mbar_wait(&bar, 0);
            long long t1 = clock64();
            cycles[blockIdx.x] = t1 - t0;
            mbar_arrive(&slot_bar2);
        }
        __syncwarp();
    } else if (variant & 2048) {          // warps 1..3 spin on try_wait during the MMAs
        if ((variant & 4096) == 0 || (tid & 31) == 0) mbar_wait(&slot_bar2, 0);
        __syncwarp();
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// The reference tight issue loop (profiles/r01_umma_probe.md): one elected thread, one MMA per
// iteration, A start moved by (j & 63) rows, accumulators alternating 0 / 256.
__global__ void __launch_bounds__(128) k_umma_rate_v1(int N, int iters, long long* __restrict__ cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (2 * 192 + 2 * 256) * 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    fence_proxy_async();
    if (warp == 0) tmem_alloc(&tmem_base, 512);
    if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base;
    if (warp == 0 && elect_one()) {
        const uint32_t idesc = idesc_bf16(128, N);
        const uint32_t a0 = smem_u32(smem), b0 = a0 + 2 * 192 * 16;
        long long t0 = clock64();
        for (int j = 0; j < iters; j++) {
            uint64_t ad = smem_desc(a0 + (uint32_t)(j & 63) * 16, 192 * 16, 128);
            uint64_t bd = smem_desc(b0, 256 * 16, 128);
            mma_bf16(tmem + (uint32_t)((j & 1) * 256), ad, bd, idesc, 1);
        }
        commit(&bar);
        mbar_wait(&bar, 0);
        cycles[blockIdx.x] = clock64() - t0;
    }
    __syncwarp();
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// TMEM -> register read bandwidth: nw warps (warp w reads lane quarter w % 4), each loading
// 32x32b.x16 (2 KB per warp-load) `iters` times; batch = loads in flight before tcgen05.wait::ld.
__global__ void __launch_bounds__(512) k_tmem_ld_rate(int iters, int batch, long long* __restrict__ cycles,
                                                      float* __restrict__ sink) {
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) tmem_alloc(&tmem_base, 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base + ((uint32_t)((warp & 3) * 32) << 16);
    float acc = 0.f;
    long long t0 = clock64();
    for (int j = 0; j < iters; j += batch) {
        float v[4][16];
#pragma unroll
        for (int q = 0; q < 4; q++)
            if (q < batch) tmem_ld16(tmem + (uint32_t)(((j + q) * 16 + warp * 64) & 511), v[q]);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 4; q++)
            if (q < batch)
#pragma unroll
                for (int e = 0; e < 16; e++) acc += v[q][e];
    }
    __syncthreads();
    if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
    if (acc == 12345.f) sink[tid] = acc;
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem_base, 512);
}


// TS-mode (A in tensor memory) GEMM: thread r of 128 writes row r of A (K = 16 nk 16-bit values,
// two per 32-bit column, even k in the low half) into TMEM lane r, columns acol + 8j + (k%16)/2;
// one thread then issues nk MMAs D = sum_j A_j B_j^T with B from shared memory (one plane per 8
// K, LBO = N*16 B).  mode bit 30: fp16 operands.
__global__ void __launch_bounds__(128) k_umma_ts_gemm(const uint32_t* __restrict__ A, const uint16_t* __restrict__ B,
                                                      int N, int nk, int acol, int f16, float* __restrict__ D) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int KB = 16 * nk, pb = KB / 8;
    uint8_t* sB = smem;
    for (int i = tid; i < N * pb; i += 128) {
        int r = i / pb, p = i % pb;
        *reinterpret_cast<uint4*>(sB + ((size_t)p * N + r) * 16) = *reinterpret_cast<const uint4*>(B + (size_t)r * KB + p * 8);
    }
    fence_proxy_async();
    if (warp == 0) tmem_alloc(&tmem_base, 512);
    if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base;
    const uint32_t lane_addr = (uint32_t)(warp * 32) << 16;
    for (int j = 0; j < nk; j++) {
        float v[8];
        for (int i = 0; i < 8; i++) v[i] = __uint_as_float(A[(size_t)tid * (8 * nk) + 8 * j + i]);
        tmem_st8(tmem + lane_addr + (uint32_t)(acol + 8 * j), v);
    }
    tmem_wait_st();
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == 0 && elect_one()) {
        const uint32_t idesc = idesc_of(128, N, f16 != 0);
        for (int j = 0; j < nk; j++) {
            const uint64_t bd = smem_desc(smem_u32(sB) + (uint32_t)(2 * j * N) * 16, N * 16, 128);
            mma_ts(tmem, tmem + (uint32_t)(acol + 8 * j), bd, idesc, j > 0);
        }
        commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    fence_after();
    for (int c = 0; c < N; c += 8) {
        float v[8];
        tmem_ld8(tmem + lane_addr + c, v);
        tmem_wait_ld();
        for (int q = 0; q < 8; q++) D[(size_t)tid * N + c + q] = v[q];
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// TS-mode issue rate: one elected thread issues `iters` back-to-back 128 x N x 16 MMAs with A read
// from TMEM (columns 320 + 8 (j % 8)), D at column 0, B fixed in shared memory.
__global__ void __launch_bounds__(128) k_umma_ts_rate(int N, int iters, long long* __restrict__ cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 256 * 2 * 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    fence_proxy_async();
    if (warp == 0) tmem_alloc(&tmem_base, 512);
    if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base;
    {
        float z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int j = 0; j < 8; j++) tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + 320u + (uint32_t)(8 * j), z);
        tmem_wait_st();
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == 0 && elect_one()) {
        const uint32_t idesc = idesc_f16(128, N);
        const uint64_t bd = smem_desc(smem_u32(smem), N * 16, 128);
        long long t0 = clock64();
        for (int j = 0; j < iters; j++) mma_ts(tmem, tmem + 320u + (uint32_t)((j & 7) * 8), bd, idesc, 1);
        commit(&bar);
        mbar_wait(&bar, 0);
        cycles[blockIdx.x] = clock64() - t0;
    }
    __syncwarp();
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

}  // namespace ci

using namespace ci;

extern "C" {

const char* ci_probe_last_error(void) { return ci::g_probe_err; }

ci_status_t ci_test_umma_gemm(const uint16_t* A, int32_t RA, int32_t KA, const uint16_t* B, int32_t N,
                              int32_t KB, int32_t shift, int32_t mode, int32_t nk, float* D,
                              ci_stream_t stream) {
    const int lbo_rows = (mode & ~(1 << 30)) >> 8;
    if (N < 16 || N > 256 || N % 16 || KA % 8 || KB % 16 || nk < 1 || shift < 0 || (mode & 0xFF) > 2 ||
        ((mode & 0xFF) == 2 && (lbo_rows < 1 || lbo_rows >= 16384 || shift + nk + lbo_rows + 127 >= RA * (KA / 8)))) {
        set_error("bad probe shape");
        return CI_ERR_INVALID_ARG;
    }
    size_t smem = (size_t)(KA / 8) * RA * 16 + (size_t)(KB / 8) * N * 16;
    CI_CUDA(cudaFuncSetAttribute(k_umma_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_umma_gemm<<<1, 128, smem, (cudaStream_t)stream>>>(A, RA, KA, B, N, KB, shift, mode, nk, D);
    CI_CHECK_LAUNCH("k_umma_gemm");
    return CI_OK;
}

ci_status_t ci_test_umma_rate(int32_t N, int32_t iters, int32_t nblocks, int64_t* cycles,
                              ci_stream_t stream) {
    int32_t ntile = (N >> 16) & 0xFF, variant = N >> 24;
    N &= 0xFFFF;
    if (variant == 15) {   // TMEM read bandwidth: N = warps (4..16), ntile = loads per wait (1..4)
        const int nw = N, batch = ntile < 1 ? 1 : (ntile > 4 ? 4 : ntile);
        if (nw < 1 || nw > 16 || iters < batch) { set_error("bad probe shape"); return CI_ERR_INVALID_ARG; }
        static float* sink = nullptr;
        if (!sink) CI_CUDA(cudaMalloc(&sink, 512 * sizeof(float)));
        k_tmem_ld_rate<<<nblocks, nw * 32, 0, (cudaStream_t)stream>>>(iters, batch, (long long*)cycles, sink);
        CI_CHECK_LAUNCH("k_tmem_ld_rate");
        return CI_OK;
    }
    if (variant == 0 && ntile == 0) {   // the reference tight loop
        if (N < 16 || N > 256 || N % 16 || iters < 1 || nblocks < 1) { set_error("bad probe shape"); return CI_ERR_INVALID_ARG; }
        size_t sm = (2 * 192 + 2 * 256) * 16;
        CI_CUDA(cudaFuncSetAttribute(k_umma_rate_v1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k_umma_rate_v1<<<nblocks, 128, sm, (cudaStream_t)stream>>>(N, iters, (long long*)cycles);
        CI_CHECK_LAUNCH("k_umma_rate_v1");
        return CI_OK;
    }
    if (ntile < 1) ntile = 2;
    if (N < 16 || N > 256 || N % 16 || iters < 1 || nblocks < 1 || ntile * N > 512) {
        set_error("bad probe shape");
        return CI_ERR_INVALID_ARG;
    }
    size_t smem = 3 * 1088 * 16 + 65536;
    CI_CUDA(cudaFuncSetAttribute(k_umma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_umma_rate<<<nblocks, 128, smem, (cudaStream_t)stream>>>(N, iters, ntile, variant, (long long*)cycles);
    CI_CHECK_LAUNCH("k_umma_rate");
    return CI_OK;
}

ci_status_t ci_test_umma_ts_gemm(const uint32_t* A, const uint16_t* B, int32_t N, int32_t nk, int32_t acol,
                                 int32_t f16, float* D, ci_stream_t stream) {
    if (N < 16 || N > 256 || N % 16 || nk < 1 || acol < N || acol + 8 * nk > 512) {
        set_error("bad probe shape");
        return CI_ERR_INVALID_ARG;
    }
    size_t smem = (size_t)2 * nk * N * 16;
    CI_CUDA(cudaFuncSetAttribute(k_umma_ts_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_umma_ts_gemm<<<1, 128, smem, (cudaStream_t)stream>>>(A, B, N, nk, acol, f16, D);
    CI_CHECK_LAUNCH("k_umma_ts_gemm");
    return CI_OK;
}

ci_status_t ci_test_umma_ts_rate(int32_t N, int32_t iters, int32_t nblocks, int64_t* cycles, ci_stream_t stream) {
    if (N < 16 || N > 256 || N % 16 || iters < 1 || nblocks < 1) { set_error("bad probe shape"); return CI_ERR_INVALID_ARG; }
    size_t sm = 256 * 2 * 16;
    CI_CUDA(cudaFuncSetAttribute(k_umma_ts_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_umma_ts_rate<<<nblocks, 128, sm, (cudaStream_t)stream>>>(N, iters, (long long*)cycles);
    CI_CHECK_LAUNCH("k_umma_ts_rate");
    return CI_OK;
}

}  // extern "C"
