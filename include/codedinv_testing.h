/*
 * codedinv_testing.h -- test-only entry points of libcodedinv (not part of the serving ABI).
 *
 * They expose the tcgen05 building blocks of the convolution kernels so tests can pin the
 * descriptor encodings the implicit 3x3 convolution depends on, and measure the raw MMA
 * issue rate on the device.  Same conventions as codedinv.h (device pointers, async on
 * `stream`, synchronous host-side argument errors).
 */
#ifndef CODEDINV_TESTING_H_
#define CODEDINV_TESTING_H_

#include "codedinv.h"

#ifdef __cplusplus
extern "C" {
#endif

/* One UMMA GEMM D[128][N] (fp32) = sum over nk K=16 steps of A-rows x B^T on tcgen05:
 *   A [RA][KA] bf16 row-major (K contiguous), B [N][KB] bf16 row-major, D [128][N] fp32.
 *   mode 0: step j uses A channels [16j, 16j+16) of rows shift..shift+127 and B columns
 *           [16j, 16j+16)   (row-shifted start address, K-planes at LBO = RA*16 B);
 *   mode 1: KA = 8; step j uses A channels 0..7 of rows shift+2j+i (K-half 0) and
 *           shift+2j+1+i (K-half 1) against B columns [16j, 16j+16) (LBO = 16 B).
 *   mode 2 | (L << 8): the A planes concatenated as one column of 16-B rows (plane p row r =
 *           row p*RA + r); step j's K-half 0 = rows shift+j+i, K-half 1 = rows shift+j+L+i
 *           against B columns [16j, 16j+16) (LBO = L*16 B: the conv kernel's vertical tap
 *           pairs, L = Wp, and cross-plane pairs, L = plane rows - Wp - 1).
 * Requires 16 <= N <= 256, N % 16 == 0, KA % 8 == 0, KB % 16 == 0, shift + 127 + 2nk < RA
 * (mode 2: 1 <= L < 16384, shift + nk + L + 127 < RA * KA/8). */
CI_API ci_status_t ci_test_umma_gemm(const uint16_t* A, int32_t RA, int32_t KA, const uint16_t* B,
                                     int32_t N, int32_t KB, int32_t shift, int32_t mode, int32_t nk,
                                     float* D, ci_stream_t stream);

/* `nblocks` CTAs each issue `iters` back-to-back 128 x N x 16 bf16 MMAs from shared memory
 * (SS mode) and record the issue-to-completion SM cycles in cycles[nblocks] (int64).
 * Plain N runs the reference tight issue loop (1 MMA per iteration, 2 accumulators).
 * N's upper bits select a variant: bits 16..23 = number of accumulators cycled,
 * bits 24..31 = variant flags (1 packed accumulators, 2 LBO=16 A pairs, 4 spinning warps,
 * 8 moving B, 16 periodic commits). */
CI_API ci_status_t ci_test_umma_rate(int32_t N, int32_t iters, int32_t nblocks, int64_t* cycles,
                                     ci_stream_t stream);

/* Kernel accounting for bench.py.
 * ci_test_prof_enable(1) makes every fused tcgen05 stage launch record a CUDA event pair on
 * its own stream, together with the launch's algorithmic FLOPs (2 MACs per 3x3-conv product,
 * no padding); ci_test_prof_read() synchronises those events and returns, per stage index
 * (0..3), the summed device milliseconds, launch count and algorithmic FLOPs, then clears them.
 * ci_test_launch_count() returns the number of kernels this library has launched since the
 * last call with reset != 0 (all kernels: stage, permute, mean, decode, classify, drops). */
CI_API ci_status_t ci_test_prof_enable(int32_t enable);
CI_API ci_status_t ci_test_prof_read(double* ms, int64_t* launches, double* flops);
CI_API int64_t ci_test_launch_count(int32_t reset);

/* Host-only: the shared-memory / TMEM plan the fused stage kernel uses for one stage
 * (H x W state, c = half channels, m = hidden width; c < 0: a residual stage whose F acts on
 * all |c| state channels).  out16 = {Wp, G, Cp, Mp, MC, nch, Nc2,
 * T, I, Rtot, k1, k2, nslot, slot_bytes, smem_bytes, packed_bytes_per_block, nhd, sstate,
 * est_cycles_per_image_per_block, tmem_cols, hst, hc, has_specialised_kernel}  (23 entries). */
CI_API ci_status_t ci_test_plan(int32_t H, int32_t W, int32_t c, int32_t m, int32_t prec3, int64_t* out16);

/* The encode-mean kernel alone: m [B][d] = (sum_{i<k} h[b][i]) / k  (as inside ci_encode). */
CI_API ci_status_t ci_test_mean(int32_t k, int64_t B, int64_t d, const float* h, float* m,
                                ci_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* CODEDINV_TESTING_H_ */
