/*
 * codedinv_probe.h -- test-only probes of the tcgen05 building blocks, exported by
 * libcodedinv_probe.so (a separate library: nothing here ships in libcodedinv.so).
 *
 * They let tests pin the shared-memory descriptor encodings the implicit 3x3 convolution of
 * the stage kernel depends on, and measure the raw MMA issue rate on the device.  Same
 * conventions as codedinv.h (device pointers, async on `stream`, synchronous host-side argument
 * errors); the message of the last error is ci_probe_last_error().
 */
#ifndef CODEDINV_PROBE_H_
#define CODEDINV_PROBE_H_

#include "codedinv.h"

#ifdef __cplusplus
extern "C" {
#endif

CI_API const char* ci_probe_last_error(void);

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
 *   mode | (1 << 30): A and B hold fp16 bits instead of bf16 (instruction descriptor a/b_format
 *           = F16, the operand type of CI_PREC_FP32's f16x2 products).
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

/* TS-mode UMMA GEMM (A in tensor memory): D[128][N] (fp32) = sum over nk K=16 steps of
 * A[:, 16j:16j+16] x B[:, 16j:16j+16]^T.  A [128][8 nk] uint32 words, row r = TMEM lane r,
 * word 8j+i = K elements 16j+2i (low half) and 16j+2i+1 (high half), stored at TMEM columns
 * acol + 8j + i; B [N][16 nk] 16-bit row-major in shared memory; f16 != 0: fp16 operands, else
 * bf16.  Requires 16 <= N <= 256, N % 16 == 0, N <= acol, acol + 8 nk <= 512. */
CI_API ci_status_t ci_test_umma_ts_gemm(const uint32_t* A, const uint16_t* B, int32_t N, int32_t nk,
                                        int32_t acol, int32_t f16, float* D, ci_stream_t stream);

/* TS-mode issue rate: `nblocks` CTAs each issue `iters` back-to-back 128 x N x 16 fp16 MMAs with
 * A in tensor memory; cycles[nblocks] (int64) = issue-to-completion SM cycles. */
CI_API ci_status_t ci_test_umma_ts_rate(int32_t N, int32_t iters, int32_t nblocks, int64_t* cycles,
                                        ci_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* CODEDINV_PROBE_H_ */
