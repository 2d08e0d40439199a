/*
 * codedinv_testing.h -- instrumentation entry points of libcodedinv (not part of the serving
 * ABI): kernel accounting that bench.py reads and the stage planner's decisions.  Same
 * conventions as codedinv.h.  The tcgen05 descriptor / issue-rate probes live in their own
 * library (include/codedinv_probe.h, libcodedinv_probe.so).
 */
#ifndef CODEDINV_TESTING_H_
#define CODEDINV_TESTING_H_

#include "codedinv.h"

#ifdef __cplusplus
extern "C" {
#endif

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
 * all |c| state channels; pm = product precision: 0 bf16 (CI_PREC_BF16), 1 f16x2 (CI_PREC_F16X2),
 * 2 f16x3 (CI_PREC_FP32)).  out16 = {Wp, G, Cp, Mp, MC, nch, Nc2,
 * T, I, Rtot, k1, k2, nslot, slot_bytes, smem_bytes, packed_bytes_per_block, nhd, sstate,
 * est_cycles_per_image_per_block, tmem_cols, hst, hc, has_specialised_kernel, ts (1: k_stage_ts,
 * 2: k_stage_ts2), nopad (1: no pad column, 2: image-row-interleaved raster)}  (25 entries). */
CI_API ci_status_t ci_test_plan(int32_t H, int32_t W, int32_t c, int32_t m, int32_t pm, int64_t* out16);

/* The encode-mean kernel alone: m [B][d] = (sum_{i<k} h[b][i]) / k  (as inside ci_encode). */
CI_API ci_status_t ci_test_mean(int32_t k, int64_t B, int64_t d, const float* h, float* m,
                                ci_stream_t stream);

/* Host-only: the node-local rendezvous ci_comm_create uses (POSIX shared memory named by `id`):
 * rank `rank` of `nranks` publishes `bytes` (<= 64) of `payload` and receives every rank's,
 * out = nranks x 64 bytes (slot q at q * 64).  CI_ERR_COMM after 60 s without all ranks. */
CI_API ci_status_t ci_test_rendezvous(const uint8_t id[CI_COMM_ID_BYTES], int32_t nranks, int32_t rank,
                                      const uint8_t* payload, int32_t bytes, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif /* CODEDINV_TESTING_H_ */
