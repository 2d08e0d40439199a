/*
 * codedinv.h -- C ABI of the B200-native Coded-InvNet hot path (arXiv 2106.06445).
 *
 * The library computes coded inference f = g o h over groups of k queries with one
 * parity worker (n = k + 1, c_{1,j} = 1/k):
 *   (1) h on the k main queries
 *   (2) exact encode x_p = h^-1((1/k) sum_i h(x_i))
 *   (3) h on the parity query                         PAPER.md:205 (every worker runs f, :330)
 *   (4) decode h(x_j) = k h(x_p) - sum_{i!=j} h(x_i)
 *   (5) linear heads g_t + argmax
 *
 * Conventions (all entry points):
 *   - Tensor arguments are DEVICE pointers (except the *_host entry point), owned by the
 *     caller, contiguous, fp32 (int32 for drop / labels), 16-byte aligned.
 *   - Layouts: images NCHW [n][in_c][in_h][in_w]; features h [n][d] are the NCHW flatten of
 *     the final state (d = C*H*W, h is dimension preserving);
 *     groups are [B][k][...]: query q belongs to group q / k, slot q % k.
 *   - Every call is asynchronous on `stream` (no hidden device sync) except ci_model_create,
 *     ci_model_destroy, ci_check and ci_serve_group_host.  Hot calls do not allocate: the
 *     caller passes a workspace of at least ci_workspace_size() bytes.  One workspace per
 *     concurrent stream.
 *   - Host-checkable errors (NULL/misaligned pointers, k < 1, B < 1, n < 0, head out of range,
 *     workspace too small, dims mismatch) return synchronously with nothing enqueued.
 *     Out-of-range drop indices found on the device are clamped to "no drop", counted in a
 *     flag inside the workspace, and reported by ci_check() as CI_ERR_INVALID_ARG.
 *   - CUDA launch failures map to CI_ERR_CUDA; ci_last_error() returns the thread-local text
 *     of the last non-OK status.
 *   - ci_model_t is immutable after create and safe to use from several streams.
 *   - Determinism: results are bitwise reproducible for the same (device, precision, n);
 *     F's accumulation order per output does not depend on tile position, so ci_inverse_h
 *     undoes ci_forward_h up to fp32 rounding of the coupling adds.
 */
#ifndef CODEDINV_H_
#define CODEDINV_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CI_API __attribute__((visibility("default")))
#else
#define CI_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

struct CUstream_st;
typedef struct CUstream_st* ci_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef struct ci_model ci_model_t; /* opaque: packed device weights for h and heads */

typedef enum {
    CI_OK = 0,
    CI_ERR_INVALID_ARG = 1,
    CI_ERR_INVALID_SHAPE = 2, /* SPEC.md:40 InvalidShape */
    CI_ERR_DIM_MISMATCH = 3,  /* SPEC.md:115 DimensionMismatch */
    CI_ERR_UNSUPPORTED = 4,   /* arch/precision combination not built */
    CI_ERR_WORKSPACE = 5,     /* workspace NULL or smaller than ci_workspace_size() */
    CI_ERR_CUDA = 6,
    CI_ERR_UNDECODABLE = 7,   /* SPEC.md:283 Undecodable: a group had fewer than k results or a
                                 singular k-subset (general codes); reported by ci_check */
    CI_ERR_COMM = 8           /* communicator bootstrap / peer mapping failed (SURVEY's CI_ERR_NCCL:
                                 the exchange is this library's own peer-memory kernels) */
} ci_status_t;

typedef enum {
    /* The parity mode (<= 1e-3 vs the f64 oracle, north star; "PyTorch", fp32):
     * fp32 state and TMEM accumulators; every conv operand split into fp16 hi + lo (22
     * significant bits each), 3 tcgen05 MMAs per product ("f16x3": hi(x)W_hi + lo(x)W_hi +
     * hi(x)W_lo; the dropped lo*lo term is 2^-22 relative). */
    CI_PREC_FP32 = 0,
    /* fp32 state, bf16 operands, 1 tcgen05 MMA per product, fp32 TMEM accumulators; error
     * bound and label agreement reported, not promised <= 1e-3. */
    CI_PREC_BF16 = 1,
    /* fp32 state, activations split into fp16 hi + lo, weights rounded once to fp16, 2 MMAs
     * per product ("f16x2").  Weight rounding is one fixed perturbation of h shared by every
     * query, so coupling inverses and the decode stay exact for it (activation rounding would
     * be per-query noise the decode amplifies k-fold): features ~2e-4 vs the
     * oracle; reported like bf16, not promised <= 1e-3 (ill-conditioned logit vectors of a
     * 2-class head exceed it). */
    CI_PREC_F16X2 = 2
} ci_precision_t;

typedef enum {
    CI_ENC_EXACT = 0,   /* x_p = h^-1((1/k) sum_i h(x_i))  (ideal encoder)       */
    CI_ENC_LEARNED = 1  /* x_p = Enc(x_1..x_k), the light learned encoder */
} ci_encode_mode_t;

typedef struct {
    int32_t squeeze_before; /* 1: psi (space-to-depth r=2) before this stage's blocks */
    int32_t n_blocks;       /* blocks in the stage */
    int32_t mid_channels;   /* m: F = conv3x3(c->m) -> act -> conv3x3(m->c); c = C/2 (coupling)
                               or C (residual) */
} ci_stage_t;

typedef struct {
    int32_t in_c, in_h, in_w; /* input image shape */
    int32_t n_stages;         /* 1..4 */
    ci_stage_t stage[4];
    int32_t act;              /* 0 = ReLU, 1 = ELU, 2 = identity */
    int32_t first_orientation;/* 0: block 0 of each stage does s_B += F(s_A); 1: s_A += F(s_B) */
    int32_t n_heads;          /* 0..4 linear heads g_t */
    int32_t head_classes[4];
    /* light learned encoder (0 = none): e_i = ReLU(E1 x_i) (in_c -> enc_c1), mean over the k
     * inputs, psi, ReLU(E2) (4 enc_c1 -> enc_mid), ReLU(E3) (enc_mid -> 4 enc_c1), psi^-1,
     * + skip(mean), E4 (enc_c1 -> in_c); all conv3x3 with bias */
    int32_t enc_c1, enc_mid;
    /* block_kind 0: additive coupling on half the state (i-RevNet).
     * block_kind 1: i-ResNet residual block y = x + F(x) on the whole state (PAPER.md:169-170,
     *   393): the weights must make Lip(F) < 1 (spectral normalisation); h^-1
     *   inverts each block by fp_iters >= 1 fixed-point updates x <- y - F(x) from x_0 = y
     *   ("exponential convergence rate via fixed-point iteration", 408, 441).
     *   first_orientation is ignored. */
    int32_t block_kind;
    int32_t fp_iters;
} ci_arch_t;

/* Thread-local description of the last non-OK status (never NULL). */
CI_API const char* ci_last_error(void);

/* Build a model on `device` from the canonical flat fp32 parameter vector (host memory,
 * copied; the caller keeps ownership):
 *   per stage s, block t: W1[m][c][3][3], b1[m], W2[c][m][3][3], b2[c]
 *   then per head t:      W[classes][d], b[classes]
 * n_params must equal the count implied by `arch` (else CI_ERR_DIM_MISMATCH). */
CI_API ci_status_t ci_model_create(const ci_arch_t* arch, const float* host_params, size_t n_params,
                            ci_precision_t precision, int device, ci_model_t** out);
CI_API void ci_model_destroy(ci_model_t* model);

CI_API int64_t ci_feature_dim(const ci_model_t* model); /* d; -1 if model == NULL */

/* Bytes of workspace needed by any call with up to B groups of k (or n = B * k images; a plain
 * ci_forward_h / ci_inverse_h on n images needs no more than ci_workspace_size(model, 1, n)). */
CI_API ci_status_t ci_workspace_size(const ci_model_t* model, int32_t k, int64_t B, size_t* bytes);

/* Synchronise `stream` and report device-side flags recorded in `ws`, then clear them:
 * CI_ERR_UNDECODABLE if a general-code group could not be decoded, else CI_ERR_INVALID_ARG if a
 * drop index was out of range. */
CI_API ci_status_t ci_check(const ci_model_t* model, void* ws, size_t ws_bytes, ci_stream_t stream);

/* h on n images: x [n][in_c][in_h][in_w] -> h [n][d].  x and h must not overlap.
 * (SPEC.md:111-118 `forward`) */
CI_API ci_status_t ci_forward_h(const ci_model_t* model, const float* x, float* h, int64_t n, void* ws,
                         size_t ws_bytes, ci_stream_t stream);

/* Exact inverse by reverse coupling: h [n][d] -> x [n][in_c][in_h][in_w]
 * (blocks in reverse order, s_B -= F(s_A) / s_A -= F(s_B), psi^-1; SPEC.md:120-128 `inverse`;
 * closed form, iteration count 0). */
CI_API ci_status_t ci_inverse_h(const ci_model_t* model, const float* h, float* x, int64_t n, void* ws,
                         size_t ws_bytes, ci_stream_t stream);

/* Encode B groups into their parity queries x_parity [B][in_c][in_h][in_w]:
 *   CI_ENC_EXACT:   h [B][k][d] -> m_b = (1/k) sum_{i<k} h[b][i] (fp32 sum in ascending i, then
 *                   /k), x_parity[b] = h^-1(m_b); mean_out [B][d] or NULL; x unused (may be NULL).
 *                   (PAPER.md:125-127 Enc(x1,x2) = f^-1((f(x1)+f(x2))/2); :241 c_{1,j} = 1/k)
 *   CI_ENC_LEARNED: x [B][k][in_c][in_h][in_w] -> x_parity = Enc(x_b1..x_bk) (model must have an
 *                   encoder, else CI_ERR_UNSUPPORTED); h and mean_out unused (may be NULL).
 *                   (PAPER.md:143-152 approximate encoder; weight-shared first layer + average,
 *                   PAPER.md:411) */
CI_API ci_status_t ci_encode(const ci_model_t* model, ci_encode_mode_t mode, int32_t k, int64_t B,
                      const float* x, const float* h, float* x_parity, float* mean_out, void* ws,
                      size_t ws_bytes, ci_stream_t stream);

/* In-place decode of B groups: for each b with j = drop[b] in [0,k):
 *   h[b][j] = k * h_parity[b] - sum_{i != j, ascending} h[b][i]
 * drop[b] = -1 leaves group b untouched; other values are flagged (see ci_check) and ignored.
 * h [B][k][d], h_parity [B][d], drop [B] int32 (float4 path when d % 4 == 0).
 * (App. C: one scalar-vector multiply, k-1 subtractions) */
CI_API ci_status_t ci_decode(int32_t k, int64_t B, int64_t d, float* h, const float* h_parity,
                      const int32_t* drop, void* ws, size_t ws_bytes, ci_stream_t stream);

/* Linear head t on n feature rows: logits [n][C_t] = z W_t^T + b_t (fp32),
 * labels [n] = smallest index attaining the max (or NULL). */
CI_API ci_status_t ci_classify(const ci_model_t* model, int32_t head, const float* z, int64_t n,
                        float* logits, int32_t* labels, ci_stream_t stream);

/* ---- Communicator: the paper's worker partition across processes (config C5) -------------
 * One process per worker (Fig. 2, 665-668: one worker per instance): ranks
 * 0..k-1 are the main workers (slot r of every group), rank k is the parity worker, which also
 * hosts the encoder.  Every rank owns a symmetric window of device
 * memory (its published features + two epoch counters) that all ranks map (CUDA IPC; NVLink
 * peer loads between GPUs, plain loads when several ranks share a GPU).  The exchange steps run
 * as fused compute + collective kernels over that peer memory:
 *   X2 exact encode: the parity rank reads the k mains' h(x_i) and forms their mean
 *   X4 decode      : rank p reads every rank's features for its 1/(k+1) share of the groups
 *                    and forms k h(x_p) - sum_{i != j} h(x_i)
 * Bootstrap: rank 0 calls ci_comm_unique_id and the caller broadcasts the bytes (e.g. with
 * torch.distributed); every rank then calls ci_comm_create with the same id, nranks, max_B and
 * d (a host rendezvous through POSIX shared memory on this node; returns CI_ERR_COMM if a rank
 * does not arrive within 120 s).  Serve calls on a communicator are collective: every rank
 * issues the same sequence of ci_serve_group calls (same k, B), one stream per communicator.
 * ci_comm_destroy is collective too (call it after all ranks finished serving). */
#define CI_COMM_ID_BYTES 128
typedef struct ci_comm ci_comm_t;
typedef enum {
    CI_SHARD_GROUPS = 0, /* data parallel: each rank serves its own groups; no exchange */
    CI_SHARD_WORKERS = 1 /* the paper's partition: one worker (slot) per rank, nranks = k + 1 */
} ci_layout_t;
CI_API ci_status_t ci_comm_unique_id(uint8_t out[CI_COMM_ID_BYTES]);
/* max_B: most groups per serve call; d: feature dim (multiple of 4).  Window = 256 B + max_B*d*4. */
CI_API ci_status_t ci_comm_create(const uint8_t id[CI_COMM_ID_BYTES], int32_t nranks, int32_t rank,
                                  ci_layout_t layout, int64_t max_B, int64_t d, int device, ci_comm_t** out);
CI_API void ci_comm_destroy(ci_comm_t* comm);

/* The whole coded path for B groups (steps 1-5 above), with the parity query from `mode`
 * (CI_ENC_LEARNED skips h^-1 and runs the learned encoder on x).
 *
 * comm == NULL, or a CI_SHARD_GROUPS communicator (nothing is exchanged: groups are independent
 * units), serves this process's B groups on one GPU:
 *   x [B][k][in_c][in_h][in_w], drop [B]
 *   h_out [B][k][d]     : h(x), with slot drop[b] replaced by its decoded estimate
 *   h_parity [B][d]     : h(x_p)
 *   x_parity [B][in_c][in_h][in_w] or NULL : the encoded query x_p
 *   logits [n_heads][B][k][C_t] (heads packed one after another), labels [n_heads][B][k]
 *   (either may be NULL to skip the heads)
 *
 * A CI_SHARD_WORKERS communicator (nranks == k + 1, B <= max_B, d == the model's d) runs this
 * rank's worker of the partition; with Bp = ceil(B / (k+1)) and this rank's groups
 * G = [rank*Bp, min(B, (rank+1)*Bp)):
 *   x        main rank r: [B][in_c][in_h][in_w] = slot r of every group;  parity rank: the k
 *            slots [B][k][in_c][in_h][in_w] in CI_ENC_LEARNED (X3: the front end hands the
 *            encoder its inputs), unused (may be NULL) in CI_ENC_EXACT;
 *   drop     [B], identical on every rank;
 *   h_out    [B][d]: this worker's result (main: h(x_r); parity: h(x_p));
 *   h_parity [Bp][d]: the decoded features of the lost slot of groups G (rows of groups with
 *            drop = -1 are zero);
 *   x_parity [B][in_c][in_h][in_w] or NULL: x_p (parity rank only; ignored elsewhere);
 *   logits   [n_heads][B + Bp][C_t], labels [n_heads][B + Bp]: rows 0..B-1 = the heads on h_out
 *            (main ranks; the parity rank leaves them unwritten), rows B.. = on the decoded rows.
 * Drops are simulated by masking: the dropped worker still computes (PAPER.md:669 injects a
 * delay instead; see ci_serve_first_k for latency). */
CI_API ci_status_t ci_serve_group(const ci_model_t* model, ci_encode_mode_t mode, int32_t k, int64_t B,
                           const float* x, const int32_t* drop, float* h_out, float* h_parity,
                           float* x_parity, float* logits, int32_t* labels, ci_comm_t* comm, void* ws,
                           size_t ws_bytes, ci_stream_t stream);

/* Same as ci_serve_group with HOST buffers (x, drop in; h_out, h_parity, logits, labels out;
 * any output may be NULL).  Stages inputs into the workspace (which must be sized by
 * ci_workspace_size_host), runs the path, copies outputs back and synchronises `stream`.
 * Host buffers should be pinned for full PCIe bandwidth. */
CI_API ci_status_t ci_workspace_size_host(const ci_model_t* model, int32_t k, int64_t B, size_t* bytes);
CI_API ci_status_t ci_serve_group_host(const ci_model_t* model, ci_encode_mode_t mode, int32_t k,
                                int64_t B, const float* x_host, const int32_t* drop_host,
                                float* h_out_host, float* h_parity_host, float* logits_host,
                                int32_t* labels_host, void* ws, size_t ws_bytes,
                                ci_stream_t stream);

/* Same as ci_serve_group_host without the final synchronisation: the whole chunked
 * H2D -> compute -> D2H pipeline is enqueued and the call returns; `stream` completes when the
 * outputs are in the host buffers.  Until then the host buffers must stay alive and unmodified
 * and the workspace must not be reused.  Calls with distinct workspaces (and streams) may be in
 * flight together: their copies and compute overlap. */
CI_API ci_status_t ci_serve_group_host_async(const ci_model_t* model, ci_encode_mode_t mode, int32_t k,
                                             int64_t B, const float* x_host, const int32_t* drop_host,
                                             float* h_out_host, float* h_parity_host, float* logits_host,
                                             int32_t* labels_host, void* ws, size_t ws_bytes,
                                             ci_stream_t stream);

/* Perturbed exact encode ("f(x_{k+1}) = sum_j c_j f(x_j) + eps",
 * SPEC.md:192-200): x_parity = h^-1(mean_i h_i + eps) with a caller-supplied perturbation
 * eps [B][d] (DEVICE fp32; e.g. i.i.d. N(0, sigma^2) drawn by the caller), modelling an
 * approximate encoder.  Decoding such a parity amplifies eps by k (f^(x_a) = f(x_a) + k eps).
 * eps = all zeros gives exactly ci_encode(CI_ENC_EXACT).  Same workspace as ci_encode. */
CI_API ci_status_t ci_encode_perturbed(const ci_model_t* model, int32_t k, int64_t B, const float* h,
                                       const float* eps, float* x_parity, float* mean_out, void* ws,
                                       size_t ws_bytes, ci_stream_t stream);

/* Online decoding for n = k + 1 (App. C).  Results reach the
 * decoder one task at a time; each call applies one "wave" of at most one completion event
 * per group:
 *   est   [B][k][d] DEVICE fp32 best-effort estimates f^(x_i) (zero before the first event);
 *   state [B]       DEVICE uint64 (zero initially): bits 0..k = tasks received, bits 32..32+k-1
 *                   = estimates finalised;
 *   task  [B]       DEVICE int32: the task completing for group b in this wave (0..k-1 main,
 *                   k = parity), or -1 for none;  value [B][d] DEVICE fp32: its result.
 * Rule (App. C, with the third case read as "when the parity task completes", DESIGN.md R-f2a):
 * a main task j sets f^(x_j) = value (final) and subtracts value from every unfinalised
 * estimate; the parity adds k*value to every unfinalised estimate.  After k distinct tasks all
 * estimates are final (= ci_decode's result); later events change nothing.  A repeated task
 * is ignored and counted in the workspace flag (ci_check).  k <= 31; ws >= 256 B. */
CI_API ci_status_t ci_online_update(int32_t k, int64_t B, int64_t d, float* est, uint64_t* state,
                                    const int32_t* task, const float* value, void* ws, size_t ws_bytes,
                                    ci_stream_t stream);

/* ---- First-k gated serving with an injected straggler (App. C
 * PAPER.md:938-952; SPEC.md:279-287 run_query_*, 317 first-k gating, 388 per-event cost) -------
 * A latency harness of Q independent queries of one group each (k CIFAR-shaped inputs):
 * k main workers and, in CI_FIRSTK_CODED, the parity worker (learned encoder + f on the encoded
 * query) run concurrently, each on its own CUDA stream; straggler[q] >= 0 delays
 * main worker straggler[q]'s result of query q by delay_ns (0.1 s on one random
 * worker).  Each result is applied on arrival by the online decoder (ci_online_update's rule,
 * reading R-f2a); the query completes when any k results are in (coded: first-k gating) or when
 * all k mains are in (CI_FIRSTK_UNCODED: no parity worker), and the heads run on the k
 * recovered features right there.  Up to max_inflight queries overlap (a slot is reused once
 * all of its workers, including a straggler, have reported).
 *   x        [Q][k][in_c][in_h][in_w] DEVICE;  straggler [Q] HOST int32 (-1: none)
 *   features [Q][k][d] DEVICE: the recovered f(x_i) (the straggler's slot decoded when the
 *            parity beat it)
 *   logits   [n_heads][Q][k][C_t], labels [n_heads][Q][k] DEVICE (may be NULL without heads)
 *   records  [Q][4] DEVICE int64: {latency_ns (submit -> predictions, device globaltimer),
 *            update_ns (the completing event's online update), heads_ns, decode-set mask
 *            (bit j = task j used, bit k = parity) | degraded << 32}
 * Synchronous: blocks while more than max_inflight queries are outstanding and returns when all
 * Q queries have finished (it creates and destroys its own k + 1 + max_inflight streams).
 * CI_FIRSTK_CODED needs a model with the learned encoder (CI_ERR_UNSUPPORTED otherwise).  Every
 * stream needs its own hardware queue: the process must have been started with
 * CUDA_DEVICE_MAX_CONNECTIONS >= k + 2 + max_inflight (<= 32), else CI_ERR_UNSUPPORTED (with
 * shared queues a delayed worker would falsely stall other queries' workers). */
typedef enum { CI_FIRSTK_CODED = 0, CI_FIRSTK_UNCODED = 1 } ci_firstk_mode_t;
CI_API ci_status_t ci_workspace_size_first_k(const ci_model_t* model, int32_t k, int32_t max_inflight,
                                             size_t* bytes);
CI_API ci_status_t ci_serve_first_k(const ci_model_t* model, ci_firstk_mode_t mode, int32_t k, int64_t Q,
                                    const float* x, const int32_t* straggler, int64_t delay_ns,
                                    int32_t max_inflight, float* features, float* logits, int32_t* labels,
                                    int64_t* records, void* ws, size_t ws_bytes, ci_stream_t stream);

/* ---- General (n, k) codes, n - k = r >= 1 parity tasks (Eq. 3, 563-597;
 * SURVEY §8f f3) ----------------------------------------------------------------------------
 * The generator is systematic: tasks 0..k-1 are the main queries (rows = I_k), task k+i is the
 * parity query x_{k+i} = h^-1(sum_j c_{i,j} h(x_j)).  coef: DEVICE float
 * [r][k] row-major c_{i,j}; any k rows of G must be full rank -- the caller
 * guarantees it (decode flags a singular subset).  avail: DEVICE uint32 [B], bit s set when task
 * s has a result (n <= 32).  Decode uses S = the k smallest available tasks and solves for the
 * missing main tasks from the parity rows in S (fp64 p x p inverse per group, p = missing
 * mains); available main results are left untouched.  Groups with fewer than k available tasks
 * or a singular subset (scaled |det G_S| <= 1e-9, rows of G_S normalised: SPEC.md:24) are left
 * untouched and counted in the workspace's undecodable flag (ci_check: CI_ERR_UNDECODABLE).
 * Exact encode only (the learned encoder of a3' produces one parity query). */
CI_API ci_status_t ci_workspace_size_general(const ci_model_t* model, int32_t k, int32_t r, int64_t B,
                                             size_t* bytes);
/* h [B][k][d] -> comb_out [B][r][d] (optional) and x_parity [B][r][C][H][W] */
CI_API ci_status_t ci_encode_general(const ci_model_t* model, int32_t k, int32_t r, int64_t B,
                                     const float* coef, const float* h, float* x_parity, float* comb_out,
                                     void* ws, size_t ws_bytes, ci_stream_t stream);
/* h [B][k][d] (in/out: missing main tasks overwritten), h_parity [B][r][d]; ws >= 256 B */
CI_API ci_status_t ci_decode_general(int32_t k, int32_t r, int64_t B, int64_t d, const float* coef, float* h,
                                     const float* h_parity, const uint32_t* avail, void* ws, size_t ws_bytes,
                                     ci_stream_t stream);
/* Whole path: h on B*k main queries -> encode r parity queries -> h on them -> decode ->
 * heads on all B*k decoded features (logits/labels layout as ci_serve_group). */
CI_API ci_status_t ci_serve_general(const ci_model_t* model, int32_t k, int32_t r, int64_t B, const float* coef,
                                    const float* x, const uint32_t* avail, float* h_out, float* h_parity,
                                    float* x_parity, float* logits, int32_t* labels, void* ws, size_t ws_bytes,
                                    ci_stream_t stream);

/* Per-group drop indices generated on the device, bit-identical to the fixtures' host
 * generator: drop[b] = (uint32)(splitmix64_at(seed, b) >> 32) % k (counter-based splitmix64;
 * one uniformly random lost main worker per group). */
CI_API ci_status_t ci_make_drops(int32_t k, int64_t B, uint64_t seed, int32_t* drop, ci_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* CODEDINV_H_ */
