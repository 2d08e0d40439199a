// Internal declarations of libcodedinv (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "codedinv.h"

namespace ci {

void set_error(const char* fmt, ...);
ci_status_t cuda_status(cudaError_t e, const char* what);

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

struct StageInfo {
    int C, H, W;   // state shape after the stage's squeeze
    int c, m, nb;  // half channels, hidden width, blocks
    int squeeze;   // psi before the stage
};

struct Model {
    ci_arch_t arch;
    ci_precision_t prec;
    int device;
    int n_stages;
    StageInfo st[4];
    int64_t d, din;
    int64_t n_params;
    float* d_params = nullptr;               // canonical flat fp32 params on device
    std::vector<int64_t> blk_off;            // offset of W1 of block (s,t), flattened
    std::vector<int> blk_first;              // first block index of each stage
    int64_t head_off[4] = {0, 0, 0, 0};
    float* d_head[4] = {nullptr, nullptr, nullptr, nullptr};  // 16-B aligned copy: W [C][d], then b [C]
    int64_t enc_off = -1;                    // learned encoder params (float offset), -1 = none
    std::vector<float> enc_host;             // host copy of E1 W, b and E4 W, b (kernel parameters)
    // tcgen05 path
    uint16_t* d_wpack = nullptr;             // packed bf16 / fp16 weights (k_umma.cu pack_block)
    float* d_bias = nullptr;                 // padded biases
    void* umma_state = nullptr;              // host-side stage plans (k_umma.cu)
    void* host_pipe = nullptr;               // streams/events of ci_serve_group_host (api.cu)
};

void release_host_pipe(Model* m);   // api.cu: streams/events of the host-buffer entry

// ---- worker-partition communicator (comm.cu)
constexpr int kCommMaxRanks = 32;
constexpr size_t kCommHeader = 256;          // window: [pub, done] epoch counters, then feat [cap_B][d]
constexpr int kCommPub = 0, kCommDone = 1;   // uint64 index of the counters in the window
struct Comm {
    int nranks = 0, rank = 0, layout = 0, device = 0;
    int64_t cap_B = 0, d = 0;
    void* win = nullptr;                     // own window (cudaMalloc, exported by CUDA IPC)
    void* peers[kCommMaxRanks] = {};         // every rank's window base in this process
    bool opened[kCommMaxRanks] = {};         // peers[q] came from cudaIpcOpenMemHandle
    void** d_peers = nullptr;                // device copy of peers[]
    uint64_t epoch = 0;                      // serve calls issued on this communicator
};
// ---- first-k gated serving harness (firstk.cu; orchestration in api.cu)
struct FkSlot {              // one in-flight query
    uint64_t t_submit;       // device globaltimer at submission
    int64_t q;               // query index using the slot
    uint32_t recv, fin;      // tasks received (bit k = parity) / estimates finalised
    int lock, complete;
    int pad[2];
};
cudaError_t launch_fk_submit(FkSlot* slot, float* est, int64_t nest, int64_t q, cudaStream_t s);
cudaError_t launch_fk_delay(int64_t delay_ns, cudaStream_t s);
cudaError_t launch_fk_arrive(FkSlot* slot, float* est, const float* v, int j, int k, int64_t d, int need_mains,
                             const float* const* heads_w, const int* head_c, int n_heads, float* feat_out,
                             float* logits, int32_t* labels, int64_t Q, int64_t* rec, cudaStream_t s);
ci_status_t comm_publish(Comm* c, const float* src, int64_t B, cudaStream_t st);
ci_status_t comm_peer_mean(Comm* c, int k, int64_t B, float* mean, cudaStream_t st);
ci_status_t comm_peer_decode(Comm* c, int k, int64_t B, const int32_t* drop, float* out, int* flag,
                             cudaStream_t st);

// ---- accounting (codedinv_testing.h)
void count_launch(int n = 1);

// ---- kernels (launchers) ------------------------------------------------------
// permutation copy between stage layouts: mode 0 identity, 1 psi, 2 psi^-1
// in: [n][C][H][W] of the SOURCE layout.  C,H,W are the source shape.
cudaError_t launch_permute(const float* in, float* out, int64_t n, int C, int H, int W, int mode,
                           cudaStream_t s);
// SIMT conv3x3 (NCHW, fp32): out = act(conv(in) + b)   (mode 0; act 0 ReLU, 1 ELU, 2 identity)
//                            out += conv(in) + b       (mode 1)
//                            out -= conv(in) + b       (mode 2)
//                            out = base - conv(in) - b (mode 3, residual fixed-point update)
// m = (sum_i h_i) / k  (+ eps when given: perturbed encode, f4)
cudaError_t launch_mean(const float* h, float* m, int k, int64_t B, int64_t d, cudaStream_t s,
                        const float* eps = nullptr);
cudaError_t launch_decode(float* h, const float* p, const int32_t* drop, int k, int64_t B,
                          int64_t d, int* flag, cudaStream_t s);
cudaError_t launch_classify(const float* z, int64_t n, int64_t d, const float* W, const float* b,
                            int C, float* logits, int32_t* labels, cudaStream_t s);
cudaError_t launch_make_drops(int k, int64_t B, uint64_t seed, int32_t* drop, cudaStream_t s);
// online decoding (k_online.cu)
cudaError_t launch_online_update(int k, int64_t B, int64_t d, float* est, uint64_t* state, const int32_t* task,
                                 const float* value, int* flag, cudaStream_t s);
// general (n, k) codes (k_codes.cu)
cudaError_t launch_combine_general(const float* h, const float* coef, float* out, int k, int r, int64_t B,
                                   int64_t d, cudaStream_t s);
cudaError_t launch_decode_general(float* h, const float* hp, const float* coef, const uint32_t* avail, int k, int r,
                                  int64_t B, int64_t d, int* flag, cudaStream_t s);
// learned encoder (k_encoder.cu): weights are HOST pointers (passed as kernel parameters)
bool enc_supported(int Ci, int C1, int H, int W);
cudaError_t launch_enc_e1_mean(const float* x, int k, int64_t B, int Ci, int H, int W, const float* hw1,
                               const float* hb1, int C1, float* m, float* zpsi, int64_t zstride, cudaStream_t s);
cudaError_t launch_enc_out(const float* z, int64_t zstride, const float* m, int64_t B, int Ci, int C1, int H, int W,
                           const float* hw4, const float* hb4, float* xp, cudaStream_t s);

// tcgen05 path (k_umma.cu)
ci_status_t umma_prepare(Model* m, const float* host_params);
void umma_release(Model* m);
// Runs one stage (all blocks) on the fp32 NCHW state `state` [n][C][H][W] in place.
// ctr: a zeroed int the launch claims batches from (null: static round-robin batches).
// TS stages can read their input from src (layout in_mode) and write to dst (layout out_mode),
// stage_io.cuh; every other stage runs in place in its own layout (src == dst, modes 0).
bool umma_stage_fuses_io(const Model* m, int stage);
ci_status_t umma_stage_io(const Model* m, int stage, const float* src, int in_mode, float* dst, int out_mode,
                          int64_t n, bool inverse, int* ctr, cudaStream_t s);
ci_status_t umma_stage(const Model* m, int stage, float* state, int64_t n, bool inverse,
                       int* ctr, cudaStream_t s);
// Learned-encoder tail: zbuf [n][2*4c1][H/2][W/2]; channels [0,4c1) = psi(mean first layer) in,
// channels [4c1, 8c1) = ReLU(E3(ReLU(E2 z))) out (tcgen05 stage kernel, fmode 1).
ci_status_t umma_encoder_tail(const Model* m, float* zbuf, int64_t n, int* ctr, cudaStream_t s);
bool umma_has_encoder(const Model* m);   // the encoder tail has a tcgen05 plan

// TS-mode stage kernel (k_stage_ts.cu): Arch C stage 1 (16x16, c = 6, m = 64, coupling + ReLU)
// with the hidden activation kept in tensor memory
struct TsArgs {
    // images in global memory: read from src in layout in_mode, written to dst in layout out_mode
    // (stage_io.cuh: 0 = the stage's own [C][H][W], 1 = the previous stage's, 2 = the next
    // stage's, i.e. psi / psi^-1 fused into the load / store).  src == dst is allowed (each image
    // is read completely before it is written; all layouts have the same size).
    const float* src;
    float* dst;
    int in_mode, out_mode;
    int64_t n;               // images
    const uint8_t* wpack;    // stage stream: block t at t * blk_bytes (pack_block, StagePlan::ts)
    int64_t blk_bytes;
    const float* bias;       // block t at t * bias_stride: [64] b1 (folded, unused), then b2 by channel
    int bias_stride;
    int nb, first_orient, inverse;
    int* ctr;                // zeroed batch counter of this launch, or null
    unsigned long long* dbg; // optional per-CTA cycle counters (CI_DEBUG_CYCLES), 16 per CTA
    int sched;               // k_stage_ts2 MMA schedule: 0 lockstep, shared weight stream; 1 offset slots
};
bool stage_ts_shape(int H, int W, int C, int c, int m, int residual, int act);
int64_t stage_ts_block_bytes(int pm);
int stage_ts_smem(int pm);
int stage_ts_n2();
void stage_ts_col(int n, int& tap, int& o);   // conv2 column -> (tap, output channel), tap -1 = padding
cudaError_t stage_ts_prepare();
bool stage_ts_stacked(int pm);   // f16x3: stacked conv1 (CI_TS_UNSTK=1: three N = 64 MMAs per k-step)
cudaError_t launch_stage_ts(const TsArgs& a, int pm, int stk, cudaStream_t st);
// TS-mode kernel for Arch C stage 2 (8x8, c = 24, m = 128; k_stage_ts2.cu)
bool stage_ts2_shape(int H, int W, int C, int c, int m, int residual, int act);
int64_t stage_ts2_block_bytes(int pm);
int stage_ts2_smem(int pm);
cudaError_t stage_ts2_prepare();
cudaError_t launch_stage_ts2(const TsArgs& a, int pm, cudaStream_t st);

}  // namespace ci
