// C ABI of libcodedinv: argument validation, model packing, workspace carving and the
// orchestration of the coded path (see include/codedinv.h for the contract).
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>

#include "ci_internal.h"
#include "codedinv_testing.h"

namespace ci {

static thread_local char g_err[512] = "no error";
static std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches += n; }

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

ci_status_t cuda_status(cudaError_t e, const char* what) {
    set_error("CUDA error %d (%s) in %s", (int)e, cudaGetErrorString(e), what);
    return CI_ERR_CUDA;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// ---------------------------------------------------------------------------
// workspace layout
// ---------------------------------------------------------------------------
static constexpr size_t kAlign = 256;
static size_t up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct WsLayout {
    size_t flag = 0, scratch = 0, mean = 0, xp = 0, hidden = 0, enc = 0, total = 0;
    mutable int ctr_next = 0;   // next batch-counter slot of this call (see next_ctr)
};

// The flag region (256 B) holds the drop-index error count (int 0) and, in ints
// kCtrBase.., one zeroed batch counter per tcgen05 stage launch of an API call: the stage
// kernel claims batches dynamically from it.  zero_ctrs runs once at the start of a call.
static constexpr int kCtrBase = 16, kCtrSlots = 48;
static cudaError_t zero_ctrs(void* ws, const WsLayout& L, cudaStream_t st) {
    L.ctr_next = 0;
    return cudaMemsetAsync(reinterpret_cast<int*>(reinterpret_cast<char*>(ws) + L.flag) + kCtrBase, 0,
                           sizeof(int) * kCtrSlots, st);
}
static int* next_ctr(void* ws, const WsLayout& L) {
    static const bool static_batches = getenv("CI_STATIC_BATCHES") != nullptr;   // A/B switch
    if (static_batches || L.ctr_next >= kCtrSlots) return nullptr;   // static round-robin batches
    return reinterpret_cast<int*>(reinterpret_cast<char*>(ws) + L.flag) + kCtrBase + L.ctr_next++;
}

// groups = false: layout of a plain h / h^-1 call on n = B*k images (no per-group buffers)
// r: parity queries per group (1 for n = k + 1; general codes r = n - k)
static WsLayout ws_layout(const Model* m, int32_t k, int64_t B, bool groups = true, int32_t r = 1) {
    WsLayout L;
    int64_t n = B * (int64_t)std::max(k, r);
    const int64_t Bg = groups ? std::max<int64_t>(B, 1) * r : 0;
    size_t off = 0;
    L.flag = off; off += up(256);
    L.scratch = off; off += up(sizeof(float) * (size_t)(std::max<int64_t>(n, 1) * m->d));
    L.mean = off; off += up(sizeof(float) * (size_t)(Bg * m->d));
    L.xp = off; off += up(sizeof(float) * (size_t)(Bg * m->din));
    L.enc = off;
    if (m->enc_off >= 0 && groups) {   // m, z, z2, z3, u of the learned encoder
        const int64_t HW = (int64_t)m->arch.in_h * m->arch.in_w;
        const int64_t per = HW * (3 * m->arch.enc_c1) + 64;   // m [c1][H][W], zbuf [8 c1][H/2][W/2]
        off += up(sizeof(float) * (size_t)(std::max<int64_t>(B, 1) * per));
    }
    L.total = off;
    return L;
}

template <class T>
static T* at(void* ws, size_t off) { return reinterpret_cast<T*>(reinterpret_cast<char*>(ws) + off); }

// ---------------------------------------------------------------------------
// h / h^-1 orchestration (both precisions share the stage-boundary permutations)
// ---------------------------------------------------------------------------
// Stage-boundary permutations fused into the TS stage kernels' load / store (stage_io.cuh): possible
// when every psi between two stages -- and the copy of x into the first stage -- is adjacent to a
// TS stage.  Then h runs in place in one buffer and no k_permute pass is launched.
static bool fused_io_forward(const Model* m) {
    static const bool off = getenv("CI_NO_FUSED_IO") != nullptr;   // A/B switch: separate k_permute passes
    if (off) return false;
    const int S = m->n_stages;
    if (!umma_stage_fuses_io(m, 0)) return false;
    for (int s = 1; s < S; s++)
        if (m->st[s].squeeze && !umma_stage_fuses_io(m, s - 1) && !umma_stage_fuses_io(m, s)) return false;
    return true;
}
static bool fused_io_inverse(const Model* m) { return fused_io_forward(m); }   // same boundaries, reversed

static ci_status_t forward_impl(const Model* m, const float* x, float* h, int64_t n, void* ws,
                                const WsLayout& L, cudaStream_t st) {
    if (n == 0) return CI_OK;
    if (fused_io_forward(m)) {
        const int S = m->n_stages;
        for (int s = 0; s < S; s++) {
            const bool ts = umma_stage_fuses_io(m, s);
            // layouts (stage_io.cuh): 1 = the previous stage's (psi on load), 2 = the next stage's (psi on store)
            const int in_mode = ts && m->st[s].squeeze && (s == 0 || !umma_stage_fuses_io(m, s - 1)) ? 1 : 0;
            const int out_mode = ts && s + 1 < S && m->st[s + 1].squeeze ? 2 : 0;
            ci_status_t r = umma_stage_io(m, s, s == 0 ? x : h, in_mode, h, out_mode, n, false, next_ctr(ws, L), st);
            if (r != CI_OK) return r;
        }
        return CI_OK;
    }
    float* scratch = at<float>(ws, L.scratch);
    // stage s starts with a copy (psi or identity) into buffer buf[s]; last buffer = h
    const int S = m->n_stages;
    const float* src = x;
    int C = m->arch.in_c, H = m->arch.in_h, W = m->arch.in_w;
    for (int s = 0; s < S; s++) {
        float* dst = ((S - 1 - s) % 2 == 0) ? h : scratch;
        CI_CUDA(launch_permute(src, dst, n, C, H, W, m->st[s].squeeze ? 1 : 0, st));
        C = m->st[s].C; H = m->st[s].H; W = m->st[s].W;
        ci_status_t r = umma_stage(m, s, dst, n, false, next_ctr(ws, L), st);
        if (r != CI_OK) return r;
        src = dst;
    }
    return CI_OK;
}

// consume_h: h is library scratch (the encode mean inside ci_serve_group) that the inverse may
// overwrite, so the last stage runs on it in place and the initial identity copy is skipped
static ci_status_t inverse_impl(const Model* m, const float* h, float* x, int64_t n, void* ws,
                                const WsLayout& L, cudaStream_t st, bool consume_h = false) {
    if (n == 0) return CI_OK;
    float* scratch = at<float>(ws, L.scratch);
    const int S = m->n_stages;
    if (fused_io_inverse(m)) {
        // cur: the working buffer (h itself when the caller hands it over); the last stage reads h
        // directly when it is a TS stage, otherwise h is copied into cur first
        float* cur = consume_h ? const_cast<float*>(h) : scratch;
        const bool ts_last = umma_stage_fuses_io(m, S - 1);
        if (!consume_h && !ts_last) {
            const StageInfo& L3 = m->st[S - 1];
            CI_CUDA(launch_permute(h, cur, n, L3.C, L3.H, L3.W, 0, st));
        }
        for (int s = S - 1; s >= 0; s--) {
            const bool ts = umma_stage_fuses_io(m, s);
            const float* src = (s == S - 1 && ts) ? h : cur;
            float* dst = s == 0 ? x : cur;
            // layouts: 2 = the next stage's (psi^-1 on load), 1 = the previous stage's (psi^-1 on store)
            const int in_mode = ts && s + 1 < S && m->st[s + 1].squeeze && !umma_stage_fuses_io(m, s + 1) ? 2 : 0;
            const int out_mode = ts && m->st[s].squeeze ? 1 : 0;
            ci_status_t r = umma_stage_io(m, s, src, in_mode, dst, out_mode, n, true, next_ctr(ws, L), st);
            if (r != CI_OK) return r;
        }
        return CI_OK;
    }
    // copies: [1 initial] + 1 after each stage, the last one lands in x
    int ncopy = consume_h ? S : S + 1, ci = 0;
    auto target = [&](int i) { return ((ncopy - 1 - i) % 2 == 0) ? x : scratch; };
    float* cur;
    if (consume_h) {
        cur = const_cast<float*>(h);
    } else {
        cur = target(ci++);
        const StageInfo& L3 = m->st[S - 1];
        CI_CUDA(launch_permute(h, cur, n, L3.C, L3.H, L3.W, 0, st));
    }
    for (int s = S - 1; s >= 0; s--) {
        ci_status_t r = umma_stage(m, s, cur, n, true, next_ctr(ws, L), st);
        if (r != CI_OK) return r;
        float* nxt = target(ci++);
        const StageInfo& Si = m->st[s];
        CI_CUDA(launch_permute(cur, nxt, n, Si.C, Si.H, Si.W, Si.squeeze ? 2 : 0, st));
        cur = nxt;
    }
    return CI_OK;
}

static ci_status_t encode_learned_impl(const Model* m, const float* x, float* xp, int32_t k, int64_t B,
                                       void* ws, const WsLayout& L, cudaStream_t st) {
    if (B == 0) return CI_OK;
    const ci_arch_t& a = m->arch;
    const int Ci = a.in_c, H = a.in_h, W = a.in_w, c1 = a.enc_c1, mid = a.enc_mid;
    const int64_t HW = (int64_t)H * W, hw4 = HW / 4;
    const float* E1W = m->enc_host.data();                         // host copies: kernel parameters
    const float* E1b = E1W + (int64_t)c1 * Ci * 9;
    const float* E4W = E1b + c1;
    const float* E4b = E4W + (int64_t)Ci * c1 * 9;
    // workspace: m [B][c1][H][W] | zbuf [B][8c1][H/2][W/2] (tail in | out, in place)
    float* Mb = at<float>(ws, L.enc);
    float* Zb = Mb + B * c1 * HW;
    const int64_t zstride = 8 * c1 * hw4;
    CI_CUDA(launch_enc_e1_mean(x, k, B, Ci, H, W, E1W, E1b, c1, Mb, Zb, zstride, st));   // E1, mean, psi
    ci_status_t r = umma_encoder_tail(m, Zb, B, next_ctr(ws, L), st);              // ReLU(E3(ReLU(E2 z)))
    if (r != CI_OK) return r;
    CI_CUDA(launch_enc_out(Zb + 4 * c1 * hw4, zstride, Mb, B, Ci, c1, H, W, E4W, E4b, xp, st));   // psi^-1 + skip, E4
    return CI_OK;
}

}  // namespace ci

using namespace ci;

// ===========================================================================
// exported C ABI
// ===========================================================================
extern "C" {

const char* ci_last_error(void) { return g_err; }

ci_status_t ci_model_create(const ci_arch_t* arch, const float* host_params, size_t n_params,
                            ci_precision_t precision, int device, ci_model_t** out) {
    if (!arch || !host_params || !out) { set_error("NULL argument"); return CI_ERR_INVALID_ARG; }
    *out = nullptr;
    if (precision != CI_PREC_FP32 && precision != CI_PREC_BF16 && precision != CI_PREC_F16X2) {
        set_error("unknown precision %d", (int)precision);
        return CI_ERR_INVALID_ARG;
    }
    const ci_arch_t& a = *arch;
    if (a.n_stages < 1 || a.n_stages > 4 || a.in_c < 1 || a.in_h < 1 || a.in_w < 1 ||
        a.n_heads < 0 || a.n_heads > 4 || a.act < 0 || a.act > 2 || a.block_kind < 0 || a.block_kind > 1 ||
        (a.block_kind == 1 && (a.fp_iters < 1 || a.fp_iters > 1000))) {
        set_error("invalid arch descriptor");
        return CI_ERR_INVALID_SHAPE;
    }
    const bool residual = a.block_kind == 1;
    Model* m = new Model();
    m->arch = a;
    m->prec = precision;
    m->device = device;
    m->n_stages = a.n_stages;
    int C = a.in_c, H = a.in_h, W = a.in_w;
    int64_t off = 0;
    for (int s = 0; s < a.n_stages; s++) {
        const ci_stage_t& sg = a.stage[s];
        if (sg.squeeze_before) {
            if (H % 2 || W % 2) { delete m; set_error("psi needs even H, W"); return CI_ERR_INVALID_SHAPE; }
            C *= 4; H /= 2; W /= 2;
        }
        if ((!residual && C % 2) || sg.n_blocks < 1 || sg.mid_channels < 1) {
            delete m; set_error("stage %d: odd channel count or empty stage", s); return CI_ERR_INVALID_SHAPE;
        }
        StageInfo& S = m->st[s];
        S.C = C; S.H = H; S.W = W; S.c = residual ? C : C / 2; S.m = sg.mid_channels; S.nb = sg.n_blocks;
        S.squeeze = sg.squeeze_before;
        m->blk_first.push_back((int)m->blk_off.size());
        for (int t = 0; t < S.nb; t++) {
            m->blk_off.push_back(off);
            off += (int64_t)S.m * S.c * 9 + S.m + (int64_t)S.c * S.m * 9 + S.c;
        }
    }
    m->d = (int64_t)C * H * W;
    m->din = (int64_t)a.in_c * a.in_h * a.in_w;
    if (m->d != m->din) { delete m; set_error("h must be dimension preserving"); return CI_ERR_INVALID_SHAPE; }
    for (int t = 0; t < a.n_heads; t++) {
        if (a.head_classes[t] < 1 || a.head_classes[t] > 16) {
            delete m; set_error("head %d: classes must be in [1,16]", t); return CI_ERR_INVALID_SHAPE;
        }
        m->head_off[t] = off;
        off += (int64_t)a.head_classes[t] * m->d + a.head_classes[t];
    }
    if (a.enc_c1 > 0 || a.enc_mid > 0) {
        if (a.enc_c1 < 1 || a.enc_mid < 1 || a.in_h % 2 || a.in_w % 2) {
            delete m; set_error("invalid learned encoder widths"); return CI_ERR_INVALID_SHAPE;
        }
        if (!enc_supported(a.in_c, a.enc_c1, a.in_h, a.in_w)) {
            delete m;
            set_error("learned encoder: in_c must be 3, enc_c1 4, 8 or 16, in_w 8, 16 or 32, in_h even, in_h * in_w <= 1024");
            return CI_ERR_UNSUPPORTED;
        }
        m->enc_off = off;
        off += (int64_t)a.enc_c1 * a.in_c * 9 + a.enc_c1 + (int64_t)a.enc_mid * 4 * a.enc_c1 * 9 + a.enc_mid +
               (int64_t)4 * a.enc_c1 * a.enc_mid * 9 + 4 * a.enc_c1 + (int64_t)a.in_c * a.enc_c1 * 9 + a.in_c;
    }
    m->n_params = off;
    if (m->enc_off >= 0) {   // E1 (W, b) and E4 (W, b) travel as kernel parameters
        const ci_arch_t& e = a;
        const float* p0 = host_params + m->enc_off;
        const int64_t n1 = (int64_t)e.enc_c1 * e.in_c * 9 + e.enc_c1;
        const int64_t mid = (int64_t)e.enc_mid * 4 * e.enc_c1 * 9 + e.enc_mid + (int64_t)4 * e.enc_c1 * e.enc_mid * 9 + 4 * e.enc_c1;
        const int64_t n4 = (int64_t)e.in_c * e.enc_c1 * 9 + e.in_c;
        if ((size_t)off == n_params) {
            m->enc_host.assign(p0, p0 + n1);
            m->enc_host.insert(m->enc_host.end(), p0 + n1 + mid, p0 + n1 + mid + n4);
        }
    }
    if ((size_t)off != n_params) {
        delete m;
        set_error("n_params %zu != %lld implied by arch", n_params, (long long)off);
        return CI_ERR_DIM_MISMATCH;
    }
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) { delete m; return cuda_status(e, "cudaSetDevice"); }
    e = cudaMalloc(&m->d_params, sizeof(float) * (size_t)off);
    if (e != cudaSuccess) { delete m; return cuda_status(e, "cudaMalloc params"); }
    e = cudaMemcpy(m->d_params, host_params, sizeof(float) * (size_t)off, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { cudaFree(m->d_params); delete m; return cuda_status(e, "cudaMemcpy params"); }
    for (int t = 0; t < a.n_heads; t++) {
        size_t nh = (size_t)a.head_classes[t] * (m->d + 1);
        e = cudaMalloc(&m->d_head[t], sizeof(float) * nh);
        if (e == cudaSuccess)
            e = cudaMemcpy(m->d_head[t], host_params + m->head_off[t], sizeof(float) * nh, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) { ci_model_destroy(reinterpret_cast<ci_model_t*>(m)); return cuda_status(e, "head weights"); }
    }
    ci_status_t r = umma_prepare(m, host_params);
    if (r != CI_OK) { ci_model_destroy(reinterpret_cast<ci_model_t*>(m)); return r; }
    if (m->enc_off >= 0 && !umma_has_encoder(m)) {   // every later learned-mode call needs the tail plan
        ci_model_destroy(reinterpret_cast<ci_model_t*>(m));
        set_error("learned encoder widths (c1=%d, mid=%d) do not fit the tcgen05 stage kernel", a.enc_c1, a.enc_mid);
        return CI_ERR_UNSUPPORTED;
    }
    *out = reinterpret_cast<ci_model_t*>(m);
    return CI_OK;
}

void ci_model_destroy(ci_model_t* model) {
    Model* m = reinterpret_cast<Model*>(model);
    if (!m) return;
    umma_release(m);
    release_host_pipe(m);
    cudaFree(m->d_params);
    for (int t = 0; t < 4; t++) cudaFree(m->d_head[t]);
    delete m;
}

int64_t ci_feature_dim(const ci_model_t* model) {
    const Model* m = reinterpret_cast<const Model*>(model);
    return m ? m->d : -1;
}

ci_status_t ci_workspace_size(const ci_model_t* model, int32_t k, int64_t B, size_t* bytes) {
    const Model* m = reinterpret_cast<const Model*>(model);
    if (!m || !bytes || k < 1 || B < 0) { set_error("invalid argument"); return CI_ERR_INVALID_ARG; }
    *bytes = ws_layout(m, k, B).total;
    return CI_OK;
}

#define CI_MODEL_OR_FAIL(mv, model)                                          \
    const Model* mv = reinterpret_cast<const Model*>(model);                 \
    if (!mv) { set_error("NULL model"); return CI_ERR_INVALID_ARG; }

static ci_status_t check_ws(const WsLayout& L, void* ws, size_t ws_bytes) {
    if (!ws || !aligned16(ws) || ws_bytes < L.total) {
        set_error("workspace %p of %zu bytes; need %zu (16-byte aligned)", ws, ws_bytes, L.total);
        return CI_ERR_WORKSPACE;
    }
    return CI_OK;
}

ci_status_t ci_check(const ci_model_t* model, void* ws, size_t ws_bytes, ci_stream_t stream) {
    (void)model;
    if (!ws || ws_bytes < 256) { set_error("workspace too small"); return CI_ERR_WORKSPACE; }
    int flag[2] = {0, 0};   // [0] drop index out of range, [1] undecodable groups
    CI_CUDA(cudaMemcpyAsync(flag, ws, sizeof(flag), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    CI_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    if (flag[0] || flag[1]) {
        CI_CUDA(cudaMemsetAsync(ws, 0, sizeof(flag), (cudaStream_t)stream));
        CI_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
        if (flag[1]) {
            set_error("%d group(s) could not be decoded (fewer than k results or a singular subset)", flag[1]);
            return CI_ERR_UNDECODABLE;
        }
        set_error("%d group(s) had a drop index outside [-1, k)", flag[0]);
        return CI_ERR_INVALID_ARG;
    }
    return CI_OK;
}

ci_status_t ci_forward_h(const ci_model_t* model, const float* x, float* h, int64_t n, void* ws,
                         size_t ws_bytes, ci_stream_t stream) {
    CI_MODEL_OR_FAIL(m, model);
    if (n < 0 || (n > 0 && (!x || !h || !aligned16(x) || !aligned16(h)))) {
        set_error("invalid x/h/n"); return CI_ERR_INVALID_ARG;
    }
    WsLayout L = ws_layout(m, 1, n, false);
    ci_status_t r = check_ws(L, ws, ws_bytes);
    if (r != CI_OK) return r;
    CI_CUDA(zero_ctrs(ws, L, (cudaStream_t)stream));
    return forward_impl(m, x, h, n, ws, L, (cudaStream_t)stream);
}

ci_status_t ci_inverse_h(const ci_model_t* model, const float* h, float* x, int64_t n, void* ws,
                         size_t ws_bytes, ci_stream_t stream) {
    CI_MODEL_OR_FAIL(m, model);
    if (n < 0 || (n > 0 && (!x || !h || !aligned16(x) || !aligned16(h)))) {
        set_error("invalid x/h/n"); return CI_ERR_INVALID_ARG;
    }
    WsLayout L = ws_layout(m, 1, n, false);
    ci_status_t r = check_ws(L, ws, ws_bytes);
    if (r != CI_OK) return r;
    CI_CUDA(zero_ctrs(ws, L, (cudaStream_t)stream));
    return inverse_impl(m, h, x, n, ws, L, (cudaStream_t)stream);
}

ci_status_t ci_encode(const ci_model_t* model, ci_encode_mode_t mode, int32_t k, int64_t B,
                      const float* x, const float* h, float* x_parity, float* mean_out, void* ws, size_t ws_bytes,
                      ci_stream_t stream) {
    CI_MODEL_OR_FAIL(m, model);
    if (mode != CI_ENC_EXACT && mode != CI_ENC_LEARNED) { set_error("unknown encode mode"); return CI_ERR_INVALID_ARG; }
    if (mode == CI_ENC_LEARNED && m->enc_off < 0) { set_error("model has no learned encoder"); return CI_ERR_UNSUPPORTED; }
    const float* in = mode == CI_ENC_EXACT ? h : x;
    if (k < 1 || B < 0 || (B > 0 && (!in || !x_parity || !aligned16(in) || !aligned16(x_parity))) ||
        (mean_out && !aligned16(mean_out))) {
        set_error("invalid argument"); return CI_ERR_INVALID_ARG;
    }
    WsLayout L = ws_layout(m, k, B);
    ci_status_t r = check_ws(L, ws, ws_bytes);
    if (r != CI_OK) return r;
    cudaStream_t st = (cudaStream_t)stream;
    CI_CUDA(zero_ctrs(ws, L, st));
    if (mode == CI_ENC_LEARNED) return encode_learned_impl(m, x, x_parity, k, B, ws, L, st);
    float* mean = mean_out ? mean_out : at<float>(ws, L.mean);
    CI_CUDA(launch_mean(h, mean, k, B, m->d, st));
    return inverse_impl(m, mean, x_parity, B, ws, L, st);
}

ci_status_t ci_encode_perturbed(const ci_model_t* model, int32_t k, int64_t B, const float* h, const float* eps,
                                float* x_parity, float* mean_out, void* ws, size_t ws_bytes, ci_stream_t stream) {
    CI_MODEL_OR_FAIL(m, model);
    if (k < 1 || B < 0 || (B > 0 && (!h || !eps || !x_parity || !aligned16(h) || !aligned16(eps) ||
                                     !aligned16(x_parity) || (mean_out && !aligned16(mean_out))))) {
        set_error("invalid argument"); return CI_ERR_INVALID_ARG;
    }
    WsLayout L = ws_layout(m, k, B);
    ci_status_t r = check_ws(L, ws, ws_bytes);
    if (r != CI_OK) return r;
    cudaStream_t st = (cudaStream_t)stream;
    CI_CUDA(zero_ctrs(ws, L, st));
    float* mean = mean_out ? mean_out : at<float>(ws, L.mean);
    CI_CUDA(launch_mean(h, mean, k, B, m->d, st, eps));
    return inverse_impl(m, mean, x_parity, B, ws, L, st);
}

ci_status_t ci_online_update(int32_t k, int64_t B, int64_t d, float* est, uint64_t* state, const int32_t* task,
                             const float* value, void* ws, size_t ws_bytes, ci_stream_t stream) {
    if (k < 1 || k > 31 || B < 0 || d < 0 || (B > 0 && (!est || !state || !task || !value || !aligned16(est) ||
                                                      !aligned16(value)))) {
        set_error("invalid argument"); return CI_ERR_INVALID_ARG;
    }
    if (!ws || ws_bytes < 256 || !aligned16(ws)) { set_error("workspace too small"); return CI_ERR_WORKSPACE; }
    CI_CUDA(launch_online_update(k, B, d, est, state, task, value, reinterpret_cast<int*>(ws), (cudaStream_t)stream));
    return CI_OK;
}

ci_status_t ci_decode(int32_t k, int64_t B, int64_t d, float* h, const float* h_parity,
                      const int32_t* drop, void* ws, size_t ws_bytes, ci_stream_t stream) {
    if (k < 1 || B < 0 || d < 0 ||
        (B > 0 && (!h || !h_parity || !drop || !aligned16(h) || !aligned16(h_parity)))) {
        set_error("invalid argument"); return CI_ERR_INVALID_ARG;
    }
    if (!ws || ws_bytes < 256 || !aligned16(ws)) { set_error("workspace too small"); return CI_ERR_WORKSPACE; }
    CI_CUDA(launch_decode(h, h_parity, drop, k, B, d, reinterpret_cast<int*>(ws), (cudaStream_t)stream));
    return CI_OK;
}

ci_status_t ci_classify(const ci_model_t* model, int32_t head, const float* z, int64_t n,
                        float* logits, int32_t* labels, ci_stream_t stream) {
    CI_MODEL_OR_FAIL(m, model);
    if (head < 0 || head >= m->arch.n_heads) { set_error("head %d out of range", head); return CI_ERR_INVALID_ARG; }
    if (n < 0 || (n > 0 && (!z || !aligned16(z)))) { set_error("invalid z/n"); return CI_ERR_INVALID_ARG; }
    const float* W = m->d_head[head];
    const float* b = W + (int64_t)m->arch.head_classes[head] * m->d;
    CI_CUDA(launch_classify(z, n, m->d, W, b, m->arch.head_classes[head], logits, labels,
                            (cudaStream_t)stream));
    return CI_OK;
}

// logits[t] / labels[t]: head t's [n][C_t] logits and [n] labels (null = not wanted)
static ci_status_t serve_impl(const Model* m, ci_encode_mode_t mode, int32_t k, int64_t B, const float* x,
                              const int32_t* drop, float* h_out, float* h_parity, float* x_parity,
                              float* const* logits, int32_t* const* labels, void* ws, const WsLayout& L,
                              cudaStream_t st) {
    const int64_t n = B * (int64_t)k;
    CI_CUDA(zero_ctrs(ws, L, st));
    ci_status_t r = forward_impl(m, x, h_out, n, ws, L, st);             // (1) h on main queries
    if (r != CI_OK) return r;
    float* mean = at<float>(ws, L.mean);
    float* xp = x_parity ? x_parity : at<float>(ws, L.xp);
    if (mode == CI_ENC_LEARNED) {
        r = encode_learned_impl(m, x, xp, k, B, ws, L, st);              // (2) learned encoder
    } else {
        CI_CUDA(launch_mean(h_out, mean, k, B, m->d, st));               // (2) encode: mean ...
        r = inverse_impl(m, mean, xp, B, ws, L, st, true);                //     ... then h^-1 (in place)
    }
    if (r != CI_OK) return r;
    r = forward_impl(m, xp, h_parity, B, ws, L, st);                      // (3) h on parity query
    if (r != CI_OK) return r;
    CI_CUDA(launch_decode(h_out, h_parity, drop, k, B, m->d, at<int>(ws, L.flag), st));  // (4)
    for (int t = 0; t < m->arch.n_heads; t++) {                           // (5) heads
        if (!logits[t] && !labels[t]) continue;
        const float* W = m->d_head[t];
        const float* b = W + (int64_t)m->arch.head_classes[t] * m->d;
        CI_CUDA(launch_classify(h_out, n, m->d, W, b, m->arch.head_classes[t], logits[t], labels[t], st));
    }
    return CI_OK;
}

// head-major output layout of logits [t][n][C_t] and labels [t][n] -> per-head pointers
static void head_ptrs(const Model* m, int64_t n, float* logits, int32_t* labels, float** lp, int32_t** bp) {
    int64_t lo = 0;
    for (int t = 0; t < 4; t++) { lp[t] = nullptr; bp[t] = nullptr; }
    for (int t = 0; t < m->arch.n_heads; t++) {
        lp[t] = logits ? logits + lo : nullptr;
        bp[t] = labels ? labels + t * n : nullptr;
        lo += n * m->arch.head_classes[t];
    }
}

// One worker of the paper's partition (CI_SHARD_WORKERS): see ci_serve_group in codedinv.h.
static ci_status_t serve_worker_impl(const Model* m, ci_encode_mode_t mode, int32_t k, int64_t B, const float* x,
                                     const int32_t* drop, float* h_out, float* h_dec, float* x_parity,
                                     float* const* logits, int32_t* const* labels, Comm* c, void* ws,
                                     const WsLayout& L, cudaStream_t st) {
    c->epoch++;
    const int r = c->rank;
    const int64_t Bp = (B + c->nranks - 1) / c->nranks;
    const int64_t b0 = std::min<int64_t>(B, (int64_t)r * Bp), nb = std::min<int64_t>(B, b0 + Bp) - b0;
    CI_CUDA(zero_ctrs(ws, L, st));
    ci_status_t rc;
    if (r < k) {
        rc = forward_impl(m, x, h_out, B, ws, L, st);                      // (1) h on slot r's queries
    } else {
        float* xp = x_parity ? x_parity : at<float>(ws, L.xp);
        if (mode == CI_ENC_LEARNED) {
            rc = encode_learned_impl(m, x, xp, k, B, ws, L, st);            // (2) X3 + learned encoder
        } else {
            float* mean = at<float>(ws, L.mean);
            rc = comm_peer_mean(c, k, B, mean, st);                         // (2) X2: mean over peers ...
            if (rc == CI_OK) rc = inverse_impl(m, mean, xp, B, ws, L, st); //     ... then h^-1
        }
        if (rc == CI_OK) rc = forward_impl(m, xp, h_out, B, ws, L, st);   // (3) h(x_p)
    }
    if (rc != CI_OK) return rc;
    rc = comm_publish(c, h_out, B, st);                                    // my result -> my window
    if (rc != CI_OK) return rc;
    rc = comm_peer_decode(c, k, B, drop, h_dec, at<int>(ws, L.flag), st);  // (4) X4 / K11 on my groups
    if (rc != CI_OK) return rc;
    for (int t = 0; t < m->arch.n_heads; t++) {                            // (5) heads
        const int64_t C = m->arch.head_classes[t];
        const float* W = m->d_head[t];
        const float* bias = W + C * m->d;
        if (r < k && (logits[t] || labels[t]))
            CI_CUDA(launch_classify(h_out, B, m->d, W, bias, (int)C, logits[t], labels[t], st));
        if (nb > 0 && (logits[t] || labels[t]))
            CI_CUDA(launch_classify(h_dec, nb, m->d, W, bias, (int)C, logits[t] ? logits[t] + B * C : nullptr,
                                    labels[t] ? labels[t] + B : nullptr, st));
    }
    return CI_OK;
}

ci_status_t ci_serve_group(const ci_model_t* model, ci_encode_mode_t mode, int32_t k, int64_t B,
                           const float* x, const int32_t* drop, float* h_out, float* h_parity,
                           float* x_parity, float* logits, int32_t* labels, ci_comm_t* comm, void* ws,
                           size_t ws_bytes, ci_stream_t stream) {
    CI_MODEL_OR_FAIL(m, model);
    if (mode != CI_ENC_EXACT && mode != CI_ENC_LEARNED) { set_error("unknown encode mode"); return CI_ERR_INVALID_ARG; }
    if (mode == CI_ENC_LEARNED && m->enc_off < 0) { set_error("model has no learned encoder"); return CI_ERR_UNSUPPORTED; }
    if (k < 1 || B < 0) { set_error("k must be >= 1 and B >= 0"); return CI_ERR_INVALID_ARG; }
    Comm* c = reinterpret_cast<Comm*>(comm);
    if (c && c->layout == CI_SHARD_WORKERS) {
        const bool parity = c->rank == k;
        const bool need_x = !parity || mode == CI_ENC_LEARNED;
        if (c->nranks != k + 1 || B > c->cap_B || c->d != m->d) {
            set_error("worker communicator: nranks %d (need k+1 = %d), B %lld (max %lld), d %lld (model %lld)",
                      c->nranks, k + 1, (long long)B, (long long)c->cap_B, (long long)c->d, (long long)m->d);
            return CI_ERR_INVALID_ARG;
        }
        if (B > 0 && ((need_x && (!x || !aligned16(x))) || !drop || !h_out || !h_parity || !aligned16(h_out) ||
                      !aligned16(h_parity) || (x_parity && !aligned16(x_parity)))) {
            set_error("invalid pointer argument"); return CI_ERR_INVALID_ARG;
        }
        WsLayout L = ws_layout(m, k, B);
        ci_status_t r = check_ws(L, ws, ws_bytes);
        if (r != CI_OK) return r;
        if (B == 0) return CI_OK;
        float* lp[4];
        int32_t* bp[4];
        head_ptrs(m, B + (B + k) / (k + 1), logits, labels, lp, bp);
        return serve_worker_impl(m, mode, k, B, x, drop, h_out, h_parity, x_parity, lp, bp, c, ws, L,
                                 (cudaStream_t)stream);
    }
    if (B > 0 && (!x || !drop || !h_out || !h_parity || !aligned16(x) || !aligned16(h_out) ||
                  !aligned16(h_parity) || (x_parity && !aligned16(x_parity)))) {
        set_error("invalid pointer argument"); return CI_ERR_INVALID_ARG;
    }
    WsLayout L = ws_layout(m, k, B);
    ci_status_t r = check_ws(L, ws, ws_bytes);
    if (r != CI_OK) return r;
    if (B == 0) return CI_OK;
    float* lp[4];
    int32_t* bp[4];
    head_ptrs(m, B * (int64_t)k, logits, labels, lp, bp);
    return serve_impl(m, mode, k, B, x, drop, h_out, h_parity, x_parity, lp, bp, ws, L, (cudaStream_t)stream);
}

// --- general (n, k) codes (f3) ------------------------------------------------------------
static bool general_args_ok(int32_t k, int32_t r, int64_t B) {
    return k >= 1 && r >= 1 && k + r <= 32 && B >= 0;
}

ci_status_t ci_workspace_size_general(const ci_model_t* model, int32_t k, int32_t r, int64_t B, size_t* bytes) {
    const Model* m = reinterpret_cast<const Model*>(model);
    if (!m || !bytes || !general_args_ok(k, r, B)) { set_error("invalid argument"); return CI_ERR_INVALID_ARG; }
    *bytes = ws_layout(m, k, B, true, r).total;
    return CI_OK;
}

ci_status_t ci_encode_general(const ci_model_t* model, int32_t k, int32_t r, int64_t B, const float* coef,
                              const float* h, float* x_parity, float* comb_out, void* ws, size_t ws_bytes,
                              ci_stream_t stream) {
    CI_MODEL_OR_FAIL(m, model);
    if (!general_args_ok(k, r, B) || (B > 0 && (!coef || !h || !x_parity || !aligned16(h) || !aligned16(x_parity) ||
                                                 (comb_out && !aligned16(comb_out))))) {
        set_error("invalid argument"); return CI_ERR_INVALID_ARG;
    }
    WsLayout L = ws_layout(m, k, B, true, r);
    ci_status_t st_ = check_ws(L, ws, ws_bytes);
    if (st_ != CI_OK) return st_;
    if (B == 0) return CI_OK;
    cudaStream_t st = (cudaStream_t)stream;
    CI_CUDA(zero_ctrs(ws, L, st));
    float* comb = comb_out ? comb_out : at<float>(ws, L.mean);
    CI_CUDA(launch_combine_general(h, coef, comb, k, r, B, m->d, st));
    return inverse_impl(m, comb, x_parity, B * r, ws, L, st);
}

ci_status_t ci_decode_general(int32_t k, int32_t r, int64_t B, int64_t d, const float* coef, float* h,
                              const float* h_parity, const uint32_t* avail, void* ws, size_t ws_bytes,
                              ci_stream_t stream) {
    if (!general_args_ok(k, r, B) || d < 0 || (B > 0 && (!coef || !h || !h_parity || !avail))) {
        set_error("invalid argument"); return CI_ERR_INVALID_ARG;
    }
    if (!ws || ws_bytes < 256 || !aligned16(ws)) { set_error("workspace too small"); return CI_ERR_WORKSPACE; }
    CI_CUDA(launch_decode_general(h, h_parity, coef, avail, k, r, B, d, reinterpret_cast<int*>(ws),
                                  (cudaStream_t)stream));
    return CI_OK;
}

ci_status_t ci_serve_general(const ci_model_t* model, int32_t k, int32_t r, int64_t B, const float* coef,
                             const float* x, const uint32_t* avail, float* h_out, float* h_parity,
                             float* x_parity, float* logits, int32_t* labels, void* ws, size_t ws_bytes,
                             ci_stream_t stream) {
    CI_MODEL_OR_FAIL(m, model);
    if (!general_args_ok(k, r, B) ||
        (B > 0 && (!coef || !x || !avail || !h_out || !h_parity || !aligned16(x) || !aligned16(h_out) ||
                   !aligned16(h_parity) || (x_parity && !aligned16(x_parity))))) {
        set_error("invalid argument"); return CI_ERR_INVALID_ARG;
    }
    WsLayout L = ws_layout(m, k, B, true, r);
    ci_status_t rc = check_ws(L, ws, ws_bytes);
    if (rc != CI_OK) return rc;
    if (B == 0) return CI_OK;
    cudaStream_t st = (cudaStream_t)stream;
    CI_CUDA(zero_ctrs(ws, L, st));
    const int64_t n = B * (int64_t)k;
    float* comb = at<float>(ws, L.mean);
    float* xp = x_parity ? x_parity : at<float>(ws, L.xp);
    rc = forward_impl(m, x, h_out, n, ws, L, st);                                // h on main queries
    if (rc != CI_OK) return rc;
    CI_CUDA(launch_combine_general(h_out, coef, comb, k, r, B, m->d, st));          // r weighted sums
    rc = inverse_impl(m, comb, xp, B * r, ws, L, st);                             // ... through h^-1
    if (rc != CI_OK) return rc;
    rc = forward_impl(m, xp, h_parity, B * r, ws, L, st);                         // h on parity queries
    if (rc != CI_OK) return rc;
    CI_CUDA(launch_decode_general(h_out, h_parity, coef, avail, k, r, B, m->d, at<int>(ws, L.flag), st));
    float* lp[4];
    int32_t* bp[4];
    head_ptrs(m, n, logits, labels, lp, bp);
    for (int t = 0; t < m->arch.n_heads; t++) {
        if (!lp[t] && !bp[t]) continue;
        const float* W = m->d_head[t];
        const float* b = W + (int64_t)m->arch.head_classes[t] * m->d;
        CI_CUDA(launch_classify(h_out, n, m->d, W, b, m->arch.head_classes[t], lp[t], bp[t], st));
    }
    return CI_OK;
}

// --- host-buffer variant -----------------------------------------------------------------
// The B groups are served in nc chunks so that PCIe traffic overlaps compute: chunk c's
// inputs go up on a copy stream, its compute runs on the caller's stream (even c) or a
// second compute stream (odd c, own device workspace), and its outputs come back on a
// third stream while later chunks compute.  Layout: dev workspace 0 (first, so ci_check
// sees its flag) | dev workspace 1 | x | drop | h | p | logits | labels (full size).
static constexpr int kMaxChunks = 8;

// chunks per call: a lone synchronous call overlaps its own copies with compute (4 chunks); async
// calls overlap with each other, so fewer, more efficient chunks (2) win (measured, bench e2e)
static int host_chunks(int64_t B, bool async_call) {
    static const int env = getenv("CI_HOST_CHUNKS") ? atoi(getenv("CI_HOST_CHUNKS")) : 0;
    int nc = env > 0 ? env : (B >= 512 ? (async_call ? 2 : 4) : B >= 64 ? 2 : 1);
    nc = std::min(nc, kMaxChunks);
    return (int)std::max<int64_t>(1, std::min<int64_t>(nc, B));
}

struct HostLayout {
    WsLayout dev;                 // per-chunk device workspace (chunk of Bc groups)
    int nc = 1;
    int64_t Bc = 0;
    size_t dev1 = 0, x = 0, drop = 0, h = 0, p = 0, logits = 0, labels = 0, total = 0;
};

static HostLayout host_layout(const Model* m, int32_t k, int64_t B, bool async_call) {
    HostLayout H;
    H.nc = host_chunks(B, async_call);
    H.Bc = (B + H.nc - 1) / H.nc;
    H.dev = ws_layout(m, k, H.Bc);
    int64_t n = B * (int64_t)k;
    int64_t ncls = 0;
    for (int t = 0; t < m->arch.n_heads; t++) ncls += m->arch.head_classes[t];
    size_t off = H.dev.total;
    H.dev1 = off; off += H.nc > 1 ? H.dev.total : 0;
    H.x = off; off += up(sizeof(float) * (size_t)(n * m->din));
    H.drop = off; off += up(sizeof(int32_t) * (size_t)B);
    H.h = off; off += up(sizeof(float) * (size_t)(n * m->d));
    H.p = off; off += up(sizeof(float) * (size_t)(B * m->d));
    H.logits = off; off += up(sizeof(float) * (size_t)(n * ncls));
    H.labels = off; off += up(sizeof(int32_t) * (size_t)(n * m->arch.n_heads));
    H.total = off;
    return H;
}

}  // extern "C"

namespace ci {
struct HostPipe {
    std::mutex mu;
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
    cudaEvent_t start = nullptr, fin = nullptr, in[kMaxChunks] = {}, done[kMaxChunks] = {};
};

static ci_status_t host_pipe(Model* m, HostPipe** out) {
    static std::mutex create_mu;
    std::lock_guard<std::mutex> g(create_mu);
    if (!m->host_pipe) {
        HostPipe* P = new HostPipe();
        const unsigned fl = cudaStreamNonBlocking;
        CI_CUDA(cudaStreamCreateWithFlags(&P->h2d, fl));
        CI_CUDA(cudaStreamCreateWithFlags(&P->comp, fl));
        CI_CUDA(cudaStreamCreateWithFlags(&P->d2h, fl));
        CI_CUDA(cudaEventCreateWithFlags(&P->start, cudaEventDisableTiming));
        CI_CUDA(cudaEventCreateWithFlags(&P->fin, cudaEventDisableTiming));
        for (int c = 0; c < kMaxChunks; c++) {
            CI_CUDA(cudaEventCreateWithFlags(&P->in[c], cudaEventDisableTiming));
            CI_CUDA(cudaEventCreateWithFlags(&P->done[c], cudaEventDisableTiming));
        }
        m->host_pipe = P;
    }
    *out = reinterpret_cast<HostPipe*>(m->host_pipe);
    return CI_OK;
}

void release_host_pipe(Model* m) {
    HostPipe* P = reinterpret_cast<HostPipe*>(m->host_pipe);
    if (!P) return;
    cudaStreamDestroy(P->h2d); cudaStreamDestroy(P->comp); cudaStreamDestroy(P->d2h);
    cudaEventDestroy(P->start); cudaEventDestroy(P->fin);
    for (int c = 0; c < kMaxChunks; c++) { cudaEventDestroy(P->in[c]); cudaEventDestroy(P->done[c]); }
    delete P;
    m->host_pipe = nullptr;
}
}  // namespace ci

extern "C" {

ci_status_t ci_workspace_size_host(const ci_model_t* model, int32_t k, int64_t B, size_t* bytes) {
    const Model* m = reinterpret_cast<const Model*>(model);
    if (!m || !bytes || k < 1 || B < 0) { set_error("invalid argument"); return CI_ERR_INVALID_ARG; }
    *bytes = std::max(host_layout(m, k, B, false).total, host_layout(m, k, B, true).total);
    return CI_OK;
}

}  // extern "C"

namespace ci {
// fold workspace 1's drop-error count into workspace 0's flag (read by ci_check)
__global__ void k_fold_flag(int* f0, int* f1) {
    if (threadIdx.x < 2 && f1[threadIdx.x]) { f0[threadIdx.x] += f1[threadIdx.x]; f1[threadIdx.x] = 0; }
}
}  // namespace ci

extern "C" {

static ci_status_t serve_host_impl(const ci_model_t* model, ci_encode_mode_t mode, int32_t k,
                                   int64_t B, const float* x_host, const int32_t* drop_host,
                                   float* h_out_host, float* h_parity_host, float* logits_host,
                                   int32_t* labels_host, void* ws, size_t ws_bytes,
                                   ci_stream_t stream, bool sync) {
    CI_MODEL_OR_FAIL(m, model);
    if (mode != CI_ENC_EXACT && mode != CI_ENC_LEARNED) { set_error("unknown encode mode"); return CI_ERR_INVALID_ARG; }
    if (mode == CI_ENC_LEARNED && m->enc_off < 0) { set_error("model has no learned encoder"); return CI_ERR_UNSUPPORTED; }
    if (k < 1 || B < 0 || (B > 0 && (!x_host || !drop_host))) { set_error("invalid argument"); return CI_ERR_INVALID_ARG; }
    HostLayout H = host_layout(m, k, B, !sync);
    if (!ws || !aligned16(ws) || ws_bytes < H.total) {
        set_error("host workspace %zu bytes; need %zu", ws_bytes, H.total); return CI_ERR_WORKSPACE;
    }
    if (B == 0) return CI_OK;
    HostPipe* P = nullptr;
    ci_status_t r = host_pipe(const_cast<Model*>(m), &P);
    if (r != CI_OK) return r;
    std::lock_guard<std::mutex> g(P->mu);
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = B * (int64_t)k, d = m->d, din = m->din;
    const int nh = m->arch.n_heads;
    float* dx = at<float>(ws, H.x);
    int32_t* ddrop = at<int32_t>(ws, H.drop);
    float* dh = at<float>(ws, H.h);
    float* dp = at<float>(ws, H.p);
    float* dl = at<float>(ws, H.logits);
    int32_t* dlab = at<int32_t>(ws, H.labels);
    float *dlp[4], *hlp[4];
    int32_t *dbp[4], *hbp[4];
    head_ptrs(m, n, dl, dlab, dlp, dbp);
    head_ptrs(m, n, logits_host, labels_host, hlp, hbp);
    CI_CUDA(cudaEventRecord(P->start, st));
    CI_CUDA(cudaStreamWaitEvent(P->h2d, P->start, 0));
    for (int c = 0; c < H.nc; c++) {
        const int64_t b0 = c * H.Bc, nb = std::min<int64_t>(H.Bc, B - b0);
        if (nb <= 0) break;
        const int64_t q0 = b0 * k, nq = nb * k;
        CI_CUDA(cudaMemcpyAsync(dx + q0 * din, x_host + q0 * din, sizeof(float) * nq * din, cudaMemcpyHostToDevice, P->h2d));
        CI_CUDA(cudaMemcpyAsync(ddrop + b0, drop_host + b0, sizeof(int32_t) * nb, cudaMemcpyHostToDevice, P->h2d));
        CI_CUDA(cudaEventRecord(P->in[c], P->h2d));
        cudaStream_t cs = (c & 1) ? P->comp : st;
        void* wsc = (c & 1) ? at<char>(ws, H.dev1) : ws;
        CI_CUDA(cudaStreamWaitEvent(cs, P->in[c], 0));
        float* clp[4];
        int32_t* cbp[4];
        for (int t = 0; t < 4; t++) {
            const int64_t C = t < nh ? m->arch.head_classes[t] : 0;
            clp[t] = dlp[t] ? dlp[t] + q0 * C : nullptr;
            cbp[t] = dbp[t] ? dbp[t] + q0 : nullptr;
        }
        r = serve_impl(m, mode, k, nb, dx + q0 * din, ddrop + b0, dh + q0 * d, dp + b0 * d, nullptr, clp, cbp,
                       wsc, H.dev, cs);
        if (r != CI_OK) return r;
        CI_CUDA(cudaEventRecord(P->done[c], cs));
        CI_CUDA(cudaStreamWaitEvent(P->d2h, P->done[c], 0));
        if (h_out_host)
            CI_CUDA(cudaMemcpyAsync(h_out_host + q0 * d, dh + q0 * d, sizeof(float) * nq * d, cudaMemcpyDeviceToHost, P->d2h));
        if (h_parity_host)
            CI_CUDA(cudaMemcpyAsync(h_parity_host + b0 * d, dp + b0 * d, sizeof(float) * nb * d, cudaMemcpyDeviceToHost, P->d2h));
        for (int t = 0; t < nh; t++) {
            const int64_t C = m->arch.head_classes[t];
            if (hlp[t] && C)
                CI_CUDA(cudaMemcpyAsync(hlp[t] + q0 * C, clp[t], sizeof(float) * nq * C, cudaMemcpyDeviceToHost, P->d2h));
            if (hbp[t])
                CI_CUDA(cudaMemcpyAsync(hbp[t] + q0, cbp[t], sizeof(int32_t) * nq, cudaMemcpyDeviceToHost, P->d2h));
        }
    }
    CI_CUDA(cudaEventRecord(P->fin, P->d2h));
    CI_CUDA(cudaStreamWaitEvent(st, P->fin, 0));
    if (H.nc > 1) {   // workspace 1's drop-error count -> workspace 0's flag (ci_check)
        ci::k_fold_flag<<<1, 32, 0, st>>>(reinterpret_cast<int*>(ws), at<int>(ws, H.dev1));
        count_launch();
        CI_CUDA(cudaGetLastError());
    }
    if (sync) CI_CUDA(cudaStreamSynchronize(st));
    return CI_OK;
}

ci_status_t ci_serve_group_host(const ci_model_t* model, ci_encode_mode_t mode, int32_t k,
                                int64_t B, const float* x_host, const int32_t* drop_host,
                                float* h_out_host, float* h_parity_host, float* logits_host,
                                int32_t* labels_host, void* ws, size_t ws_bytes,
                                ci_stream_t stream) {
    return serve_host_impl(model, mode, k, B, x_host, drop_host, h_out_host, h_parity_host, logits_host,
                           labels_host, ws, ws_bytes, stream, true);
}

ci_status_t ci_serve_group_host_async(const ci_model_t* model, ci_encode_mode_t mode, int32_t k,
                                      int64_t B, const float* x_host, const int32_t* drop_host,
                                      float* h_out_host, float* h_parity_host, float* logits_host,
                                      int32_t* labels_host, void* ws, size_t ws_bytes,
                                      ci_stream_t stream) {
    return serve_host_impl(model, mode, k, B, x_host, drop_host, h_out_host, h_parity_host, logits_host,
                           labels_host, ws, ws_bytes, stream, false);
}

ci_status_t ci_test_mean(int32_t k, int64_t B, int64_t d, const float* h, float* m, ci_stream_t stream) {
    if (k < 1 || B < 0 || d < 0 || (B > 0 && (!h || !m))) { set_error("invalid argument"); return CI_ERR_INVALID_ARG; }
    CI_CUDA(launch_mean(h, m, k, B, d, (cudaStream_t)stream));
    return CI_OK;
}

int64_t ci_test_launch_count(int32_t reset) {
    long long v = reset ? g_launches.exchange(0) : g_launches.load();
    return (int64_t)v;
}

// --- first-k gated serving harness (f2) --------------------------------------------------
// Workspace: (k+1) per-worker device workspaces for one-group calls | per in-flight slot: FkSlot,
// worker results [k+1][d], estimates [k][d], x_p [din] | head pointer / class tables.
struct FkLayout {
    WsLayout w;          // one worker's workspace (B = 1 group)
    size_t wstride = 0, slots = 0, sstride = 0, tables = 0, total = 0;
};
static FkLayout fk_layout(const Model* m, int32_t k, int32_t S) {
    FkLayout F;
    F.w = ws_layout(m, k, 1);
    F.wstride = up(F.w.total);
    F.slots = F.wstride * (size_t)(k + 1);
    F.sstride = up(sizeof(FkSlot)) + up(sizeof(float) * (size_t)((2 * k + 1) * m->d)) + up(sizeof(float) * (size_t)m->din);
    F.tables = F.slots + F.sstride * (size_t)S;
    F.total = F.tables + up(4 * sizeof(void*) + 4 * sizeof(int));
    return F;
}

ci_status_t ci_workspace_size_first_k(const ci_model_t* model, int32_t k, int32_t max_inflight, size_t* bytes) {
    const Model* m = reinterpret_cast<const Model*>(model);
    if (!m || !bytes || k < 1 || k > 30 || max_inflight < 1 || max_inflight > 256) {
        set_error("invalid argument"); return CI_ERR_INVALID_ARG;
    }
    *bytes = fk_layout(m, k, max_inflight).total;
    return CI_OK;
}

ci_status_t ci_serve_first_k(const ci_model_t* model, ci_firstk_mode_t mode, int32_t k, int64_t Q, const float* x,
                             const int32_t* straggler, int64_t delay_ns, int32_t max_inflight, float* features,
                             float* logits, int32_t* labels, int64_t* records, void* ws, size_t ws_bytes,
                             ci_stream_t stream) {
    CI_MODEL_OR_FAIL(m, model);
    if ((mode != CI_FIRSTK_CODED && mode != CI_FIRSTK_UNCODED) || k < 1 || k > 30 || Q < 0 || delay_ns < 0 ||
        max_inflight < 1 || max_inflight > 256 || m->d % 4 ||
        (Q > 0 && (!x || !straggler || !features || !records || !aligned16(x) || !aligned16(features) ||
                   (m->arch.n_heads > 0 && (!logits || !labels))))) {
        set_error("invalid argument"); return CI_ERR_INVALID_ARG;
    }
    if (mode == CI_FIRSTK_CODED && m->enc_off < 0) {
        set_error("coded first-k serving needs the learned encoder (the parity worker encodes from the raw "
                  "queries, PAPER.md:667)");
        return CI_ERR_UNSUPPORTED;
    }
    for (int64_t q = 0; q < Q; q++)
        if (straggler[q] < -1 || straggler[q] >= k) { set_error("straggler[%lld] out of range", (long long)q); return CI_ERR_INVALID_ARG; }
    {   // every worker / delay stream needs its own hardware queue: with shared queues a delayed
        // worker's wait falsely blocks unrelated streams (measured: 30 ms stalls in other queries)
        const char* env = getenv("CUDA_DEVICE_MAX_CONNECTIONS");
        const int need = k + 2 + max_inflight, have = env ? atoi(env) : 8;
        if (need > 32 || have < need) {
            set_error("first-k serving needs CUDA_DEVICE_MAX_CONNECTIONS >= k + 2 + max_inflight = %d (<= 32) set "
                      "before the CUDA context is created (have %d)", need, have);
            return CI_ERR_UNSUPPORTED;
        }
    }
    const int S = max_inflight;
    FkLayout F = fk_layout(m, k, S);
    if (!ws || !aligned16(ws) || ws_bytes < F.total) {
        set_error("workspace %zu bytes; need %zu", ws_bytes, F.total); return CI_ERR_WORKSPACE;
    }
    if (Q == 0) return CI_OK;
    cudaStream_t front = (cudaStream_t)stream;
    const int nw = mode == CI_FIRSTK_CODED ? k + 1 : k;   // the uncoded arm has no parity worker
    const int64_t d = m->d, din = m->din;
    // head tables (device): weight pointers and class counts
    const float** hw = at<const float*>(ws, F.tables);
    int* hc = reinterpret_cast<int*>(hw + 4);
    {
        const float* hp[4] = {m->d_head[0], m->d_head[1], m->d_head[2], m->d_head[3]};
        int cc[4] = {0, 0, 0, 0};
        for (int t = 0; t < m->arch.n_heads; t++) cc[t] = m->arch.head_classes[t];
        CI_CUDA(cudaMemcpyAsync(hw, hp, sizeof(hp), cudaMemcpyHostToDevice, front));
        CI_CUDA(cudaMemcpyAsync(hc, cc, sizeof(cc), cudaMemcpyHostToDevice, front));
        CI_CUDA(cudaStreamSynchronize(front));
    }
    std::vector<cudaStream_t> wst(nw), dst(S);
    std::vector<cudaEvent_t> esub(S), eall(S), ework((size_t)S * nw);
    ci_status_t rc = CI_OK;
    auto cleanup = [&]() {
        for (auto sv : wst) if (sv) cudaStreamDestroy(sv);
        for (auto sv : dst) if (sv) cudaStreamDestroy(sv);
        for (auto ev : esub) if (ev) cudaEventDestroy(ev);
        for (auto ev : eall) if (ev) cudaEventDestroy(ev);
        for (auto ev : ework) if (ev) cudaEventDestroy(ev);
    };
#define FK_CUDA(call)                                                   \
    do {                                                                \
        cudaError_t e_ = (call);                                        \
        if (e_ != cudaSuccess) { rc = cuda_status(e_, #call); cleanup(); return rc; } \
    } while (0)
#define FK_OK(call)                                                     \
    do {                                                                \
        rc = (call);                                                    \
        if (rc != CI_OK) { cleanup(); return rc; }                      \
    } while (0)
    for (auto& sv : wst) FK_CUDA(cudaStreamCreateWithFlags(&sv, cudaStreamNonBlocking));
    for (auto& sv : dst) FK_CUDA(cudaStreamCreateWithFlags(&sv, cudaStreamNonBlocking));
    for (auto& ev : esub) FK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    for (auto& ev : eall) FK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    for (auto& ev : ework) FK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    FK_CUDA(cudaEventRecord(esub[0], front));   // workers start after the caller's prior work
    for (int w = 0; w < nw; w++) FK_CUDA(cudaStreamWaitEvent(wst[w], esub[0], 0));
    for (int64_t q = 0; q < Q; q++) {
        const int s_ = (int)(q % S);
        if (q >= S) FK_CUDA(cudaEventSynchronize(eall[s_]));   // slot s_ free: its last query fully done
        char* sb = at<char>(ws, F.slots + F.sstride * (size_t)s_);
        FkSlot* slot = reinterpret_cast<FkSlot*>(sb);
        float* hres = reinterpret_cast<float*>(sb + up(sizeof(FkSlot)));   // [k+1][d] worker results
        float* est = hres + (size_t)(k + 1) * d;                              // [k][d]
        float* xp = reinterpret_cast<float*>(sb + up(sizeof(FkSlot)) + up(sizeof(float) * (size_t)((2 * k + 1) * d)));
        FK_CUDA(launch_fk_submit(slot, est, (int64_t)k * d, q, front));
        FK_CUDA(cudaEventRecord(esub[s_], front));
        for (int w = 0; w < nw; w++) {
            cudaStream_t st = wst[w];
            void* wsw = at<char>(ws, F.wstride * (size_t)w);
            FK_CUDA(cudaStreamWaitEvent(st, esub[s_], 0));
            FK_CUDA(zero_ctrs(wsw, F.w, st));
            float* res = hres + (size_t)w * d;
            if (w < k) {
                FK_OK(forward_impl(m, x + (q * k + w) * din, res, 1, wsw, F.w, st));     // main worker w
            } else {
                FK_OK(encode_learned_impl(m, x + q * k * din, xp, k, 1, wsw, F.w, st));  // parity worker:
                FK_OK(forward_impl(m, xp, res, 1, wsw, F.w, st));                        // Enc, then f
            }
            cudaStream_t ast = st;
            if (w == straggler[q]) {   // its result reaches the decoder delay_ns late
                FK_CUDA(cudaEventRecord(ework[(size_t)s_ * nw + w], st));
                ast = dst[s_];
                FK_CUDA(cudaStreamWaitEvent(ast, ework[(size_t)s_ * nw + w], 0));
                FK_CUDA(launch_fk_delay(delay_ns, ast));
            }
            FK_CUDA(launch_fk_arrive(slot, est, res, w, k, d, mode == CI_FIRSTK_UNCODED, hw, hc, m->arch.n_heads,
                                     features, logits, labels, Q, records, ast));
            FK_CUDA(cudaEventRecord(ework[(size_t)s_ * nw + w], ast));
        }
        for (int w = 0; w < nw; w++) FK_CUDA(cudaStreamWaitEvent(dst[s_], ework[(size_t)s_ * nw + w], 0));
        FK_CUDA(cudaEventRecord(eall[s_], dst[s_]));
    }
    for (int s2 = 0; s2 < S; s2++) FK_CUDA(cudaStreamWaitEvent(front, eall[s2], 0));
    FK_CUDA(cudaStreamSynchronize(front));   // the harness owns its streams: finish before destroying them
    cleanup();
#undef FK_CUDA
#undef FK_OK
    return CI_OK;
}

ci_status_t ci_make_drops(int32_t k, int64_t B, uint64_t seed, int32_t* drop, ci_stream_t stream) {
    if (k < 1 || B < 0 || (B > 0 && !drop)) { set_error("invalid argument"); return CI_ERR_INVALID_ARG; }
    CI_CUDA(launch_make_drops(k, B, seed, drop, (cudaStream_t)stream));
    return CI_OK;
}

}  // extern "C"
