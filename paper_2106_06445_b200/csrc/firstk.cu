// First-k gated serving with online decoding ("randomly add artificial latencies
// of 0.1 s to one of the k workers", App. C).
//
// Device side of ci_serve_first_k (orchestration in api.cu): every worker (k mains + the parity
// worker, each on its own CUDA stream) ends its task with k_arrive, one CTA that takes the
// query slot's lock and applies the App. C update for its result (reading R-f2a):
//   main j :  f^(x_j) = f(x_j) (final);  f^(x_i) -= f(x_j) for every unfinalised i != j
//   parity :  f^(x_i) += k f(x_{k+1})    for every unfinalised i
// The event that brings the k-th distinct result (coded) -- or the k-th main result (uncoded
// arm: no parity worker) -- completes the query: it runs the linear heads on the k recovered
// features inside the same CTA, copies them out and stamps the device globaltimer.  Events
// after completion only record their arrival (they change nothing).
#include "ci_internal.h"

namespace ci {

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_fk_submit(FkSlot* slot, float* est, int64_t nest, int64_t q) {
    // clear the slot's estimates (zero before the first event, App. C) and state, stamp submit
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nest; i += (int64_t)gridDim.x * blockDim.x)
        est[i] = 0.f;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        slot->recv = 0; slot->fin = 0; slot->complete = 0; slot->lock = 0; slot->q = q;
        slot->t_submit = gtimer();
    }
}

// the straggler: its result is delivered delay_ns late (the artificial latency of PAPER.md:669)
__global__ void k_fk_delay(int64_t delay_ns) {
    const uint64_t t0 = gtimer();
    while ((int64_t)(gtimer() - t0) < delay_ns) __nanosleep(20000);
}

// one completion event: task j (< k main, == k parity) with result v [d] of query slot `slot`
__global__ void __launch_bounds__(256) k_fk_arrive(FkSlot* slot, float* __restrict__ est, const float* __restrict__ v,
                                                   int j, int k, int64_t d, int need_mains, const float* const* heads_w,
                                                   const int* head_c, int n_heads, float* feat_out, float* logits,
                                                   int32_t* labels, int64_t Q, int64_t* rec) {
    __shared__ int s_apply, s_done;
    __shared__ uint32_t s_fin;
    __shared__ uint64_t s_t0;
    const int tid = threadIdx.x;
    if (tid == 0) {
        while (atomicCAS(&slot->lock, 0, 1) != 0) __nanosleep(64);
        __threadfence();
        s_t0 = gtimer();
        const uint32_t R = *((volatile uint32_t*)&slot->recv);
        const int complete = *((volatile int*)&slot->complete);
        s_apply = !complete && !((R >> j) & 1u);
        s_fin = *((volatile uint32_t*)&slot->fin);
        const uint32_t R2 = R | (1u << j);
        const int have = need_mains ? __popc(R2 & ((1u << k) - 1u)) : __popc(R2);
        s_done = s_apply && have == k;
        slot->recv = R2;
    }
    __syncthreads();
    const int apply = s_apply, done = s_done;
    const uint32_t F = s_fin;
    if (apply) {
        const float fk = (float)k;
        const int64_t d4 = d / 4;
        const float4* v4 = reinterpret_cast<const float4*>(v);
        float4* e4 = reinterpret_cast<float4*>(est);
        for (int64_t c = tid; c < d4; c += blockDim.x) {
            const float4 x = v4[c];
            for (int i = 0; i < k; i++) {
                if ((F >> i) & 1u) continue;
                float4 t = __ldcg(&e4[i * d4 + c]);   // written by other CTAs under the slot lock: L2
                if (j < k) {
                    if (i == j) t = x;
                    else { t.x = __fsub_rn(t.x, x.x); t.y = __fsub_rn(t.y, x.y); t.z = __fsub_rn(t.z, x.z); t.w = __fsub_rn(t.w, x.w); }
                } else {
                    t.x = __fmaf_rn(fk, x.x, t.x); t.y = __fmaf_rn(fk, x.y, t.y);
                    t.z = __fmaf_rn(fk, x.z, t.z); t.w = __fmaf_rn(fk, x.w, t.w);
                }
                __stcg(&e4[i * d4 + c], t);
            }
        }
    }
    __syncthreads();
    uint64_t t_upd = 0;
    if (done) {
        if (tid == 0) t_upd = gtimer();
        // the k recovered features out, then the heads: one warp per (slot, class) dot product
        const int64_t d4 = d / 4;
        const int64_t q = slot->q;
        const float4* e4 = reinterpret_cast<const float4*>(est);
        float4* o4 = reinterpret_cast<float4*>(feat_out + q * k * d);
        for (int64_t c = tid; c < (int64_t)k * d4; c += blockDim.x) o4[c] = __ldcg(&e4[c]);
        const int warp = tid >> 5, lane = tid & 31;
        int64_t lo = 0;
        for (int t = 0; t < n_heads; t++) {
            const int C = head_c[t];
            const float4* W4 = reinterpret_cast<const float4*>(heads_w[t]);
            const float* bias = heads_w[t] + (int64_t)C * d;
            float* lg = logits + lo + q * k * C;
            for (int p = warp; p < k * C; p += blockDim.x / 32) {
                const int i = p / C, cl = p % C;
                float acc = 0.f;
                for (int64_t c = lane; c < d4; c += 32) {
                    const float4 a = __ldcg(&e4[i * d4 + c]), w = __ldg(&W4[cl * d4 + c]);
                    acc = fmaf(a.x, w.x, acc); acc = fmaf(a.y, w.y, acc);
                    acc = fmaf(a.z, w.z, acc); acc = fmaf(a.w, w.w, acc);
                }
                for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (lane == 0) lg[i * C + cl] = acc + bias[cl];
            }
            __syncthreads();
            for (int i = tid; i < k; i += blockDim.x) {   // first index attaining the max
                int best = 0;
                for (int cl = 1; cl < C; cl++)
                    if (lg[i * C + cl] > lg[i * C + best]) best = cl;
                labels[(int64_t)t * Q * k + q * k + i] = best;
            }
            lo += Q * k * C;
        }
        __syncthreads();
    }
    if (tid == 0) {
        if (apply) {
            uint32_t Fn = F;
            if (j < k) Fn |= 1u << j;
            if (done) Fn = (1u << k) - 1u;
            slot->fin = Fn;
        }
        if (done) {
            const uint64_t t2 = gtimer();
            slot->complete = 1;
            const int64_t q = slot->q;
            const uint32_t R = slot->recv;
            rec[q * 4 + 0] = (int64_t)(t2 - slot->t_submit);   // latency: submit -> predictions
            rec[q * 4 + 1] = (int64_t)(t_upd - s_t0);          // the completing event's online update
            rec[q * 4 + 2] = (int64_t)(t2 - t_upd);            // heads on the k recovered features
            const int degraded = (R >> k) & 1u && __popc(R & ((1u << k) - 1u)) < k;
            rec[q * 4 + 3] = (int64_t)R | ((int64_t)degraded << 32);
        }
        __threadfence();
        atomicExch(&slot->lock, 0);
    }
}

cudaError_t launch_fk_submit(FkSlot* slot, float* est, int64_t nest, int64_t q, cudaStream_t s) {
    k_fk_submit<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((nest + 255) / 256, 64)), 256, 0, s>>>(slot, est,
                                                                                                        nest, q);
    count_launch();
    return cudaGetLastError();
}
cudaError_t launch_fk_delay(int64_t delay_ns, cudaStream_t s) {
    k_fk_delay<<<1, 1, 0, s>>>(delay_ns);
    count_launch();
    return cudaGetLastError();
}
cudaError_t launch_fk_arrive(FkSlot* slot, float* est, const float* v, int j, int k, int64_t d, int need_mains,
                             const float* const* heads_w, const int* head_c, int n_heads, float* feat_out,
                             float* logits, int32_t* labels, int64_t Q, int64_t* rec, cudaStream_t s) {
    k_fk_arrive<<<1, 256, 0, s>>>(slot, est, v, j, k, d, need_mains, heads_w, head_c, n_heads, feat_out, logits,
                                  labels, Q, rec);
    count_launch();
    return cudaGetLastError();
}

}  // namespace ci
