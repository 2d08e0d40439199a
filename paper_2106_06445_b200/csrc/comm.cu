// Worker-partitioned coded serving (config C5): one process
// per worker, k main workers + 1 parity worker, exchanging features through a symmetric
// "window" of device memory that every rank maps (CUDA IPC: NVLink P2P loads between GPUs; the
// same code runs with several ranks on one GPU, which is how it is tested).
//
// The two exchange steps are fused compute + collective kernels over peer memory:
//   X2 (exact encode)  k_peer_mean   : the parity rank reads the k main ranks' published h(x_i)
//                                      and writes m = (sum_i h_i) / k  (== k_mean bit for bit)
//   X4 (decode, K11)   k_peer_decode : rank p reads every rank's features for its partition of
//                                      the groups and writes k P - sum_{i != j} h_i (== k_decode)
// Synchronisation: each window starts with two epoch counters (pub: my features of call e are
// in the window; done: I finished reading every peer's window for call e).  A rank publishes
// call e only after every peer is done with call e-1; consumers wait for pub >= e.  Counters
// are written by a one-thread kernel after the producing kernel (stream order) with
// st.release.sys and polled with ld.acquire.sys; a wait that exceeds ~20 s traps (a peer that
// never arrives is a deadlock, reported as a launch failure instead of a hung GPU).
//
// Bootstrap (host): ci_comm_unique_id names a POSIX shared-memory rendezvous on this node;
// ci_comm_create exchanges the windows' IPC handles through it (single node: the scope of this
// library's multi-GPU path, 8 GPUs of one box).
#include <errno.h>
#include <fcntl.h>
#include <stdio.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include "ci_internal.h"
#include "codedinv_testing.h"

namespace ci {

// ------------------------------------------------------------------------------------------
// device side
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// thread 0 of the block polls counter `which` of ranks [q0, q1) until >= e; the block waits
__device__ void wait_ranks(void* const* peers, int q0, int q1, int which, uint64_t e) {
    if (threadIdx.x == 0) {
        for (int q = q0; q < q1; q++) {
            const uint64_t* f = reinterpret_cast<const uint64_t*>(peers[q]) + which;
            unsigned long long n = 0;
            while (ld_acquire_sys(f) < e) {
                __nanosleep(512);
                if (++n > (1ull << 25)) __trap();   // ~20 s: a peer never arrived
            }
        }
    }
    __syncthreads();
}

__device__ __forceinline__ const float4* feat_of(void* const* peers, int q) {
    return reinterpret_cast<const float4*>(reinterpret_cast<const char*>(peers[q]) + kCommHeader);
}

__global__ void k_signal(uint64_t* flag, uint64_t e) {
    __threadfence_system();
    st_release_sys(flag, e);
}

// window feat <- src after every peer is done with the previous call
__global__ void k_publish(void* const* peers, int rank, int nranks, uint64_t e, const float4* __restrict__ src,
                          int64_t total4) {
    if (e > 1) wait_ranks(peers, 0, nranks, kCommDone, e - 1);
    float4* dst = const_cast<float4*>(feat_of(peers, rank));
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total4; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

// X2: m[b] = (sum_{i<k, ascending} h_i[b]) / k from the k main ranks' windows
__global__ void k_peer_mean(void* const* peers, int k, uint64_t e, int64_t total4, float4* __restrict__ m) {
    wait_ranks(peers, 0, k, kCommPub, e);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int q = 0; q < k; q++) {
            const float4 v = feat_of(peers, q)[i];
            acc.x = __fadd_rn(acc.x, v.x); acc.y = __fadd_rn(acc.y, v.y);
            acc.z = __fadd_rn(acc.z, v.z); acc.w = __fadd_rn(acc.w, v.w);
        }
        const float fk = (float)k;
        m[i] = make_float4(__fdiv_rn(acc.x, fk), __fdiv_rn(acc.y, fk), __fdiv_rn(acc.z, fk), __fdiv_rn(acc.w, fk));
    }
}

// X4 / K11: decoded features of groups [b0, b0 + nb): out[b - b0] = k P[b] - sum_{i != j} h_i[b]
// (ascending i, one fma: == k_decode); drop = -1 -> zeros; other out-of-range drops -> zeros + flag
__global__ void k_peer_decode(void* const* peers, int k, int nranks, uint64_t e, const int32_t* __restrict__ drop,
                              int64_t b0, int64_t nb, int64_t d4, float4* __restrict__ out, int* __restrict__ flag) {
    wait_ranks(peers, 0, nranks, kCommPub, e);
    const float fk = (float)k;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < nb * d4;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t bl = idx / d4, c = idx - bl * d4, g = (b0 + bl) * d4 + c;
        const int j = __ldg(drop + b0 + bl);
        if (j < 0 || j >= k) {
            if (j != -1 && c == 0) atomicAdd(flag, 1);
            out[idx] = make_float4(0.f, 0.f, 0.f, 0.f);
            continue;
        }
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int q = 0; q < k; q++) {
            if (q == j) continue;
            const float4 v = feat_of(peers, q)[g];
            acc.x = __fadd_rn(acc.x, v.x); acc.y = __fadd_rn(acc.y, v.y);
            acc.z = __fadd_rn(acc.z, v.z); acc.w = __fadd_rn(acc.w, v.w);
        }
        const float4 p = feat_of(peers, k)[g];
        out[idx] = make_float4(__fmaf_rn(fk, p.x, -acc.x), __fmaf_rn(fk, p.y, -acc.y), __fmaf_rn(fk, p.z, -acc.z),
                               __fmaf_rn(fk, p.w, -acc.w));
    }
}

static int grid_of(int64_t total, int block) {
    int64_t g = (total + block - 1) / block, cap = 148 * (2048 / block) * 4;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, cap));
}

ci_status_t comm_publish(Comm* c, const float* src, int64_t B, cudaStream_t st) {
    const int64_t total4 = B * c->d / 4;
    k_publish<<<grid_of(total4, 256), 256, 0, st>>>(c->d_peers, c->rank, c->nranks, c->epoch, (const float4*)src,
                                                     total4);
    count_launch();
    CI_CHECK_LAUNCH("k_publish");
    k_signal<<<1, 1, 0, st>>>(reinterpret_cast<uint64_t*>(c->win) + kCommPub, c->epoch);
    count_launch();
    CI_CHECK_LAUNCH("k_signal");
    return CI_OK;
}

ci_status_t comm_peer_mean(Comm* c, int k, int64_t B, float* mean, cudaStream_t st) {
    const int64_t total4 = B * c->d / 4;
    k_peer_mean<<<grid_of(total4, 256), 256, 0, st>>>(c->d_peers, k, c->epoch, total4, (float4*)mean);
    count_launch();
    CI_CHECK_LAUNCH("k_peer_mean");
    return CI_OK;
}

ci_status_t comm_peer_decode(Comm* c, int k, int64_t B, const int32_t* drop, float* out, int* flag,
                             cudaStream_t st) {
    const int64_t Bp = (B + c->nranks - 1) / c->nranks;
    const int64_t b0 = std::min<int64_t>(B, (int64_t)c->rank * Bp), nb = std::min<int64_t>(B, b0 + Bp) - b0;
    const int64_t d4 = c->d / 4;
    if (nb > 0) {
        k_peer_decode<<<grid_of(nb * d4, 256), 256, 0, st>>>(c->d_peers, k, c->nranks, c->epoch, drop, b0, nb, d4,
                                                              (float4*)out, flag);
        count_launch();
        CI_CHECK_LAUNCH("k_peer_decode");
    }
    k_signal<<<1, 1, 0, st>>>(reinterpret_cast<uint64_t*>(c->win) + kCommDone, c->epoch);
    count_launch();
    CI_CHECK_LAUNCH("k_signal");
    return CI_OK;
}

// ------------------------------------------------------------------------------------------
// host side: rendezvous and window mapping
// ------------------------------------------------------------------------------------------
namespace {
constexpr uint32_t kMagic = 0x43494331u;   // "CIC1"
struct RvSlot {
    cudaIpcMemHandle_t handle;
    int32_t device, pid;
    int32_t ready;
    int32_t pad;
};
struct RvHeader {
    uint32_t magic;
    int32_t nranks;
    int32_t pad[2];
};

void shm_name_of(const uint8_t id[CI_COMM_ID_BYTES], char* out, size_t n) {
    static const char* hex = "0123456789abcdef";
    size_t p = (size_t)snprintf(out, n, "/codedinv_");
    for (int i = 0; i < 16 && p + 2 < n; i++) {
        out[p++] = hex[id[i] >> 4];
        out[p++] = hex[id[i] & 15];
    }
    out[p] = 0;
}

double now_s() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}
}  // namespace

// Host rendezvous of nranks processes through POSIX shared memory named by `id`: every rank
// publishes `payload` (<= 64 bytes) in its slot and receives everyone's (out: nranks x 64 B).
ci_status_t rendezvous(const uint8_t id[CI_COMM_ID_BYTES], int nranks, int rank, const void* payload, size_t bytes,
                       void* out, double timeout_s) {
    if (bytes > sizeof(cudaIpcMemHandle_t)) { set_error("rendezvous payload too large"); return CI_ERR_INVALID_ARG; }
    char name[64];
    shm_name_of(id, name, sizeof(name));
    const size_t size = sizeof(RvHeader) + (size_t)nranks * sizeof(RvSlot);
    int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
    if (fd < 0) { set_error("shm_open(%s): %s", name, strerror(errno)); return CI_ERR_COMM; }
    if (ftruncate(fd, (off_t)size) != 0) {
        close(fd);
        set_error("ftruncate(%s): %s", name, strerror(errno));
        return CI_ERR_COMM;
    }
    void* mem = mmap(nullptr, size, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (mem == MAP_FAILED) { set_error("mmap(%s): %s", name, strerror(errno)); return CI_ERR_COMM; }
    RvHeader* hdr = reinterpret_cast<RvHeader*>(mem);
    RvSlot* slots = reinterpret_cast<RvSlot*>(hdr + 1);
    __atomic_store_n(&hdr->magic, kMagic, __ATOMIC_SEQ_CST);
    __atomic_store_n(&hdr->nranks, nranks, __ATOMIC_SEQ_CST);
    memcpy(&slots[rank].handle, payload, bytes);
    slots[rank].pid = (int32_t)getpid();
    __atomic_store_n(&slots[rank].ready, 1, __ATOMIC_SEQ_CST);
    const double t0 = now_s();
    ci_status_t st = CI_OK;
    for (int q = 0; q < nranks && st == CI_OK; q++) {
        while (!__atomic_load_n(&slots[q].ready, __ATOMIC_SEQ_CST)) {
            if (now_s() - t0 > timeout_s) {
                set_error("rendezvous %s: rank %d did not arrive within %.0f s", name, q, timeout_s);
                st = CI_ERR_COMM;
                break;
            }
            usleep(200);
        }
    }
    if (st == CI_OK) {
        for (int q = 0; q < nranks; q++) memcpy((char*)out + (size_t)q * 64, &slots[q].handle, bytes);
        if (__atomic_load_n(&hdr->nranks, __ATOMIC_SEQ_CST) != nranks) {
            set_error("rendezvous %s: ranks disagree on nranks", name);
            st = CI_ERR_COMM;
        }
    }
    munmap(mem, size);
    // every rank has opened and filled the segment once all slots are ready: the name can go
    if (st == CI_OK) shm_unlink(name);
    return st;
}

}  // namespace ci

using namespace ci;

extern "C" {

ci_status_t ci_comm_unique_id(uint8_t out[CI_COMM_ID_BYTES]) {
    if (!out) { set_error("NULL id buffer"); return CI_ERR_INVALID_ARG; }
    memset(out, 0, CI_COMM_ID_BYTES);
    int fd = open("/dev/urandom", O_RDONLY);
    if (fd < 0 || read(fd, out, 16) != 16) {
        if (fd >= 0) close(fd);
        set_error("/dev/urandom: %s", strerror(errno));
        return CI_ERR_COMM;
    }
    close(fd);
    return CI_OK;
}

ci_status_t ci_comm_create(const uint8_t id[CI_COMM_ID_BYTES], int32_t nranks, int32_t rank, ci_layout_t layout,
                           int64_t max_B, int64_t d, int device, ci_comm_t** out) {
    if (!id || !out || nranks < 2 || nranks > kCommMaxRanks || rank < 0 || rank >= nranks ||
        (layout != CI_SHARD_GROUPS && layout != CI_SHARD_WORKERS) || max_B < 1 || d < 4 || d % 4) {
        set_error("invalid communicator arguments");
        return CI_ERR_INVALID_ARG;
    }
    *out = nullptr;
    CI_CUDA(cudaSetDevice(device));
    Comm* c = new Comm();
    c->nranks = nranks; c->rank = rank; c->layout = layout; c->device = device; c->cap_B = max_B; c->d = d;
    const size_t bytes = kCommHeader + (size_t)max_B * (size_t)d * sizeof(float);
    cudaError_t e = cudaMalloc(&c->win, bytes);
    if (e == cudaSuccess) e = cudaMemset(c->win, 0, bytes);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaIpcMemHandle_t mine;
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&mine, c->win);
    if (e != cudaSuccess) { cudaFree(c->win); delete c; return cuda_status(e, "ci_comm_create window"); }
    std::vector<uint8_t> all((size_t)nranks * 64);
    ci_status_t st = rendezvous(id, nranks, rank, &mine, sizeof(mine), all.data(), 120.0);
    if (st != CI_OK) { cudaFree(c->win); delete c; return st; }
    for (int q = 0; q < nranks && e == cudaSuccess; q++) {
        if (q == rank) { c->peers[q] = c->win; continue; }
        cudaIpcMemHandle_t h;
        memcpy(&h, all.data() + (size_t)q * 64, sizeof(h));
        e = cudaIpcOpenMemHandle(&c->peers[q], h, cudaIpcMemLazyEnablePeerAccess);
        if (e == cudaSuccess) c->opened[q] = true;
    }
    if (e == cudaSuccess) e = cudaMalloc(&c->d_peers, sizeof(void*) * nranks);
    if (e == cudaSuccess) e = cudaMemcpy(c->d_peers, c->peers, sizeof(void*) * nranks, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        ci_comm_destroy(reinterpret_cast<ci_comm_t*>(c));
        return cuda_status(e, "ci_comm_create peers");
    }
    *out = reinterpret_cast<ci_comm_t*>(c);
    return CI_OK;
}

void ci_comm_destroy(ci_comm_t* comm) {
    Comm* c = reinterpret_cast<Comm*>(comm);
    if (!c) return;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (int q = 0; q < c->nranks; q++)
        if (c->opened[q]) cudaIpcCloseMemHandle(c->peers[q]);
    if (c->d_peers) cudaFree(c->d_peers);
    if (c->win) cudaFree(c->win);
    delete c;
}

ci_status_t ci_test_rendezvous(const uint8_t id[CI_COMM_ID_BYTES], int32_t nranks, int32_t rank, const uint8_t* payload,
                               int32_t bytes, uint8_t* out) {
    if (!id || !payload || !out || nranks < 1 || rank < 0 || rank >= nranks || bytes < 0 || bytes > 64) {
        set_error("invalid argument");
        return CI_ERR_INVALID_ARG;
    }
    return rendezvous(id, nranks, rank, payload, (size_t)bytes, out, 60.0);
}

}  // extern "C"
