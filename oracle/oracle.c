/*
 * oracle.c -- plain, slow, obviously-correct f64 CPU oracle for the Coded-InvNet
 * hot path (arXiv 2106.06445).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2106_06445_b200/) never links or calls it, and this file shares no code,
 * header, table or constant with the CUDA path.
 *
 * Everything is direct nested loops over NCHW arrays in double precision.  Inputs
 * and parameters arrive as fp32 (the seeded fixtures) and are promoted exactly.
 *
 * What is computed, with the passage each step follows:
 *   psi / psi^-1 .......... invertible space-to-depth r=2 of i-RevNet
 *                           (PAPER.md:168, 393 footnote, 555; SURVEY Q4 channel
 *                           order out[c*4+2dy+dx][y][x] = in[c][2y+dy][2x+dx])
 *   conv3x3 ............... cross-correlation, zero padding 1, stride 1, bias
 *                           ("blocks of 3x3 convolutions",
 *                           BASELINE.json north_star)
 *   F = conv -> act -> conv (SURVEY Q3 reading; act = ReLU, ELU or identity)
 *   additive coupling ..... s_B += F(s_A) / s_A += F(s_B), inverse by subtraction
 *                           in reverse order (i-RevNet)
 *   i-ResNet residual ..... y = x + G(x), G = conv -> ELU -> conv on the whole state;
 *                           inverse by the fixed-point iteration x <- y - G(x) from
 *                           x_0 = y, which converges geometrically when Lip(G) < 1
 *                           ("invert a residual block with an
 *                           exponential convergence rate via fixed-point iteration",
 *                           393, 408, 441 "solving fixed point equations"; stopping
 *                           rule of SPEC.md:123, 147: step <= 1e-12 or 200 iterations,
 *                           or a stated fixed count)
 *   h, h^-1 ............... stages of [psi, blocks]; no injective padding so h is
 *                           dimension preserving
 *   exact encode .......... m_b = (1/k) sum_i h(x_{b,i}); x_p = h^-1(m_b)
 *                           (PAPER.md:125-127, 135, 241 c_{1,j}=1/k, 259)
 *   decode ................ f^(x_a) = k f(x_{k+1}) - sum_{i!=a} f(x_i)
 *                           (PAPER.md:273-276, 471 Eq. decode with the Q9 reading,
 *                           934-936 App. C)
 *   classify .............. linear heads g_t(z) = W_t z + b_t, label = first argmax
 *
 *   learned encode ........ light encoder with a weight-shared first layer on each of the k
 *                           inputs, averaged after that layer (reading
 *                           Q13), then a small U-Net-style tail:
 *                             e_i = ReLU(conv(E1, x_i)); m = (1/k) sum_i e_i; z = psi(m);
 *                             z = ReLU(conv(E2, z)); z = ReLU(conv(E3, z));
 *                             u = psi^-1(z) + m; x_p = conv(E4, u)     (SURVEY §8a Arch E)
 *
 * Parity pins: see tests/test_oracle_pins.py (every function here is pinned; none
 * is "parity unpinned").
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int in_c, in_h, in_w;
    int n_stages;
    int squeeze[4];
    int n_blocks[4];
    int mid[4];
    int act;          /* 0 = ReLU, 2 = identity */
    int first_orient; /* 0: block 0 updates s_B, 1: block 0 updates s_A */
    int n_heads;
    int head_classes[4];
    int enc_c1, enc_mid; /* learned encoder widths; 0 = no encoder */
    int block_kind;      /* 0 = additive coupling on half the state, 1 = i-ResNet residual */
    int fp_iters;        /* residual inverse: fixed-point iterations per block; 0 = until
                            the step is <= 1e-12 (max 200) */
} or_arch_t;

/* ------------------------------------------------------------------------ */
/* shapes and parameter offsets (canonical flat layout, see fixtures)        */
/* ------------------------------------------------------------------------ */
static void stage_shape(const or_arch_t* a, int s, int* C, int* H, int* W) {
    int c = a->in_c, h = a->in_h, w = a->in_w;
    for (int i = 0; i <= s; i++)
        if (a->squeeze[i]) { c *= 4; h /= 2; w /= 2; }
    *C = c; *H = h; *W = w;
}

long oracle_d(const or_arch_t* a) {
    int C, H, W;
    stage_shape(a, a->n_stages - 1, &C, &H, &W);
    return (long)C * H * W;
}

/* offset of block (s,t)'s W1 in the flat vector */
static long block_offset(const or_arch_t* a, int s_target, int t_target) {
    long off = 0;
    for (int s = 0; s < a->n_stages; s++) {
        int C, H, W;
        stage_shape(a, s, &C, &H, &W);
        long c = a->block_kind ? C : C / 2, m = a->mid[s];
        long per = m * c * 9 + m + c * m * 9 + c;
        for (int t = 0; t < a->n_blocks[s]; t++) {
            if (s == s_target && t == t_target) return off;
            off += per;
        }
    }
    return off; /* == start of heads when called with (n_stages, 0) */
}

static long head_offset(const or_arch_t* a, int head) {
    long off = block_offset(a, a->n_stages, 0);
    long d = oracle_d(a);
    for (int i = 0; i < head; i++) off += (long)a->head_classes[i] * d + a->head_classes[i];
    return off;
}

/* ------------------------------------------------------------------------ */
/* psi (space-to-depth, r = 2) and its inverse                               */
/* ------------------------------------------------------------------------ */
void oracle_psi(const double* in, int C, int H, int W, double* out) {
    int Ho = H / 2, Wo = W / 2;
    for (int c = 0; c < C; c++)
        for (int dy = 0; dy < 2; dy++)
            for (int dx = 0; dx < 2; dx++)
                for (int y = 0; y < Ho; y++)
                    for (int x = 0; x < Wo; x++)
                        out[(((long)(c * 4 + 2 * dy + dx)) * Ho + y) * Wo + x] =
                            in[((long)c * H + 2 * y + dy) * W + 2 * x + dx];
}

void oracle_psi_inv(const double* in, int C4, int Ho, int Wo, double* out) {
    int C = C4 / 4, H = Ho * 2, W = Wo * 2;
    for (int c = 0; c < C; c++)
        for (int dy = 0; dy < 2; dy++)
            for (int dx = 0; dx < 2; dx++)
                for (int y = 0; y < Ho; y++)
                    for (int x = 0; x < Wo; x++)
                        out[((long)c * H + 2 * y + dy) * W + 2 * x + dx] =
                            in[(((long)(c * 4 + 2 * dy + dx)) * Ho + y) * Wo + x];
}

/* ------------------------------------------------------------------------ */
/* conv3x3: y[o][i][j] = b[o] + sum_c sum_{u,v in -1..1} W[o][c][u+1][v+1] x[c][i+u][j+v] */
/* ------------------------------------------------------------------------ */
void oracle_conv3x3(const double* x, int Cin, int H, int W, const float* Wt, const float* b,
                    int Cout, double* y) {
    for (int o = 0; o < Cout; o++)
        for (int i = 0; i < H; i++)
            for (int j = 0; j < W; j++) {
                double acc = (double)b[o];
                for (int c = 0; c < Cin; c++)
                    for (int u = -1; u <= 1; u++)
                        for (int v = -1; v <= 1; v++) {
                            int ii = i + u, jj = j + v;
                            if (ii < 0 || ii >= H || jj < 0 || jj >= W) continue;
                            acc += (double)Wt[(((long)o * Cin + c) * 3 + (u + 1)) * 3 + (v + 1)] *
                                   x[((long)c * H + ii) * W + jj];
                        }
                y[((long)o * H + i) * W + j] = acc;
            }
}

/* F(z) = conv3x3(W2, b2, act(conv3x3(W1, b1, z)))   (z: [c][H][W] -> out: [c][H][W]) */
static void coupling_F(const or_arch_t* a, const float* blk, int c, int m, int H, int W,
                       const double* z, double* hid, double* out) {
    const float* W1 = blk;
    const float* b1 = W1 + (long)m * c * 9;
    const float* W2 = b1 + m;
    const float* b2 = W2 + (long)c * m * 9;
    oracle_conv3x3(z, c, H, W, W1, b1, m, hid);
    long n = (long)m * H * W;
    if (a->act == 0) {
        for (long i = 0; i < n; i++) hid[i] = hid[i] > 0.0 ? hid[i] : 0.0;
    } else if (a->act == 1) {   /* ELU(z) = z for z > 0, exp(z) - 1 otherwise (1-Lipschitz) */
        for (long i = 0; i < n; i++) hid[i] = hid[i] > 0.0 ? hid[i] : expm1(hid[i]);
    }
    oracle_conv3x3(hid, m, H, W, W2, b2, c, out);
}

/* Inverse of one residual block y = x + G(x) by x <- y - G(x) from x_0 = y
 * (PAPER.md:169).  iters > 0: exactly that many updates; iters == 0: until
 * max|x_{i+1} - x_i| <= 1e-12 or 200 updates.  Returns the number of
 * updates.  ybuf, tmp: [C][H][W]; hid: [m][H][W]. */
int oracle_residual_inverse_block(const or_arch_t* a, const float* blk, int C, int m, int H, int W,
                                  const double* y, double* x, int iters, double* tmp, double* hid) {
    long n = (long)C * H * W;
    memcpy(x, y, sizeof(double) * n);
    int it = 0;
    for (;;) {
        if (iters > 0 && it == iters) break;
        coupling_F(a, blk, C, m, H, W, x, hid, tmp);
        double step = 0.0;
        for (long i = 0; i < n; i++) {
            double xn = y[i] - tmp[i];
            double dlt = fabs(xn - x[i]);
            if (dlt > step) step = dlt;
            x[i] = xn;
        }
        it++;
        if (iters == 0 && (step <= 1e-12 || it == 200)) break;
    }
    return it;
}

/* ------------------------------------------------------------------------ */
/* h and h^-1 on one image                                                   */
/* ------------------------------------------------------------------------ */
static long max_elems(const or_arch_t* a) {
    long mx = (long)a->in_c * a->in_h * a->in_w;
    for (int s = 0; s < a->n_stages; s++) {
        int C, H, W;
        stage_shape(a, s, &C, &H, &W);
        long e1 = (long)C * H * W, e2 = (long)a->mid[s] * H * W;
        if (e1 > mx) mx = e1;
        if (e2 > mx) mx = e2;
    }
    return mx;
}

/* x: [in_c][in_h][in_w] -> h: [d] (NCHW flatten of the final state) */
static void forward_one(const or_arch_t* a, const float* params, const double* x, double* hout,
                        double* buf /* 4 * max_elems */) {
    long mx = max_elems(a);
    double* s = buf;          /* state */
    double* tmp = buf + mx;   /* psi scratch / F output */
    double* hid = buf + 2 * mx;
    int C = a->in_c, H = a->in_h, W = a->in_w;
    memcpy(s, x, sizeof(double) * C * H * W);
    for (int st = 0; st < a->n_stages; st++) {
        if (a->squeeze[st]) {
            oracle_psi(s, C, H, W, tmp);
            C *= 4; H /= 2; W /= 2;
            memcpy(s, tmp, sizeof(double) * C * H * W);
        }
        int c = C / 2, m = a->mid[st];
        long half = (long)c * H * W;
        if (a->block_kind == 1) {   /* i-ResNet: s <- s + G(s) */
            long n = (long)C * H * W;
            for (int t = 0; t < a->n_blocks[st]; t++) {
                coupling_F(a, params + block_offset(a, st, t), C, m, H, W, s, hid, tmp);
                for (long i = 0; i < n; i++) s[i] += tmp[i];
            }
            continue;
        }
        for (int t = 0; t < a->n_blocks[st]; t++) {
            const float* blk = params + block_offset(a, st, t);
            int orient = (a->first_orient + t) & 1;
            double* src = orient == 0 ? s : s + half;        /* s_A or s_B */
            double* dst = orient == 0 ? s + half : s;        /* updated half */
            coupling_F(a, blk, c, m, H, W, src, hid, tmp);
            for (long i = 0; i < half; i++) dst[i] += tmp[i];
        }
    }
    memcpy(hout, s, sizeof(double) * C * H * W);
}

/* h: [d] -> x: [in_c][in_h][in_w]; exact reverse of forward_one */
static void inverse_one(const or_arch_t* a, const float* params, const double* hin, double* xout,
                        double* buf) {
    long mx = max_elems(a);
    double* s = buf;
    double* tmp = buf + mx;
    double* hid = buf + 2 * mx;
    int C, H, W;
    stage_shape(a, a->n_stages - 1, &C, &H, &W);
    memcpy(s, hin, sizeof(double) * C * H * W);
    for (int st = a->n_stages - 1; st >= 0; st--) {
        int c = C / 2, m = a->mid[st];
        long half = (long)c * H * W;
        if (a->block_kind == 1) {   /* i-ResNet: blocks reversed, each by fixed point */
            double* y = buf + 3 * mx;
            for (int t = a->n_blocks[st] - 1; t >= 0; t--) {
                memcpy(y, s, sizeof(double) * C * H * W);
                oracle_residual_inverse_block(a, params + block_offset(a, st, t), C, m, H, W, y, s,
                                              a->fp_iters, tmp, hid);
            }
        } else
        for (int t = a->n_blocks[st] - 1; t >= 0; t--) {
            const float* blk = params + block_offset(a, st, t);
            int orient = (a->first_orient + t) & 1;
            double* src = orient == 0 ? s : s + half;
            double* dst = orient == 0 ? s + half : s;
            coupling_F(a, blk, c, m, H, W, src, hid, tmp);
            for (long i = 0; i < half; i++) dst[i] -= tmp[i];
        }
        if (a->squeeze[st]) {
            oracle_psi_inv(s, C, H, W, tmp);
            C /= 4; H *= 2; W *= 2;
            memcpy(s, tmp, sizeof(double) * C * H * W);
        }
    }
    memcpy(xout, s, sizeof(double) * C * H * W);
}

/* ------------------------------------------------------------------------ */
/* parallel drivers (std pthreads, static split over images)                 */
/* ------------------------------------------------------------------------ */
typedef struct {
    const or_arch_t* a;
    const float* params;
    const double* in;
    double* out;
    long lo, hi, in_stride, out_stride;
    int inverse;
} job_t;

static void* run_job(void* p) {
    job_t* j = (job_t*)p;
    long mx = max_elems(j->a);
    double* buf = (double*)malloc(sizeof(double) * 4 * mx);
    for (long i = j->lo; i < j->hi; i++) {
        if (j->inverse)
            inverse_one(j->a, j->params, j->in + i * j->in_stride, j->out + i * j->out_stride, buf);
        else
            forward_one(j->a, j->params, j->in + i * j->in_stride, j->out + i * j->out_stride, buf);
    }
    free(buf);
    return NULL;
}

static void run_parallel(const or_arch_t* a, const float* params, long n, const double* in,
                         long in_stride, double* out, long out_stride, int inverse, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > n) nthreads = (int)(n > 0 ? n : 1);
    pthread_t th[256];
    job_t jobs[256];
    if (nthreads > 256) nthreads = 256;
    for (int t = 0; t < nthreads; t++) {
        jobs[t].a = a; jobs[t].params = params; jobs[t].in = in; jobs[t].out = out;
        jobs[t].lo = n * t / nthreads; jobs[t].hi = n * (t + 1) / nthreads;
        jobs[t].in_stride = in_stride; jobs[t].out_stride = out_stride; jobs[t].inverse = inverse;
        pthread_create(&th[t], NULL, run_job, &jobs[t]);
    }
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
}

/* h on n images: x [n][in_c][in_h][in_w] (f64) -> h [n][d] */
int oracle_forward_h(const or_arch_t* a, const float* params, long n, const double* x, double* h,
                     int nthreads) {
    long din = (long)a->in_c * a->in_h * a->in_w;
    run_parallel(a, params, n, x, din, h, oracle_d(a), 0, nthreads);
    return 0;
}

/* h^-1 on n vectors: h [n][d] -> x [n][in_c][in_h][in_w] */
int oracle_inverse_h(const or_arch_t* a, const float* params, long n, const double* h, double* x,
                     int nthreads) {
    long din = (long)a->in_c * a->in_h * a->in_w;
    run_parallel(a, params, n, h, oracle_d(a), x, din, 1, nthreads);
    return 0;
}

/* m_b = (sum_{i=0}^{k-1} H[b][i]) / k      (c_{1,j} = 1/k) */
void oracle_mean(int k, long B, long d, const double* Hf, double* m) {
    for (long b = 0; b < B; b++)
        for (long e = 0; e < d; e++) {
            double acc = 0.0;
            for (int i = 0; i < k; i++) acc += Hf[((long)b * k + i) * d + e];
            m[b * d + e] = acc / (double)k;
        }
}

/* R[b][j] = k P[b] - sum_{i != j} H[b][i] for j = drop[b] >= 0; other slots copy H.
 * (PAPER.md:275 f^(x_a) = k f(x_{k+1}) - sum_{i != a} f(x_i)) */
void oracle_decode(int k, long B, long d, const double* Hf, const double* P, const int* drop,
                   double* R) {
    for (long b = 0; b < B; b++) {
        int j = drop[b];
        for (int i = 0; i < k; i++) {
            double* r = R + ((long)b * k + i) * d;
            const double* hsrc = Hf + ((long)b * k + i) * d;
            if (i != j) { memcpy(r, hsrc, sizeof(double) * d); continue; }
            for (long e = 0; e < d; e++) {
                double acc = 0.0;
                for (int q = 0; q < k; q++)
                    if (q != j) acc += Hf[((long)b * k + q) * d + e];
                r[e] = (double)k * P[b * d + e] - acc;
            }
        }
    }
}

/* logits[n][C] = W z + b ; labels[n] = smallest index attaining the max */
void oracle_classify(const or_arch_t* a, const float* params, int head, long n, const double* z,
                     double* logits, int* labels) {
    long d = oracle_d(a);
    int C = a->head_classes[head];
    const float* Wg = params + head_offset(a, head);
    const float* bg = Wg + (long)C * d;
    for (long r = 0; r < n; r++) {
        int best = 0;
        double bestv = 0.0;
        for (int c = 0; c < C; c++) {
            double acc = (double)bg[c];
            for (long e = 0; e < d; e++) acc += (double)Wg[(long)c * d + e] * z[r * d + e];
            logits[r * C + c] = acc;
            if (c == 0 || acc > bestv) { bestv = acc; best = c; }
        }
        if (labels) labels[r] = best;
    }
}

static long encoder_offset(const or_arch_t* a) {
    long off = head_offset(a, a->n_heads);
    return off;
}

/* Learned encoder on one group: x [k][in_c][H][W] (f64) -> xp [in_c][H][W] */
static void encode_one(const or_arch_t* a, const float* params, int k, const double* x, double* xp) {
    const int ci = a->in_c, H = a->in_h, W = a->in_w, c1 = a->enc_c1, mid = a->enc_mid;
    const long HW = (long)H * W, hw4 = HW / 4;
    const float* E1W = params + encoder_offset(a);
    const float* E1b = E1W + (long)c1 * ci * 9;
    const float* E2W = E1b + c1;
    const float* E2b = E2W + (long)mid * 4 * c1 * 9;
    const float* E3W = E2b + mid;
    const float* E3b = E3W + (long)4 * c1 * mid * 9;
    const float* E4W = E3b + 4 * c1;
    const float* E4b = E4W + (long)ci * c1 * 9;
    double* e = (double*)malloc(sizeof(double) * c1 * HW);
    double* m = (double*)calloc((size_t)c1 * HW, sizeof(double));
    double* z = (double*)malloc(sizeof(double) * 4 * c1 * hw4);
    double* z2 = (double*)malloc(sizeof(double) * (mid > 4 * c1 ? mid : 4 * c1) * hw4);
    double* u = (double*)malloc(sizeof(double) * c1 * HW);
    for (int i = 0; i < k; i++) {                       /* weight-shared first layer */
        oracle_conv3x3(x + (long)i * ci * HW, ci, H, W, E1W, E1b, c1, e);
        for (long q = 0; q < c1 * HW; q++) m[q] += e[q] > 0.0 ? e[q] : 0.0;
    }
    for (long q = 0; q < c1 * HW; q++) m[q] /= (double)k; /* average after the first layer */
    oracle_psi(m, c1, H, W, z);                          /* [4c1][H/2][W/2] */
    oracle_conv3x3(z, 4 * c1, H / 2, W / 2, E2W, E2b, mid, z2);
    for (long q = 0; q < mid * hw4; q++) z2[q] = z2[q] > 0.0 ? z2[q] : 0.0;
    oracle_conv3x3(z2, mid, H / 2, W / 2, E3W, E3b, 4 * c1, z);
    for (long q = 0; q < 4 * c1 * hw4; q++) z[q] = z[q] > 0.0 ? z[q] : 0.0;
    oracle_psi_inv(z, 4 * c1, H / 2, W / 2, u);          /* [c1][H][W] */
    for (long q = 0; q < c1 * HW; q++) u[q] += m[q];    /* skip connection */
    oracle_conv3x3(u, c1, H, W, E4W, E4b, ci, xp);
    free(e); free(m); free(z); free(z2); free(u);
}

typedef struct {
    const or_arch_t* a;
    const float* params;
    int k;
    const double* x;
    double* xp;
    long lo, hi;
} enc_job_t;

static void* run_enc(void* p) {
    enc_job_t* j = (enc_job_t*)p;
    long din = (long)j->a->in_c * j->a->in_h * j->a->in_w;
    for (long b = j->lo; b < j->hi; b++) encode_one(j->a, j->params, j->k, j->x + b * j->k * din, j->xp + b * din);
    return NULL;
}

/* Learned encode of B groups: x [B][k][in_c][H][W] (f64) -> x_parity [B][in_c][H][W] */
int oracle_encode_learned(const or_arch_t* a, const float* params, int k, long B, const double* x,
                          double* xp, int nthreads) {
    if (a->enc_c1 <= 0) return -1;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > B) nthreads = (int)(B > 0 ? B : 1);
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    enc_job_t jobs[256];
    for (int t = 0; t < nthreads; t++) {
        jobs[t].a = a; jobs[t].params = params; jobs[t].k = k; jobs[t].x = x; jobs[t].xp = xp;
        jobs[t].lo = B * t / nthreads; jobs[t].hi = B * (t + 1) / nthreads;
        pthread_create(&th[t], NULL, run_enc, &jobs[t]);
    }
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    return 0;
}

/* Whole coded path for B groups of k queries (exact encode, n = k + 1):
 *   H  = h(x)                         [B][k][d]
 *   m  = mean_i H                     [B][d]
 *   xp = h^-1(m)                      [B][in_c][in_h][in_w]
 *   P  = h(xp)                        [B][d]
 *   R  = decode(H, P, drop)           [B][k][d]
 *   logits[t] = g_t(R), labels[t]     [n_heads][B][k][C_t]   (degraded slots decoded)
 *   logits_n[t] = g_t(H), labels_n[t] (normal mode, no loss)
 * Outputs for heads are packed head after head with each head's own class count. */
int oracle_serve_group(const or_arch_t* a, const float* params, int k, long B, const float* x,
                       const int* drop, double* Hf, double* m, double* xp, double* P, double* R,
                       double* logits, int* labels, double* logits_n, int* labels_n,
                       int nthreads, int learned) {
    long din = (long)a->in_c * a->in_h * a->in_w, d = oracle_d(a);
    long n = B * k;
    double* xd = (double*)malloc(sizeof(double) * n * din);
    for (long i = 0; i < n * din; i++) xd[i] = (double)x[i];
    oracle_forward_h(a, params, n, xd, Hf, nthreads);
    oracle_mean(k, B, d, Hf, m);
    if (learned) oracle_encode_learned(a, params, k, B, xd, xp, nthreads);  /* Enc(x_1..x_k) */
    else oracle_inverse_h(a, params, B, m, xp, nthreads);                   /* h^-1(mean h) */
    free(xd);
    oracle_forward_h(a, params, B, xp, P, nthreads);
    oracle_decode(k, B, d, Hf, P, drop, R);
    long lo = 0, lab = 0;
    for (int t = 0; t < a->n_heads; t++) {
        if (logits) oracle_classify(a, params, t, n, R, logits + lo, labels ? labels + lab : NULL);
        if (logits_n)
            oracle_classify(a, params, t, n, Hf, logits_n + lo, labels_n ? labels_n + lab : NULL);
        lo += n * a->head_classes[t];
        lab += n;
    }
    return 0;
}
