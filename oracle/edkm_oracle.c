/*
 * edkm_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, dense fp64 CPU implementation of DKM as eDKM uses it
 * (arXiv 2309.00964).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product
 * path (paper_2309_00964_b200/) never imports, links or executes it, and this
 * file shares no code, header, table or constant with the CUDA path.
 *
 * Citations are to /root/reference/PAPER.md lines ("P:77 S2.2" = line 77,
 * section 2.2) and to DESIGN.md "Readings" R1..R16 where the paper is silent.
 * The paper never writes the DKM formulas (P:39 defers to DKM [3]);
 * the forward below is the north star's statement of them: attention
 * softmax(-|w-c|^2/tau) over k = 2^b centroids, soft-centroid update,
 * W~ = A.C, unrolled iterations (R1-R6).
 *
 * Every function is a direct transcription of its definition:
 *   - the attention map is evaluated weight by weight over ALL |W| x |C|
 *     entries ("O(|W||C|)"), recomputed rather than stored;
 *   - sums are plain fp64 loops.  Threads split the weights into contiguous
 *     chunks whose partial sums are added in chunk order, so results are
 *     deterministic for a given thread count.  No blocking, fusion or
 *     reordering beyond that.
 *
 * Pins (tests/test_oracle.py): brute-force histogram + Fig. 3 example;
 * decode vs numpy/torch; attention rows sum to 1; tau->0 equals textbook
 * Lloyd k-means; tau->inf and k=1 closed forms; scale law; permutation
 * invariance; backward vs torch fp64 autograd of an independently written
 * graph and vs central finite differences; table form vs dense form;
 * hard assignment vs brute force; the eps > 0 stop (R4) against textbook
 * Lloyd k-means in exact rational arithmetic at tau = 1e-9.  Parity is pinned
 * for every function.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define ORACLE_MAX_K 256
#define ORACLE_MAX_THREADS 256

/* ------------------------------------------------------------------------ */
/* 16-bit decoding: IEEE-754 binary16 and bfloat16 (upper half of binary32).  */
/* P:77 "16bit (e.g., BF16 or FP16)".                                         */
/* ------------------------------------------------------------------------ */
static double decode_bf16(uint16_t b) {
    /* bfloat16 = sign(1) exponent(8, bias 127) fraction(7) */
    int sign = (b >> 15) & 1, e = (b >> 7) & 0xFF, f = b & 0x7F;
    double mag;
    if (e == 0xFF) mag = (f == 0) ? INFINITY : NAN;
    else if (e == 0) mag = ldexp((double)f, -126 - 7);            /* subnormal */
    else mag = ldexp((double)(128 + f), e - 127 - 7);
    return sign ? -mag : mag;
}

static double decode_fp16(uint16_t b) {
    /* binary16 = sign(1) exponent(5, bias 15) fraction(10) */
    int sign = (b >> 15) & 1, e = (b >> 10) & 0x1F, f = b & 0x3FF;
    double mag;
    if (e == 0x1F) mag = (f == 0) ? INFINITY : NAN;
    else if (e == 0) mag = ldexp((double)f, -14 - 10);            /* subnormal */
    else mag = ldexp((double)(1024 + f), e - 15 - 10);
    return sign ? -mag : mag;
}

/* dtype: 0 = bf16, 1 = fp16.  Returns 0, or -1 on a bad dtype. */
int oracle_decode16(const uint16_t* bits, int64_t n, int dtype, double* out) {
    if (dtype != 0 && dtype != 1) return -1;
    for (int64_t i = 0; i < n; ++i) out[i] = dtype == 0 ? decode_bf16(bits[i]) : decode_fp16(bits[i]);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Uniquification (Fig. 3): the index of weight i is its */
/* 16-bit pattern itself, and the attention table has one row per pattern.  */
/* counts[u] = #{i : bits(w_i) = u}, u in [0, 65536).                         */
/* ------------------------------------------------------------------------ */
void oracle_histogram(const uint16_t* bits, int64_t n, int64_t* counts) {
    for (int u = 0; u < 65536; ++u) counts[u] = 0;
    for (int64_t i = 0; i < n; ++i) counts[bits[i]] += 1;
}

/* ------------------------------------------------------------------------ */
/* DKM attention of one weight to all centroids (north star; R1):  */
/*   A[j] = exp(-(w - C[j])^2 / tau) / sum_l exp(-(w - C[l])^2 / tau)        */
/* written with the row minimum of the squared distance subtracted, which    */
/* leaves every A[j] unchanged mathematically and keeps exp() in range.      */
/* ------------------------------------------------------------------------ */
static void attention_row(double w, const double* C, int k, double tau, double* A) {
    double d[ORACLE_MAX_K];
    double dmin = INFINITY;
    for (int j = 0; j < k; ++j) {
        d[j] = (w - C[j]) * (w - C[j]);
        if (d[j] < dmin) dmin = d[j];
    }
    double Z = 0.0;
    for (int j = 0; j < k; ++j) {
        A[j] = exp(-(d[j] - dmin) / tau);
        Z += A[j];
    }
    for (int j = 0; j < k; ++j) A[j] /= Z;
}

/* Exported for the row-sum and identical-bits pins. */
void oracle_attention(const double* w, int64_t n, const double* C, int k, double tau, double* A /* n*k */) {
    for (int64_t i = 0; i < n; ++i) attention_row(w[i], C, k, tau, A + i * k);
}

/* ------------------------------------------------------------------------ */
/* Minimal thread pool: run fn(task) for nthreads contiguous chunks of       */
/* [0, n) and wait.  Each task owns its partial-sum arrays.                  */
/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t lo, hi;
    const void* ctx;
    double part[4 * ORACLE_MAX_K];  /* per-chunk partial sums */
} chunk_t;

typedef void (*chunk_fn)(chunk_t*);

static int resolve_threads(int nthreads, int64_t n) {
    if (nthreads <= 0) {
        long c = sysconf(_SC_NPROCESSORS_ONLN);
        nthreads = c > 0 ? (int)c : 1;
    }
    if (nthreads > ORACLE_MAX_THREADS) nthreads = ORACLE_MAX_THREADS;
    if (n < (int64_t)nthreads * 64) nthreads = (int)(n / 64) + 1;
    return nthreads;
}

static void* chunk_trampoline(void* arg) {
    chunk_t* c = (chunk_t*)arg;
    ((chunk_fn)(((void**)c->ctx)[0]))(c);
    return NULL;
}

/* ctx must begin with the chunk_fn pointer. */
static void parallel_chunks(int nthreads, int64_t n, const void* ctx, chunk_t* chunks) {
    pthread_t th[ORACLE_MAX_THREADS];
    for (int t = 0; t < nthreads; ++t) {
        chunks[t].lo = n * t / nthreads;
        chunks[t].hi = n * (t + 1) / nthreads;
        chunks[t].ctx = ctx;
        memset(chunks[t].part, 0, sizeof(chunks[t].part));
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, chunk_trampoline, &chunks[t]);
    chunk_trampoline(&chunks[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* ------------------------------------------------------------------------ */
/* Forward: unrolled soft k-means (R2-R6).                          */
/*   for t = 0 .. max_iter-1:                                                 */
/*     A_t[i][j] = attention(w_i, C_t)                       (dense |W|x|C|)  */
/*     S_t[j] = sum_i m_i A_t[i][j];  M_t[j] = sum_i m_i A_t[i][j] w_i         */
/*     C_{t+1}[j] = M_t[j] / S_t[j]   (C_t[j] kept if S_t[j] == 0, R6)         */
/*     if eps > 0 and max_j |C_{t+1}[j] - C_t[j]| <= eps: T = t+1, stop (R4)  */
/* m_i is the multiplicity of w_i: 1 for the dense map (mult == NULL), or    */
/* the count n_u of a unique pattern for the attention-table form.    */
/* Non-finite weights are excluded from the sums (R10).                       */
/* Outputs: C_traj[(max_iter+1)*k] (C_0..C_T), S_traj[max_iter*k], *T_out.   */
/* Returns 0, or -1 on bad arguments.                                         */
/* ------------------------------------------------------------------------ */
typedef struct {
    chunk_fn fn;
    const double* w;
    const double* mult;
    const double* C;
    int k;
    double tau;
} fwd_ctx;

static void fwd_chunk(chunk_t* c) {
    const fwd_ctx* x = (const fwd_ctx*)c->ctx;
    double A[ORACLE_MAX_K];
    double* S = c->part;
    double* M = c->part + ORACLE_MAX_K;
    for (int64_t i = c->lo; i < c->hi; ++i) {
        double w = x->w[i];
        if (!isfinite(w)) continue;
        double m = x->mult ? x->mult[i] : 1.0;
        attention_row(w, x->C, x->k, x->tau, A);
        for (int j = 0; j < x->k; ++j) {
            S[j] += m * A[j];
            M[j] += m * A[j] * w;
        }
    }
}

int oracle_dkm_forward(const double* w, const double* mult, int64_t n, int k, const double* C0, double tau,
                       int max_iter, double eps, int nthreads, double* C_traj, double* S_traj, int* T_out) {
    if (k < 1 || k > ORACLE_MAX_K || !(tau > 0) || !isfinite(tau) || max_iter < 0 || !(eps >= 0) || n < 0) return -1;
    nthreads = resolve_threads(nthreads, n);
    chunk_t* chunks = (chunk_t*)malloc(sizeof(chunk_t) * nthreads);
    for (int j = 0; j < k; ++j) C_traj[j] = C0[j];
    int T = max_iter;
    for (int t = 0; t < max_iter; ++t) {
        const double* Ct = C_traj + (int64_t)t * k;
        double* Cn = C_traj + (int64_t)(t + 1) * k;
        fwd_ctx ctx = {fwd_chunk, w, mult, Ct, k, tau};
        parallel_chunks(nthreads, n, &ctx, chunks);
        double S[ORACLE_MAX_K] = {0}, M[ORACLE_MAX_K] = {0};
        for (int c = 0; c < nthreads; ++c)
            for (int j = 0; j < k; ++j) {
                S[j] += chunks[c].part[j];
                M[j] += chunks[c].part[ORACLE_MAX_K + j];
            }
        double delta = 0.0;
        for (int j = 0; j < k; ++j) {
            S_traj[(int64_t)t * k + j] = S[j];
            Cn[j] = (S[j] == 0.0) ? Ct[j] : M[j] / S[j];
            double dj = fabs(Cn[j] - Ct[j]);
            if (dj > delta) delta = dj;
        }
        if (eps > 0.0 && delta <= eps) {
            T = t + 1;
            break;
        }
    }
    *T_out = T;
    free(chunks);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Reconstruction W~ (Fig. 1; R2):                       */
/*   W~_i = sum_j A[i][j] C[j],  A = attention(w_i, C).  Pass C = C_T.         */
/* Non-finite weights give NaN (R10).                                         */
/* ------------------------------------------------------------------------ */
void oracle_reconstruct(const double* w, int64_t n, const double* C, int k, double tau, double* Wt) {
    double A[ORACLE_MAX_K];
    for (int64_t i = 0; i < n; ++i) {
        if (!isfinite(w[i])) { Wt[i] = NAN; continue; }
        attention_row(w[i], C, k, tau, A);
        double s = 0.0;
        for (int j = 0; j < k; ++j) s += A[j] * C[j];
        Wt[i] = s;
    }
}

/* ------------------------------------------------------------------------ */
/* Hard palettisation ("a lookup table and a list of low-precision      */
/* indices"): idx_i = argmin_j (w_i - C[j])^2, lowest j on ties (R9).  C is   */
/* the fp32 lookup table itself; distances in fp64 from its exact values.    */
/* ------------------------------------------------------------------------ */
void oracle_hard_assign(const double* w, int64_t n, const float* C, int k, int32_t* idx) {
    for (int64_t i = 0; i < n; ++i) {
        int best = 0;
        double bd = (w[i] - (double)C[0]) * (w[i] - (double)C[0]);
        for (int j = 1; j < k; ++j) {
            double d = (w[i] - (double)C[j]) * (w[i] - (double)C[j]);
            if (d < bd) { bd = d; best = j; }
        }
        idx[i] = best;
    }
}

/* ------------------------------------------------------------------------ */
/* Backward, dense (chain rule through the forward above; R3, R6).  */
/* Given G_i = dL/dW~_i and the saved C_0..C_T, S_0..S_{T-1}:                 */
/*   gamma_T[l] = sum_i G_i A_T[i][l] (1 + (C_T[l] - W~_i) 2(w_i - C_T[l])/tau)*/
/*   dW_i       = G_i sum_l A_T[i][l] (C_T[l] - W~_i) (-2(w_i - C_T[l])/tau)  */
/*   for t = T-1 .. 0:                                                       */
/*     ghat[i][j] = gamma_{t+1}[j] (w_i - C_{t+1}[j]) / S_t[j]                */
/*     r[i][l]    = A_t[i][l] (ghat[i][l] - sum_j A_t[i][j] ghat[i][j])        */
/*     dW_i      += sum_j gamma_{t+1}[j] A_t[i][j] / S_t[j]                    */
/*                + sum_l r[i][l] (-2(w_i - C_t[l])/tau)                       */
/*     gamma_t[l] = sum_i r[i][l] 2(w_i - C_t[l])/tau                          */
/*                  (+ gamma_{t+1}[l] where S_t[l] == 0: C_{t+1}[l] = C_t[l])  */
/*   dC_0 = gamma_0                                                           */
/* Non-finite weights: dW_i = NaN and no contribution to gamma (R10).        */
/* ------------------------------------------------------------------------ */
typedef struct {
    chunk_fn fn;
    const double* w;
    const double* G;
    double* dW;
    const double* C;      /* C_T (last) or C_t (loop)    */
    const double* Cnext;  /* C_{t+1} (loop)              */
    const double* S;      /* S_t (loop)                  */
    const double* gnext;  /* gamma_{t+1} (loop)          */
    int k;
    double tau;
} bwd_ctx;

static void bwd_last_chunk(chunk_t* c) {
    const bwd_ctx* x = (const bwd_ctx*)c->ctx;
    double A[ORACLE_MAX_K];
    double* gamma = c->part;
    for (int64_t i = c->lo; i < c->hi; ++i) {
        double w = x->w[i];
        if (!isfinite(w)) { x->dW[i] = NAN; continue; }
        attention_row(w, x->C, x->k, x->tau, A);
        double Wt = 0.0;
        for (int l = 0; l < x->k; ++l) Wt += A[l] * x->C[l];
        double direct = 0.0;
        for (int l = 0; l < x->k; ++l) {
            gamma[l] += x->G[i] * A[l] * (1.0 + (x->C[l] - Wt) * 2.0 * (w - x->C[l]) / x->tau);
            direct += A[l] * (x->C[l] - Wt) * (-2.0 * (w - x->C[l]) / x->tau);
        }
        x->dW[i] = x->G[i] * direct;
    }
}

static void bwd_iter_chunk(chunk_t* c) {
    const bwd_ctx* x = (const bwd_ctx*)c->ctx;
    double A[ORACLE_MAX_K], ghat[ORACLE_MAX_K];
    double* gamma = c->part;
    for (int64_t i = c->lo; i < c->hi; ++i) {
        double w = x->w[i];
        if (!isfinite(w)) continue;
        attention_row(w, x->C, x->k, x->tau, A);
        double s = 0.0;
        for (int j = 0; j < x->k; ++j) {
            ghat[j] = (x->S[j] == 0.0) ? 0.0 : x->gnext[j] * (w - x->Cnext[j]) / x->S[j];
            s += A[j] * ghat[j];
        }
        double dw = 0.0;
        for (int l = 0; l < x->k; ++l) {
            double r = A[l] * (ghat[l] - s);
            if (x->S[l] != 0.0) dw += x->gnext[l] * A[l] / x->S[l];
            dw += r * (-2.0 * (w - x->C[l]) / x->tau);
            gamma[l] += r * 2.0 * (w - x->C[l]) / x->tau;
        }
        x->dW[i] += dw;
    }
}

int oracle_dkm_backward(const double* w, const double* G, int64_t n, int k, double tau, int T,
                        const double* C_traj, const double* S_traj, int nthreads, double* dW, double* dC) {
    if (k < 1 || k > ORACLE_MAX_K || !(tau > 0) || T < 0 || n < 0) return -1;
    nthreads = resolve_threads(nthreads, n);
    chunk_t* chunks = (chunk_t*)malloc(sizeof(chunk_t) * nthreads);
    double gamma[ORACLE_MAX_K] = {0};
    bwd_ctx ctx = {bwd_last_chunk, w, G, dW, C_traj + (int64_t)T * k, NULL, NULL, NULL, k, tau};
    parallel_chunks(nthreads, n, &ctx, chunks);
    for (int c = 0; c < nthreads; ++c)
        for (int l = 0; l < k; ++l) gamma[l] += chunks[c].part[l];
    for (int t = T - 1; t >= 0; --t) {
        bwd_ctx it = {bwd_iter_chunk, w, G, dW, C_traj + (int64_t)t * k, C_traj + (int64_t)(t + 1) * k,
                      S_traj + (int64_t)t * k, gamma, k, tau};
        parallel_chunks(nthreads, n, &it, chunks);
        double g[ORACLE_MAX_K] = {0};
        for (int c = 0; c < nthreads; ++c)
            for (int l = 0; l < k; ++l) g[l] += chunks[c].part[l];
        for (int l = 0; l < k; ++l) gamma[l] = g[l] + (S_traj[(int64_t)t * k + l] == 0.0 ? gamma[l] : 0.0);
    }
    for (int l = 0; l < k; ++l) dC[l] = gamma[l];
    free(chunks);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Backward on the attention table ("attention table ... and the index */
/* list"; equal bits => equal attention).  Every per-weight quantity   */
/* of the dense backward depends on w_i only through its pattern u, except  */
/* G_i, which enters linearly; hence                                         */
/*   dW_i = G_i phi[u_i] + psi[u_i],   gamma_T = sum_u B[u] f_T(u, .)          */
/* with B[u] = sum_{i in u} G_i and n_u = counts.  Inputs are the m unique     */
/* finite values v[u], their counts cnt[u] and bucket sums B[u]; outputs     */
/* phi[u], psi[u], dC.  Used only to check the paper's central claim against */
/* the dense form above (tests) and to reach large sizes quickly.            */
/* ------------------------------------------------------------------------ */
/* gammaT_in: if non-NULL, gamma_T is taken from it (e.g. the sum of per-learner partials,
 * P:79) instead of being accumulated from B, which may then be NULL. */
int oracle_dkm_backward_table(const double* v, const double* cnt, const double* B, int64_t m, int k, double tau,
                              int T, const double* C_traj, const double* S_traj, const double* gammaT_in,
                              double* phi, double* psi, double* dC) {
    if (k < 1 || k > ORACLE_MAX_K || !(tau > 0) || T < 0 || m < 0 || (!B && !gammaT_in)) return -1;
    double A[ORACLE_MAX_K], ghat[ORACLE_MAX_K];
    double gamma[ORACLE_MAX_K] = {0};
    const double* CT = C_traj + (int64_t)T * k;
    for (int64_t u = 0; u < m; ++u) {
        attention_row(v[u], CT, k, tau, A);
        double Wt = 0.0;
        for (int l = 0; l < k; ++l) Wt += A[l] * CT[l];
        double direct = 0.0;
        for (int l = 0; l < k; ++l) {
            if (!gammaT_in) gamma[l] += B[u] * A[l] * (1.0 + (CT[l] - Wt) * 2.0 * (v[u] - CT[l]) / tau);
            direct += A[l] * (CT[l] - Wt) * (-2.0 * (v[u] - CT[l]) / tau);
        }
        phi[u] = direct;
        psi[u] = 0.0;
    }
    if (gammaT_in)
        for (int l = 0; l < k; ++l) gamma[l] = gammaT_in[l];
    for (int t = T - 1; t >= 0; --t) {
        const double* Ct = C_traj + (int64_t)t * k;
        const double* Cn = C_traj + (int64_t)(t + 1) * k;
        const double* S = S_traj + (int64_t)t * k;
        double g[ORACLE_MAX_K] = {0};
        for (int64_t u = 0; u < m; ++u) {
            attention_row(v[u], Ct, k, tau, A);
            double s = 0.0;
            for (int j = 0; j < k; ++j) {
                ghat[j] = (S[j] == 0.0) ? 0.0 : gamma[j] * (v[u] - Cn[j]) / S[j];
                s += A[j] * ghat[j];
            }
            for (int l = 0; l < k; ++l) {
                double r = A[l] * (ghat[l] - s);
                if (S[l] != 0.0) psi[u] += gamma[l] * A[l] / S[l];
                psi[u] += r * (-2.0 * (v[u] - Ct[l]) / tau);
                g[l] += cnt[u] * r * 2.0 * (v[u] - Ct[l]) / tau;
            }
        }
        for (int l = 0; l < k; ++l) gamma[l] = g[l] + (S[l] == 0.0 ? gamma[l] : 0.0);
    }
    for (int l = 0; l < k; ++l) dC[l] = gamma[l];
    return 0;
}
