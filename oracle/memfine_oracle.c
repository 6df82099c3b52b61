/*
 * memfine_oracle.c — the CPU ORACLE for the MemFine chunked MoE layer.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2511_21431_b200/, libmemfine.so) never links, imports or calls it, and
 * this file shares no code, header, table or constant with the CUDA path.
 *
 * Plain, slow, obviously-correct C.  Floating point is computed in double (fp64);
 * integer work (counts, permutation, plan) in 64-bit integers.  Citations are
 * PAPER.md:<line> (arXiv 2511.21431 LaTeX) plus section / equation / table, and
 * SPEC.md:<line> where the CPU-program spec fixes an interface or test vector.
 *
 *  - Chunk partition X_1..X_c of Eq. 6 (§4.1): chunk j holds the
 *    tokens [floor(j*T/C), floor((j+1)*T/C)) (reading R1).
 *  - MoE layer Eq. 4:  Y = combine(expert(dispatch(X))), with
 *    the expert a bias-free SwiGLU MLP (Table 2 row 12 stores 2*g_e per copy,
 *    PAPER.md:86; reading R14) and combine the top-k score-weighted sum
 *    (Table 2 row 13 "score mul").
 *  - Backward Eq. 5 and the chunked recompute backward Eq. 7
 *    (PAPER.md:147-151): for each chunk, recompute F_w(X_j) then back-propagate.
 *  - Activation memory Eq. 2 + Table 2, s'_max Eq. 8
 *    (PAPER.md:194-198), c Eq. 9, bins.
 *
 * Parity status: every function here is pinned by tests/test_oracle_pins.py
 * (finite differences, hand-computed golden values, library reductions,
 * SPEC/paper printed vectors, invariants).  None is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ------------------------------------------------------------------------- */
/* Problem description.                                                       */
/* ------------------------------------------------------------------------- */
typedef struct {
    int64_t T;        /* tokens per rank (b*s of Table 1)                     */
    int32_t h;        /* hidden size h                                        */
    int32_t g;        /* expert FFN size g_e                                  */
    int32_t E;        /* number of (global) experts                           */
    int32_t k;        /* top-k t_k                                            */
    int32_t EP;       /* expert-parallel size e (paper), ranks emulated here  */
    int32_t in_dtype; /* x, dy, weights: 0 float32, 1 raw bf16 bits, 2 float64 */
} oracle_dims;

/* bf16 raw bits -> double, exactly. */
static double bf16_to_double(uint16_t b)
{
    uint32_t u = ((uint32_t)b) << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
}

static double load(const void* p, int64_t i, int dtype)
{
    if (dtype == 1) return bf16_to_double(((const uint16_t*)p)[i]);
    if (dtype == 2) return ((const double*)p)[i];
    return (double)((const float*)p)[i];
}

/* Chunk boundary, reading R1: floor(j*T/C). */
int64_t oracle_chunk_begin(int64_t T, int32_t C, int32_t j)
{
    return (int64_t)(((__int128)j * (__int128)T) / (__int128)C);
}

/* ------------------------------------------------------------------------- */
/* Routing counts: "the first notification".                   */
/* counts[j'][e] = number of (token, slot) copies of sub-chunk j' routed to e. */
/* Returns the number of expert ids outside [0, E) (they are not counted).     */
/* ------------------------------------------------------------------------- */
int64_t oracle_route_counts(const oracle_dims* d, int32_t nsub, const int32_t* ids, int64_t* counts)
{
    int64_t bad = 0;
    for (int64_t i = 0; i < (int64_t)nsub * d->E; i++) counts[i] = 0;
    for (int32_t j = 0; j < nsub; j++) {
        int64_t t0 = oracle_chunk_begin(d->T, nsub, j);
        int64_t t1 = oracle_chunk_begin(d->T, nsub, j + 1);
        for (int64_t i = t0; i < t1; i++) {
            for (int32_t s = 0; s < d->k; s++) {
                int32_t e = ids[i * d->k + s];
                if (e < 0 || e >= d->E) { bad++; continue; }
                counts[(int64_t)j * d->E + e] += 1;
            }
        }
    }
    return bad;
}

/* ------------------------------------------------------------------------- */
/* Memory model.                                                              */
/* ------------------------------------------------------------------------- */
typedef struct {
    int64_t m_g, t, c, D_t, b, s, h, a, h_d, k_a, e_n, g_e;
} oracle_act_cfg;

/* Eq. 2, closed form:
 *   M^act = (m_g/(t c)) D_t b ( s(5h + a h_d + 2 k_a h_d + e_n) + s'(2h + 2 g_e) ).
 * Integer bytes: all integer factors multiplied first, one floor division by t*c. */
uint64_t oracle_act_bytes_eq2(const oracle_act_cfg* q, int64_t s_prime)
{
    __int128 s_term = (__int128)q->s * (5 * q->h + q->a * q->h_d + 2 * q->k_a * q->h_d + q->e_n);
    __int128 sp_term = (__int128)s_prime * (2 * q->h + 2 * q->g_e);
    __int128 num = (__int128)q->m_g * q->D_t * q->b * (s_term + sp_term);
    return (uint64_t)(num / ((__int128)q->t * q->c));
}

/* Table 2, row by row, before the 1/(tc) and m_g factors:
 * rows[0..13] = stored bytes of input IDs 1..14 (rows 7 and 14 "add" store 0). */
void oracle_act_table2_rows(const oracle_act_cfg* q, int64_t s_prime, int64_t rows[14])
{
    int64_t Db = q->D_t * q->b;
    rows[0]  = Db * q->s * q->h;               /* 1  norm               */
    rows[1]  = Db * q->s * q->h;               /* 2  q, k, v            */
    rows[2]  = Db * q->s * q->a * q->h_d;      /* 3  attention          */
    rows[3]  = Db * q->s * q->k_a * q->h_d;    /* 4  attention          */
    rows[4]  = Db * q->s * q->k_a * q->h_d;    /* 5  attention          */
    rows[5]  = Db * q->s * q->h;               /* 6  o                  */
    rows[6]  = 0;                              /* 7  add                */
    rows[7]  = Db * q->s * q->h;               /* 8  norm               */
    rows[8]  = Db * q->s * q->h;               /* 9  router             */
    rows[9]  = Db * q->s * q->e_n;             /* 10 router             */
    rows[10] = Db * s_prime * q->h;            /* 11 activated expert   */
    rows[11] = 2 * Db * s_prime * q->g_e;      /* 12 activated expert   */
    rows[12] = Db * s_prime * q->h;            /* 13 score mul          */
    rows[13] = 0;                              /* 14 add                */
}

/* Eq. 8 in integer bytes (reading R9):
 *   s'_max = floor( (B - M_sta - (m_g/(tc)) D_t b s(5h+a h_d+2k_a h_d+e_n)) * t c
 *                   / (m_g D_t b (2h + 2 g_e)) )
 * B = floor(alpha * M^GPU) is passed already floored.  May return <= 0. */
int64_t oracle_s_prime_max_eq8(const oracle_act_cfg* q, uint64_t budget, uint64_t static_bytes)
{
    __int128 s_term_bytes = (__int128)q->m_g * q->D_t * q->b * q->s *
                            (5 * q->h + q->a * q->h_d + 2 * q->k_a * q->h_d + q->e_n) /
                            ((__int128)q->t * q->c);
    __int128 num = (__int128)budget - (__int128)static_bytes - s_term_bytes;
    __int128 den = (__int128)q->m_g * q->D_t * q->b * (2 * q->h + 2 * q->g_e);
    __int128 v = num * q->t * q->c;
    /* floor division toward -inf */
    __int128 qv = v / den;
    if ((v % den != 0) && ((v < 0) != (den < 0))) qv -= 1;
    return (int64_t)qv;
}

/* ------------------------------------------------------------------------- */
/* MACT plan (§4.2), reading of SURVEY §8(c).2.             */
/* ------------------------------------------------------------------------- */
typedef struct {
    uint64_t budget_bytes;     /* B = floor(alpha * M^GPU), Eq. 3 right side     */
    uint64_t static_bytes;     /* M^sta (Eq. 1), caller-supplied                 */
    uint64_t other_act_bytes;  /* Eq. 2 s-term, caller-supplied                  */
    int64_t  m_g, tp, cp, micro_batch, D_t;
    const int32_t* bins; int32_t nbins;
    int32_t rule;              /* 0 = EQ9 (paper), 1 = EXACT                     */
} oracle_budget;

typedef struct {
    int32_t C, c_theory, clamped, feasible, hot_rank, exact_peak;
    int64_t s_dd_max;          /* max_r s''_r                                     */
    int64_t s_prime_max;       /* Eq. 8                                           */
    int64_t s_chunk_max;       /* max_r max_j s''_{r,j}(C)  (or the ceil estimate)*/
    uint64_t predicted_peak_bytes; /* paper model for s_chunk_max                 */
} oracle_plan_out;

/* Return codes follow SPEC.md's exit-code contract:
 * 0 ok, 1 invalid argument, 2 infeasible. */
int32_t oracle_plan(const int64_t* counts /*[EP][nsub][E]*/, int32_t nsub,
                    const oracle_dims* d, const oracle_budget* b, oracle_plan_out* out)
{
    memset(out, 0, sizeof *out);
    if (nsub < 1 || d->EP < 1 || d->E % d->EP != 0 || b->nbins < 1) return 1;
    for (int32_t i = 0; i < b->nbins; i++) {
        if (b->bins[i] < 1) return 1;
        if (i > 0 && b->bins[i] <= b->bins[i - 1]) return 1;
    }
    if (b->m_g < 1 || b->tp < 1 || b->cp < 1 || b->micro_batch < 1 || b->D_t < 1) return 1;
    int32_t E_l = d->E / d->EP;

    /* Eq. 8 numerator: B - M^sta - s-term.  <= 0 -> infeasible. */
    __int128 num = (__int128)b->budget_bytes - (__int128)b->static_bytes - (__int128)b->other_act_bytes;
    if (num <= 0) return 2;
    __int128 den = (__int128)b->m_g * b->D_t * b->micro_batch * (2 * (__int128)d->h + 2 * (__int128)d->g);
    int64_t s_prime_max = (int64_t)((num * b->tp * b->cp) / den);
    out->s_prime_max = s_prime_max;
    if (s_prime_max <= 0) return 2;

    /* s''_r = sum over sources, sub-chunks and the experts hosted by r. */
    int64_t s_dd_max = -1; int32_t hot = 0;
    for (int32_t r = 0; r < d->EP; r++) {
        int64_t s = 0;
        for (int32_t src = 0; src < d->EP; src++)
            for (int32_t j = 0; j < nsub; j++)
                for (int32_t e = r * E_l; e < (r + 1) * E_l; e++)
                    s += counts[((int64_t)src * nsub + j) * d->E + e];
        if (s > s_dd_max) { s_dd_max = s; hot = r; }
    }
    out->s_dd_max = s_dd_max;
    out->hot_rank = hot;

    /* Eq. 9: c = ceil(s'' / s'_max), at least 1. */
    int64_t c = (s_dd_max + s_prime_max - 1) / s_prime_max;
    if (c < 1) c = 1;
    out->c_theory = (int32_t)(c > 0x7fffffff ? 0x7fffffff : c);

    int32_t C = -1;
    if (b->rule == 0) {
        /* "select the large bin that is closest to c": smallest bin >= c. */
        for (int32_t i = 0; i < b->nbins; i++) if (b->bins[i] >= c) { C = b->bins[i]; break; }
    } else {
        /* EXACT: smallest bin whose true per-chunk maximum fits s'_max.  Every bin
         * must nest in the nsub sub-chunks so that its chunk counts are exact. */
        for (int32_t i = 0; i < b->nbins; i++) if (nsub % b->bins[i] != 0) return 1;
        for (int32_t i = 0; i < b->nbins && C < 0; i++) {
            int32_t Cb = b->bins[i], per = nsub / Cb;
            int64_t mx = 0;
            for (int32_t r = 0; r < d->EP; r++)
                for (int32_t jc = 0; jc < Cb; jc++) {
                    int64_t s = 0;
                    for (int32_t src = 0; src < d->EP; src++)
                        for (int32_t j = jc * per; j < (jc + 1) * per; j++)
                            for (int32_t e = r * E_l; e < (r + 1) * E_l; e++)
                                s += counts[((int64_t)src * nsub + j) * d->E + e];
                    if (s > mx) mx = s;
                }
            if (mx <= s_prime_max) C = Cb;
        }
    }
    if (C < 0) { C = b->bins[b->nbins - 1]; out->clamped = 1; }
    out->C = C;

    /* Per-chunk maximum for the chosen C: exact when the C chunks nest in the
     * sub-chunks, else the Eq. 9 estimate ceil(s''/C) (SPEC.md mact invariant). */
    int64_t mx = 0;
    if (nsub % C == 0) {
        int32_t per = nsub / C;
        out->exact_peak = 1;
        for (int32_t r = 0; r < d->EP; r++)
            for (int32_t jc = 0; jc < C; jc++) {
                int64_t s = 0;
                for (int32_t src = 0; src < d->EP; src++)
                    for (int32_t j = jc * per; j < (jc + 1) * per; j++)
                        for (int32_t e = r * E_l; e < (r + 1) * E_l; e++)
                            s += counts[((int64_t)src * nsub + j) * d->E + e];
                if (s > mx) mx = s;
            }
    } else {
        out->exact_peak = 0;
        mx = (s_dd_max + C - 1) / C;
    }
    out->s_chunk_max = mx;
    out->feasible = (mx <= s_prime_max) ? 1 : 0;
    out->predicted_peak_bytes = (uint64_t)(((__int128)b->m_g * b->D_t * b->micro_batch * mx *
                                            (2 * (__int128)d->h + 2 * (__int128)d->g)) /
                                           ((__int128)b->tp * b->cp));
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Canonical dispatch order on rank r for chunk j of C (reading R3):           */
/* ascending (expert, src rank, src token, slot) over all copies of chunk j   */
/* whose expert is hosted by r (experts [r*E_l, (r+1)*E_l), reading R4).       */
/* perm[p] = src*T*k + i*k + slot.  Returns the number of rows (or -1 if the   */
/* capacity is too small).                                                     */
/* ------------------------------------------------------------------------- */
int64_t oracle_dispatch_order(const oracle_dims* d, const int32_t* ids_all /*[EP][T][k]*/,
                              int32_t rank, int32_t C, int32_t j, int64_t* perm, int64_t cap)
{
    int32_t E_l = d->E / d->EP;
    int64_t n = 0;
    int64_t t0 = oracle_chunk_begin(d->T, C, j), t1 = oracle_chunk_begin(d->T, C, j + 1);
    for (int32_t e = rank * E_l; e < (rank + 1) * E_l; e++)
        for (int32_t src = 0; src < d->EP; src++)
            for (int64_t i = t0; i < t1; i++)
                for (int32_t s = 0; s < d->k; s++) {
                    int64_t q = ((int64_t)src * d->T + i) * d->k + s;
                    if (ids_all[q] != e) continue;
                    if (n >= cap) return -1;
                    perm[n++] = q;
                }
    return n;
}

/* ------------------------------------------------------------------------- */
/* The expert: bias-free SwiGLU MLP (reading R14), one routed copy.           */
/*   G = W_gate[e] x,  U = W_up[e] x,  a = silu(G) (.) U,  o = W_down[e] a     */
/* silu(z) = z / (1 + exp(-z)).                                                */
/* ------------------------------------------------------------------------- */
static double sigmoid(double z) { return 1.0 / (1.0 + exp(-z)); }

static void expert_forward(const oracle_dims* d, const void* x, int64_t xoff,
                           const void* wg, const void* wu, const void* wd, int32_t e,
                           double* G, double* U, double* A, double* O)
{
    int64_t h = d->h, g = d->g;
    for (int64_t n = 0; n < g; n++) {
        double sg = 0.0, su = 0.0;
        for (int64_t c = 0; c < h; c++) {
            double xv = load(x, xoff + c, d->in_dtype);
            sg += load(wg, ((int64_t)e * g + n) * h + c, d->in_dtype) * xv;
            su += load(wu, ((int64_t)e * g + n) * h + c, d->in_dtype) * xv;
        }
        G[n] = sg; U[n] = su;
        A[n] = sg * sigmoid(sg) * su;
    }
    for (int64_t m = 0; m < h; m++) {
        double so = 0.0;
        for (int64_t n = 0; n < g; n++)
            so += load(wd, ((int64_t)e * h + m) * g + n, d->in_dtype) * A[n];
        O[m] = so;
    }
}

/* Forward, Eq. 4, per token (the plain definition):
 *   Y_i = sum_{slot ascending} w_{i,slot} * expert_{ids[i,slot]}(x_i).
 * x, ids, w, y are [EP][T][...] (all emulated ranks); weights hold all E experts.
 * Copies with an out-of-range expert id contribute nothing. */
void oracle_moe_forward(const oracle_dims* d, const void* x, const int32_t* ids, const double* w,
                        const void* wg, const void* wu, const void* wd, double* y)
{
    int64_t h = d->h, g = d->g, ntok = (int64_t)d->EP * d->T;
    #pragma omp parallel
    {
        double* G = (double*)malloc(sizeof(double) * (size_t)(3 * g + h));
        double *U = G + g, *A = U + g, *O = A + g;
        #pragma omp for schedule(dynamic, 1)
        for (int64_t t = 0; t < ntok; t++) {
            double* yt = y + t * h;
            for (int64_t m = 0; m < h; m++) yt[m] = 0.0;
            for (int32_t s = 0; s < d->k; s++) {
                int32_t e = ids[t * d->k + s];
                if (e < 0 || e >= d->E) continue;
                double ws = w[t * d->k + s];
                expert_forward(d, x, t * h, wg, wu, wd, e, G, U, A, O);
                for (int64_t m = 0; m < h; m++) yt[m] += ws * O[m];
            }
        }
        free(G);
    }
}

/* Per-copy backward quantities (Eq. 5; reading R15 for d_score):
 *   d_w = <dY_i, o>,  dO = w dY_i,  dA = W_down^T dO,
 *   dG = dA (.) U (.) sig(G)(1 + G(1 - sig(G))),  dU = dA (.) silu(G),
 *   dX_copy = W_gate^T dG + W_up^T dU.
 * Writes a, dO, dG, dU into the copy's slots for the weight-gradient phase. */
static void expert_backward(const oracle_dims* d, const void* x, int64_t xoff, const void* dy, int64_t dyoff,
                            double ws, const void* wg, const void* wu, const void* wd, int32_t e,
                            double* scratch, double* a_out, double* dO_out, double* dG_out, double* dU_out,
                            double* dx_copy, double* dscore)
{
    int64_t h = d->h, g = d->g;
    double *G = scratch, *U = G + g, *A = U + g, *O = A + g, *dA = O + h;
    expert_forward(d, x, xoff, wg, wu, wd, e, G, U, A, O);
    double dwv = 0.0;
    for (int64_t m = 0; m < h; m++) dwv += load(dy, dyoff + m, d->in_dtype) * O[m];
    *dscore = dwv;
    for (int64_t m = 0; m < h; m++) dO_out[m] = ws * load(dy, dyoff + m, d->in_dtype);
    for (int64_t n = 0; n < g; n++) {
        double s = 0.0;
        for (int64_t m = 0; m < h; m++) s += load(wd, ((int64_t)e * h + m) * g + n, d->in_dtype) * dO_out[m];
        dA[n] = s;
    }
    for (int64_t n = 0; n < g; n++) {
        double sg = sigmoid(G[n]);
        dG_out[n] = dA[n] * U[n] * sg * (1.0 + G[n] * (1.0 - sg));
        dU_out[n] = dA[n] * G[n] * sg;
        a_out[n] = A[n];
    }
    for (int64_t c = 0; c < h; c++) {
        double s1 = 0.0, s2 = 0.0;
        for (int64_t n = 0; n < g; n++) {
            s1 += load(wg, ((int64_t)e * g + n) * h + c, d->in_dtype) * dG_out[n];
            s2 += load(wu, ((int64_t)e * g + n) * h + c, d->in_dtype) * dU_out[n];
        }
        dx_copy[c] = s1 + s2;
    }
}

/* Weight gradients: one running accumulator per element, copies visited in the
 * order given by `order` (reading R18: W_grad = sum over chunks). */
static void accumulate_dw(const oracle_dims* d, const void* x, const int32_t* ids,
                          const int64_t* order, int64_t norder,
                          const double* a_all, const double* dO_all, const double* dG_all, const double* dU_all,
                          double* dwg, double* dwu, double* dwd)
{
    int64_t h = d->h, g = d->g;
    memset(dwg, 0, sizeof(double) * (size_t)d->E * g * h);
    memset(dwu, 0, sizeof(double) * (size_t)d->E * g * h);
    memset(dwd, 0, sizeof(double) * (size_t)d->E * h * g);
    /* dW_gate / dW_up rows: (e, n); dW_down rows: (e, m).  Each row owned by one thread. */
    #pragma omp parallel for schedule(dynamic, 4)
    for (int64_t row = 0; row < (int64_t)d->E * (g + h); row++) {
        int32_t e = (int32_t)(row / (g + h));
        int64_t r = row % (g + h);
        for (int64_t p = 0; p < norder; p++) {
            int64_t q = order[p];
            if (ids[q] != e) continue;
            int64_t t = q / d->k;
            if (r < g) {
                int64_t n = r;
                double gd = dG_all[q * g + n], ud = dU_all[q * g + n];
                double* rg = dwg + ((int64_t)e * g + n) * h;
                double* ru = dwu + ((int64_t)e * g + n) * h;
                for (int64_t c = 0; c < h; c++) {
                    double xv = load(x, t * h + c, d->in_dtype);
                    rg[c] += gd * xv;
                    ru[c] += ud * xv;
                }
            } else {
                int64_t m = r - g;
                double od = dO_all[q * h + m];
                double* rd = dwd + ((int64_t)e * h + m) * g;
                for (int64_t n = 0; n < g; n++) rd[n] += od * a_all[q * g + n];
            }
        }
    }
}

static void backward_copies(const oracle_dims* d, const void* dy, const void* x, const int32_t* ids, const double* w,
                            const void* wg, const void* wu, const void* wd,
                            double* dx, double* dscore, double* a_all, double* dO_all, double* dG_all, double* dU_all)
{
    int64_t h = d->h, g = d->g, ntok = (int64_t)d->EP * d->T;
    #pragma omp parallel
    {
        double* scratch = (double*)malloc(sizeof(double) * (size_t)(4 * g + 2 * h + h));
        double* dxc = scratch + 4 * g + 2 * h;
        #pragma omp for schedule(dynamic, 1)
        for (int64_t t = 0; t < ntok; t++) {
            for (int64_t c = 0; c < h; c++) dx[t * h + c] = 0.0;
            for (int32_t s = 0; s < d->k; s++) {
                int64_t q = t * d->k + s;
                int32_t e = ids[q];
                dscore[q] = 0.0;
                if (e < 0 || e >= d->E) {
                    memset(a_all + q * g, 0, sizeof(double) * (size_t)g);
                    memset(dG_all + q * g, 0, sizeof(double) * (size_t)g);
                    memset(dU_all + q * g, 0, sizeof(double) * (size_t)g);
                    memset(dO_all + q * h, 0, sizeof(double) * (size_t)h);
                    continue;
                }
                expert_backward(d, x, t * h, dy, t * h, w[q], wg, wu, wd, e, scratch,
                                a_all + q * g, dO_all + q * h, dG_all + q * g, dU_all + q * g, dxc, dscore + q);
                for (int64_t c = 0; c < h; c++) dx[t * h + c] += dxc[c];
            }
        }
        free(scratch);
    }
}

/* Backward, Eq. 5, unchunked.  dW of expert e accumulates its copies in the
 * canonical order (src rank, token, slot).  Outputs: dx [EP][T][h],
 * dscore [EP][T][k], dwg/dwu [E][g][h], dwd [E][h][g]. */
int32_t oracle_moe_backward(const oracle_dims* d, const void* dy, const void* x, const int32_t* ids, const double* w,
                            const void* wg, const void* wu, const void* wd,
                            double* dx, double* dscore, double* dwg, double* dwu, double* dwd)
{
    int64_t h = d->h, g = d->g, nq = (int64_t)d->EP * d->T * d->k;
    double* a_all = (double*)malloc(sizeof(double) * (size_t)nq * g);
    double* dG_all = (double*)malloc(sizeof(double) * (size_t)nq * g);
    double* dU_all = (double*)malloc(sizeof(double) * (size_t)nq * g);
    double* dO_all = (double*)malloc(sizeof(double) * (size_t)nq * h);
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nq > 0 ? nq : 1));
    if (!a_all || !dG_all || !dU_all || !dO_all || !order) {
        free(a_all); free(dG_all); free(dU_all); free(dO_all); free(order);
        return 1;
    }
    backward_copies(d, dy, x, ids, w, wg, wu, wd, dx, dscore, a_all, dO_all, dG_all, dU_all);
    for (int64_t q = 0; q < nq; q++) order[q] = q;   /* (src, token, slot) ascending */
    accumulate_dw(d, x, ids, order, nq, a_all, dO_all, dG_all, dU_all, dwg, dwu, dwd);
    free(a_all); free(dG_all); free(dU_all); free(dO_all); free(order);
    return 0;
}

/* Eq. 5 for a subset of experts: dx and dscore as oracle_moe_backward, and the weight gradients of
 * the experts sel[0..nsel) only (dwg/dwu [nsel][g][h], dwd [nsel][h][g]), each accumulated over its
 * copies in the canonical order exactly as oracle_moe_backward does - for full-size checks, where
 * all experts' fp64 gradients would not fit in host memory at once. */
int32_t oracle_moe_backward_experts(const oracle_dims* d, const void* dy, const void* x, const int32_t* ids,
                                    const double* w, const void* wg, const void* wu, const void* wd, int32_t nsel,
                                    const int32_t* sel, double* dx, double* dscore, double* dwg, double* dwu,
                                    double* dwd)
{
    int64_t h = d->h, g = d->g, nq = (int64_t)d->EP * d->T * d->k;
    double* a_all = (double*)malloc(sizeof(double) * (size_t)(nq > 0 ? nq : 1) * g);
    double* dG_all = (double*)malloc(sizeof(double) * (size_t)(nq > 0 ? nq : 1) * g);
    double* dU_all = (double*)malloc(sizeof(double) * (size_t)(nq > 0 ? nq : 1) * g);
    double* dO_all = (double*)malloc(sizeof(double) * (size_t)(nq > 0 ? nq : 1) * h);
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nq > 0 ? nq : 1));
    int32_t* ids_e = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nq > 0 ? nq : 1));
    if (!a_all || !dG_all || !dU_all || !dO_all || !order || !ids_e) {
        free(a_all); free(dG_all); free(dU_all); free(dO_all); free(order); free(ids_e);
        return 1;
    }
    backward_copies(d, dy, x, ids, w, wg, wu, wd, dx, dscore, a_all, dO_all, dG_all, dU_all);
    for (int64_t q = 0; q < nq; q++) order[q] = q;   /* (src, token, slot) ascending */
    /* expert sel[i] becomes expert i of a problem with nsel experts: accumulate_dw visits the same
     * copies in the same order */
    for (int64_t q = 0; q < nq; q++) {
        ids_e[q] = -1;
        for (int32_t i = 0; i < nsel; i++) if (ids[q] == sel[i]) { ids_e[q] = i; break; }
    }
    oracle_dims ds = *d;
    ds.E = nsel;
    accumulate_dw(&ds, x, ids_e, order, nq, a_all, dO_all, dG_all, dU_all, dwg, dwu, dwd);
    free(a_all); free(dG_all); free(dU_all); free(dO_all); free(order); free(ids_e);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* FCDA, Eq. 6 / Eq. 7, written as the paper's chunk loop with the meter.     */
/* ------------------------------------------------------------------------- */
/* Meter: at the start of chunk j, rank r charges
 * Table 2 rows 11-13 for its received copies, D_t * s''_{r,j} * (h + 2g + h),
 * and releases them at chunk end; peak = max over chunks.
 * chunk_bytes[r*C + j] and peak[r] are written when non-NULL. */
static void meter_chunk(const oracle_dims* d, const int32_t* ids_all, int32_t C, int32_t j, int64_t D_t,
                        uint64_t* chunk_bytes, uint64_t* peak)
{
    int32_t E_l = d->E / d->EP;
    int64_t t0 = oracle_chunk_begin(d->T, C, j), t1 = oracle_chunk_begin(d->T, C, j + 1);
    for (int32_t r = 0; r < d->EP; r++) {
        int64_t s = 0;
        for (int32_t src = 0; src < d->EP; src++)
            for (int64_t i = t0; i < t1; i++)
                for (int32_t sl = 0; sl < d->k; sl++) {
                    int32_t e = ids_all[((int64_t)src * d->T + i) * d->k + sl];
                    if (e >= r * E_l && e < (r + 1) * E_l) s++;
                }
        uint64_t bytes = (uint64_t)(D_t * s * (2 * (int64_t)d->h + 2 * (int64_t)d->g));
        if (chunk_bytes) chunk_bytes[(int64_t)r * C + j] = bytes;
        if (peak && bytes > peak[r]) peak[r] = bytes;
    }
}

/* Eq. 6: Y = concat(F_w(X_1), ..., F_w(X_c)).  For chunk j: dispatch (gather
 * the chunk's copies into each rank's canonical expert-major buffer), expert
 * (one SwiGLU per received row), combine (score-weighted sum back at the
 * source token, slot order). */
int32_t oracle_moe_fcda_forward(const oracle_dims* d, int32_t C, const void* x, const int32_t* ids, const double* w,
                                const void* wg, const void* wu, const void* wd, double* y,
                                int64_t D_t, uint64_t* chunk_bytes, uint64_t* peak)
{
    int64_t h = d->h, g = d->g, nq = (int64_t)d->EP * d->T * d->k;
    if (C < 1) return 1;
    int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nq > 0 ? nq : 1));
    double* orows = (double*)malloc(sizeof(double) * (size_t)(nq > 0 ? nq : 1) * h);  /* expert output per copy */
    if (!perm || !orows) { free(perm); free(orows); return 1; }
    if (peak) for (int32_t r = 0; r < d->EP; r++) peak[r] = 0;
    for (int32_t j = 0; j < C; j++) {
        meter_chunk(d, ids, C, j, D_t, chunk_bytes, peak);
        int64_t t0 = oracle_chunk_begin(d->T, C, j), t1 = oracle_chunk_begin(d->T, C, j + 1);
        /* dispatch + expert, rank by rank */
        for (int32_t r = 0; r < d->EP; r++) {
            int64_t n = oracle_dispatch_order(d, ids, r, C, j, perm, nq);
            #pragma omp parallel
            {
                double* G = (double*)malloc(sizeof(double) * (size_t)(3 * g + h));
                double *U = G + g, *A = U + g, *O = A + g;
                #pragma omp for schedule(dynamic, 1)
                for (int64_t p = 0; p < n; p++) {
                    int64_t q = perm[p], t = q / d->k;
                    expert_forward(d, x, t * h, wg, wu, wd, ids[q], G, U, A, O);
                    memcpy(orows + q * h, O, sizeof(double) * (size_t)h);
                }
                free(G);
            }
        }
        /* combine: Y_i = sum_slot w * o, slot ascending, for the chunk's tokens */
        for (int32_t src = 0; src < d->EP; src++)
            for (int64_t i = t0; i < t1; i++) {
                int64_t t = (int64_t)src * d->T + i;
                for (int64_t m = 0; m < h; m++) y[t * h + m] = 0.0;
                for (int32_t s = 0; s < d->k; s++) {
                    int64_t q = t * d->k + s;
                    int32_t e = ids[q];
                    if (e < 0 || e >= d->E) continue;
                    for (int64_t m = 0; m < h; m++) y[t * h + m] += w[q] * orows[q * h + m];
                }
            }
    }
    free(perm); free(orows);
    return 0;
}

/* Eq. 7: X_grad = concat(B_w(Y_grad, F_w(X_1)), ..., B_w(Y_grad, F_w(X_c))),
 * Y_grad sliced by the same partition (reading R16); each chunk recomputes its
 * forward just before its gradients; W_grad = sum over chunks (reading R18),
 * one running accumulator visiting chunk-major canonical order
 * (chunk, src rank, token, slot). */
int32_t oracle_moe_fcda_backward(const oracle_dims* d, int32_t C, const void* dy, const void* x, const int32_t* ids,
                                 const double* w, const void* wg, const void* wu, const void* wd,
                                 double* dx, double* dscore, double* dwg, double* dwu, double* dwd,
                                 int64_t D_t, uint64_t* chunk_bytes, uint64_t* peak)
{
    int64_t h = d->h, g = d->g, nq = (int64_t)d->EP * d->T * d->k;
    if (C < 1) return 1;
    double* a_all = (double*)malloc(sizeof(double) * (size_t)(nq > 0 ? nq : 1) * g);
    double* dG_all = (double*)malloc(sizeof(double) * (size_t)(nq > 0 ? nq : 1) * g);
    double* dU_all = (double*)malloc(sizeof(double) * (size_t)(nq > 0 ? nq : 1) * g);
    double* dO_all = (double*)malloc(sizeof(double) * (size_t)(nq > 0 ? nq : 1) * h);
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nq > 0 ? nq : 1));
    if (!a_all || !dG_all || !dU_all || !dO_all || !order) {
        free(a_all); free(dG_all); free(dU_all); free(dO_all); free(order);
        return 1;
    }
    if (peak) for (int32_t r = 0; r < d->EP; r++) peak[r] = 0;
    for (int64_t q = 0; q < nq; q++) dscore[q] = 0.0;
    int64_t norder = 0;
    for (int32_t j = 0; j < C; j++) {
        meter_chunk(d, ids, C, j, D_t, chunk_bytes, peak);
        int64_t t0 = oracle_chunk_begin(d->T, C, j), t1 = oracle_chunk_begin(d->T, C, j + 1);
        /* recompute + backward for the chunk's copies (token-local quantities) */
        #pragma omp parallel
        {
            double* scratch = (double*)malloc(sizeof(double) * (size_t)(4 * g + 3 * h));
            double* dxc = scratch + 4 * g + 2 * h;
            #pragma omp for schedule(dynamic, 1) collapse(2)
            for (int32_t src = 0; src < d->EP; src++)
                for (int64_t i = t0; i < t1; i++) {
                    int64_t t = (int64_t)src * d->T + i;
                    for (int64_t c = 0; c < h; c++) dx[t * h + c] = 0.0;
                    for (int32_t s = 0; s < d->k; s++) {
                        int64_t q = t * d->k + s;
                        int32_t e = ids[q];
                        if (e < 0 || e >= d->E) continue;
                        expert_backward(d, x, t * h, dy, t * h, w[q], wg, wu, wd, e, scratch,
                                        a_all + q * g, dO_all + q * h, dG_all + q * g, dU_all + q * g,
                                        dxc, dscore + q);
                        for (int64_t c = 0; c < h; c++) dx[t * h + c] += dxc[c];
                    }
                }
            free(scratch);
        }
        /* this chunk's copies, appended in (src, token, slot) order */
        for (int32_t src = 0; src < d->EP; src++)
            for (int64_t i = t0; i < t1; i++)
                for (int32_t s = 0; s < d->k; s++)
                    order[norder++] = ((int64_t)src * d->T + i) * d->k + s;
    }
    accumulate_dw(d, x, ids, order, norder, a_all, dO_all, dG_all, dU_all, dwg, dwu, dwd);
    free(a_all); free(dG_all); free(dU_all); free(dO_all); free(order);
    return 0;
}

/* Outputs for a list of tokens only (global index src*T + i): y, dx, dscore.
 * Used for sampled checks at full size, where the per-copy work is small. */
void oracle_moe_tokens(const oracle_dims* d, int64_t ntok, const int64_t* toks,
                       const void* dy, const void* x, const int32_t* ids, const double* w,
                       const void* wg, const void* wu, const void* wd,
                       double* y /*[ntok][h]*/, double* dx /*[ntok][h]*/, double* dscore /*[ntok][k]*/)
{
    int64_t h = d->h, g = d->g;
    #pragma omp parallel
    {
        double* scratch = (double*)malloc(sizeof(double) * (size_t)(4 * g + 3 * h));
        double* dxc = scratch + 4 * g + 2 * h;
        double* a1 = (double*)malloc(sizeof(double) * (size_t)(3 * g + h));
        double *dG1 = a1 + g, *dU1 = dG1 + g, *dO1 = dU1 + g;
        #pragma omp for schedule(dynamic, 1)
        for (int64_t p = 0; p < ntok; p++) {
            int64_t t = toks[p];
            for (int64_t c = 0; c < h; c++) { y[p * h + c] = 0.0; dx[p * h + c] = 0.0; }
            for (int32_t s = 0; s < d->k; s++) {
                int64_t q = t * d->k + s;
                int32_t e = ids[q];
                dscore[p * d->k + s] = 0.0;
                if (e < 0 || e >= d->E) continue;
                double* Gs = scratch; double* O = scratch + 3 * g;
                expert_backward(d, x, t * h, dy, t * h, w[q], wg, wu, wd, e, scratch,
                                a1, dO1, dG1, dU1, dxc, dscore + p * d->k + s);
                (void)Gs;
                for (int64_t c = 0; c < h; c++) {
                    y[p * h + c] += w[q] * O[c];
                    dx[p * h + c] += dxc[c];
                }
            }
        }
        free(scratch); free(a1);
    }
}

/* ------------------------------------------------------------------------- */
/* Router (Table 2 rows 9-10: the router stores its input and  */
/* its e_n logits).  logits = x W_r^T; the k largest logits (ties: lower expert id first);        */
/* scores = softmax over the k selected logits (the renormalised top-k convention).               */
/* x [ntok][h] and W_r [E][h] as in_dtype; logits, scores double; ids int32.                     */
/* ------------------------------------------------------------------------- */
void oracle_router_forward(const oracle_dims* d, int64_t ntok, const void* x, const void* wr,
                           double* logits, int32_t* ids, double* scores)
{
    int64_t h = d->h, E = d->E, k = d->k;
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t t = 0; t < ntok; t++) {
        double* lg = logits + t * E;
        for (int64_t e = 0; e < E; e++) {
            double s = 0.0;
            for (int64_t c = 0; c < h; c++) s += load(x, t * h + c, d->in_dtype) * load(wr, e * h + c, d->in_dtype);
            lg[e] = s;
        }
        /* selection: k passes of argmax over the not-yet-chosen experts */
        for (int64_t j = 0; j < k; j++) {
            int64_t best = -1;
            for (int64_t e = 0; e < E; e++) {
                int taken = 0;
                for (int64_t q = 0; q < j; q++) if (ids[t * k + q] == e) taken = 1;
                if (taken) continue;
                if (best < 0 || lg[e] > lg[best]) best = e;
            }
            ids[t * k + j] = (int32_t)best;
        }
        double mx = lg[ids[t * k]], z = 0.0;
        for (int64_t j = 0; j < k; j++) z += exp(lg[ids[t * k + j]] - mx);
        for (int64_t j = 0; j < k; j++) scores[t * k + j] = exp(lg[ids[t * k + j]] - mx) / z;
    }
}

/* Router backward given d_score (the MoE layer's dL/dw) for the selected slots:
 *   d_logit[e_j] = s_j (ds_j - sum_q s_q ds_q) for the selected e_j, 0 elsewhere (softmax Jacobian);
 *   dx = d_logits W_r,  dW_r = d_logits^T x. */
void oracle_router_backward(const oracle_dims* d, int64_t ntok, const void* x, const void* wr, const int32_t* ids,
                            const double* scores, const double* dscore, double* dx, double* dwr)
{
    int64_t h = d->h, E = d->E, k = d->k;
    double* dl = (double*)calloc((size_t)(ntok > 0 ? ntok : 1) * E, sizeof(double));
    for (int64_t t = 0; t < ntok; t++) {
        double dot = 0.0;
        for (int64_t j = 0; j < k; j++) dot += scores[t * k + j] * dscore[t * k + j];
        for (int64_t j = 0; j < k; j++) dl[t * E + ids[t * k + j]] += scores[t * k + j] * (dscore[t * k + j] - dot);
    }
    #pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < ntok; t++)
        for (int64_t c = 0; c < h; c++) {
            double s = 0.0;
            for (int64_t e = 0; e < E; e++) s += dl[t * E + e] * load(wr, e * h + c, d->in_dtype);
            dx[t * h + c] = s;
        }
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; e++)
        for (int64_t c = 0; c < h; c++) {
            double s = 0.0;
            for (int64_t t = 0; t < ntok; t++) s += dl[t * E + e] * load(x, t * h + c, d->in_dtype);
            dwr[e * h + c] = s;
        }
    free(dl);
}

/* ------------------------------------------------------------------------- */
/* MXFP8 variant of the expert GEMMs (reading R28). */
/* The paper trains in BF16 and says nothing about FP8; this    */
/* variant is this build's extension, defined here as:                          */
/*  - blocks of 32 consecutive elements along each GEMM's contraction dim K;    */
/*  - one shared power-of-two scale X = 2^E per block (E8M0), E the smallest    */
/*    integer with amax <= 448 * 2^E (no element clips), E clamped to [-127,127]*/
/*    and E = 0 for an all-zero block;                                          */
/*  - elements v / X rounded to FP8 E4M3 (bias 7, max 448, no inf) by          */
/*    round-to-nearest-even, saturating at +-448;  dequant = e4m3(code) * X.    */
/* Quantised operands: forward/recompute x and W_gate/W_up rows along h, a and */
/* W_down rows along g; backward dX: dG/dU and W_gate/W_up columns along g;    */
/* weight gradients (wgrad_C >= 1, reading R28c): x, dY, dG/dU and a_w columns  */
/* along the copies (tokens) of each expert in each chunk.  The dA GEMM         */
/* (dY W_down, epilogue-bound) keeps unquantised operands.                      */
/* mode 0 replaces every quantiser by the identity (then these functions equal */
/* oracle_moe_forward / oracle_moe_tokens exactly) - a structural pin.          */
/* ------------------------------------------------------------------------- */
double oracle_e4m3_decode(uint8_t c)
{
    int sgn = c >> 7, ex = (c >> 3) & 15, m = c & 7;
    if (ex == 15 && m == 7) return NAN;
    double v = ex == 0 ? ldexp((double)m / 8.0, -6) : ldexp(1.0 + (double)m / 8.0, ex - 7);
    return sgn ? -v : v;
}

/* round-to-nearest-even onto the E4M3 grid, saturating at 448 */
uint8_t oracle_e4m3_encode(double v)
{
    uint8_t sgn = (v < 0.0 || (v == 0.0 && signbit(v))) ? 0x80 : 0;
    double a = fabs(v);
    if (!(a == a)) return 0x7F;                           /* NaN */
    if (a >= 448.0) return (uint8_t)(sgn | 0x7E);
    int e = a > 0.0 ? ilogb(a) : -6;                      /* binade of a */
    if (e < -6) e = -6;                                   /* subnormal quantum 2^-9 */
    double q = ldexp(1.0, e - 3);                         /* spacing in this binade */
    double r = nearbyint(a / q);                          /* ties to even (default rounding mode) */
    double val = r * q;                                   /* may step up into the next binade */
    if (val > 448.0) val = 448.0;
    /* encode val exactly */
    if (val == 0.0) return sgn;
    int ev = ilogb(val);
    if (ev < -6) return (uint8_t)(sgn | (uint8_t)(val / ldexp(1.0, -9)));   /* subnormal: m * 2^-9 */
    int m = (int)(ldexp(val, -ev) * 8.0 - 8.0);
    return (uint8_t)(sgn | (uint8_t)((ev + 7) << 3) | (uint8_t)m);
}

/* E of one block from its amax: smallest integer E with amax <= 448 * 2^E */
int32_t oracle_mx_scale_exp(double amax)
{
    if (amax == 0.0) return 0;
    int e0 = ilogb(amax);
    double mant = ldexp(amax, -e0);                       /* [1, 2) */
    int e = e0 - 8 + (mant > 1.75 ? 1 : 0);
    if (e < -127) e = -127;
    if (e > 127) e = 127;
    return e;
}

/* Quantise n values (n % 32 == 0, consecutive = one block per 32) from in_dtype
 * storage: codes[n], scale codes[n / 32] (E + 127). */
void oracle_mx_quantize(const void* v, int32_t in_dtype, int64_t n, uint8_t* codes, uint8_t* scales)
{
    for (int64_t b = 0; b < n / 32; b++) {
        double amax = 0.0;
        for (int i = 0; i < 32; i++) amax = fmax(amax, fabs(load(v, b * 32 + i, in_dtype)));
        int32_t E = oracle_mx_scale_exp(amax);
        scales[b] = (uint8_t)(E + 127);
        for (int i = 0; i < 32; i++) codes[b * 32 + i] = oracle_e4m3_encode(ldexp(load(v, b * 32 + i, in_dtype), -E));
    }
}

/* Every quantiser below acts on the EXACT value of its operand (fp64 here), as the definition
 * above states; an implementation that holds the operand in a narrower format before quantising
 * may decide a neighbouring code at a near-tie.  For parity against such an implementation the
 * layer functions accept the other side's decisions ("fed" codes, dequantised per copy) and also
 * return the exact pre-quantisation values, so a test can (i) check every fed code against the
 * exact value it encodes and (ii) compare everything downstream of the decisions.  Without fed
 * codes the oracle decides every code itself. */
typedef struct {
    const double* a_q;       /* [nq][g]  a (forward, along g), dequantised                   */
    const double* dgu_q;     /* [nq][2g] dG || dU (dX operand, along g), dequantised          */
    const double* dgu_col_q; /* [nq][2g] dG || dU columnwise (R28c weight gradients)          */
    const double* aw_col_q;  /* [nq][g]  a_w = w a columnwise (R28c)                          */
} oracle_mx_fed;
typedef struct {
    double* a;               /* [nq][g]  exact a = silu(G) U                                  */
    double* dgu;             /* [nq][2g] exact dG || dU                                       */
    double* gu;              /* [nq][2g] exact G || U (what a, dG, dU are functions of)        */
    double* da;              /* [nq][g]  exact dA = w W_down^T dY                             */
} oracle_mx_exact;

/* quantise-dequantise n strided doubles in place (blocks of 32 along the stride) */
static void mx_qdq(double* v, int64_t n, int64_t stride, int mode)
{
    if (!mode) return;
    for (int64_t b = 0; b < n / 32; b++) {
        double amax = 0.0;
        for (int i = 0; i < 32; i++) amax = fmax(amax, fabs(v[(b * 32 + i) * stride]));
        int32_t E = oracle_mx_scale_exp(amax);
        for (int i = 0; i < 32; i++) {
            double* p = v + (b * 32 + i) * stride;
            *p = ldexp(oracle_e4m3_decode(oracle_e4m3_encode(ldexp(*p, -E))), E);
        }
    }
}

/* Dequantised weights of all E experts, fp64, 5 arrays:
 *  wq[0] W_gate rows along h [E][g][h]   wq[3] W_gate columns along g [E][g][h]
 *  wq[1] W_up   rows along h              wq[4] W_up columns along g
 *  wq[2] W_down rows along g [E][h][g] */
void oracle_mx_weights(const oracle_dims* d, int32_t mode, const void* wg, const void* wu, const void* wd,
                       double* const* wq)
{
    int64_t h = d->h, g = d->g, E = d->E, n = E * g * h;
    for (int64_t i = 0; i < n; i++) {
        wq[0][i] = wq[3][i] = load(wg, i, d->in_dtype);
        wq[1][i] = wq[4][i] = load(wu, i, d->in_dtype);
        wq[2][i] = load(wd, i, d->in_dtype);
    }
    for (int64_t e = 0; e < E; e++) {
        for (int64_t r = 0; r < g; r++) {       /* gate/up rows: contiguous h */
            mx_qdq(wq[0] + (e * g + r) * h, h, 1, mode);
            mx_qdq(wq[1] + (e * g + r) * h, h, 1, mode);
        }
        for (int64_t c = 0; c < h; c++) {       /* gate/up columns: stride h over g */
            mx_qdq(wq[3] + e * g * h + c, g, h, mode);
            mx_qdq(wq[4] + e * g * h + c, g, h, mode);
        }
        for (int64_t r = 0; r < h; r++) mx_qdq(wq[2] + (e * h + r) * g, g, 1, mode);   /* down rows */
    }
}

/* One copy, MX variant: forward (o), backward (dx term, d_score, and the exact dW operands a,
 * dO, dG, dU).  Same loop orders as expert_forward / expert_backward, quantisers inserted.
 * aq_in / dgq_in: fed dequantised a [g] / dG || dU [2g] (NULL: quantise the exact values). */
static void expert_mx(const oracle_dims* d, int mode, const void* x, int64_t xoff, const void* dy, int64_t dyoff,
                      double ws, double* const* wq, int32_t ew, const void* wd, int32_t e, double* scratch,
                      double* O, double* a_out, double* dO_out, double* dG_out, double* dU_out, double* dxc,
                      double* dscore, const double* aq_in, const double* dgq_in, double* gu_out, double* da_out)
{
    int64_t h = d->h, g = d->g;
    double *xq = scratch, *G = xq + h, *U = G + g, *A = U + g, *Aq = A + g, *dyq = Aq + g, *dA = dyq + h;
    double *dGq = dA + g, *dUq = dGq + g;
    for (int64_t c = 0; c < h; c++) xq[c] = load(x, xoff + c, d->in_dtype);
    mx_qdq(xq, h, 1, mode);
    for (int64_t n = 0; n < g; n++) {
        double sg = 0.0, su = 0.0;
        for (int64_t c = 0; c < h; c++) {
            sg += wq[0][((int64_t)ew * g + n) * h + c] * xq[c];
            su += wq[1][((int64_t)ew * g + n) * h + c] * xq[c];
        }
        G[n] = sg; U[n] = su;
        A[n] = sg * sigmoid(sg) * su;
        Aq[n] = aq_in ? aq_in[n] : A[n];
    }
    if (!aq_in) mx_qdq(Aq, g, 1, mode);
    for (int64_t m = 0; m < h; m++) {
        double so = 0.0;
        for (int64_t n = 0; n < g; n++) so += wq[2][((int64_t)ew * h + m) * g + n] * Aq[n];
        O[m] = so;
    }
    for (int64_t n = 0; n < g; n++) a_out[n] = A[n];
    if (gu_out) { memcpy(gu_out, G, sizeof(double) * (size_t)g); memcpy(gu_out + g, U, sizeof(double) * (size_t)g); }
    if (!dy) return;
    for (int64_t m = 0; m < h; m++) dyq[m] = load(dy, dyoff + m, d->in_dtype);   /* dA: unquantised */
    /* u = W_down^T dY (BF16 operands);  d_score = <u, a>;  dA = w u (reading R15) */
    double dwv = 0.0;
    for (int64_t n = 0; n < g; n++) {
        double s = 0.0;
        for (int64_t m = 0; m < h; m++) s += load(wd, ((int64_t)e * h + m) * g + n, d->in_dtype) * dyq[m];
        dwv += s * A[n];
        dA[n] = ws * s;
    }
    *dscore = dwv;
    if (da_out) memcpy(da_out, dA, sizeof(double) * (size_t)g);
    for (int64_t m = 0; m < h; m++) dO_out[m] = ws * load(dy, dyoff + m, d->in_dtype);
    for (int64_t n = 0; n < g; n++) {
        double sg = sigmoid(G[n]);
        dG_out[n] = dA[n] * U[n] * sg * (1.0 + G[n] * (1.0 - sg));
        dU_out[n] = dA[n] * G[n] * sg;
        dGq[n] = dgq_in ? dgq_in[n] : dG_out[n];
        dUq[n] = dgq_in ? dgq_in[g + n] : dU_out[n];
    }
    if (!dgq_in) {
        mx_qdq(dGq, g, 1, mode);
        mx_qdq(dUq, g, 1, mode);
    }
    for (int64_t c = 0; c < h; c++) {
        double s1 = 0.0, s2 = 0.0;
        for (int64_t n = 0; n < g; n++) {
            s1 += wq[3][((int64_t)ew * g + n) * h + c] * dGq[n];
            s2 += wq[4][((int64_t)ew * g + n) * h + c] * dUq[n];
        }
        dxc[c] = s1 + s2;
    }
}

/* MXFP8 weight gradients (reading R28c; the Transformer-Engine-style "columnwise"
 * operands): W_grad = sum over chunks (reading R18), and inside chunk j (partition of reading R1)
 * the K dimension of expert e's weight-gradient GEMMs is its copies in the canonical order
 * (src rank, token, slot; reading R3).  Every operand column is quantised in blocks of 32
 * consecutive copies counted from the start of that list (the last block zero-padded - the
 * 128-row segment padding).  Operands: x and dY (the layer's inputs), dG, dU and a_w = w a, all
 * exact values (or, for dG || dU and a_w, the fed dequantised columnwise values).
 * dW_gate[e] += dG^T x, dW_up[e] += dU^T x, dW_down[e] += dY^T a_w, accumulated in fp64.
 * mode 0: no quantiser - then this equals accumulate_dw up to summation order. */
static int accumulate_dw_mx(const oracle_dims* d, int mode, int32_t C, const void* x, const void* dy,
                            const int32_t* ids, const double* w, const double* a_all, const double* dG_all,
                            const double* dU_all, const oracle_mx_fed* fed, double* dwg, double* dwu, double* dwd)
{
    int64_t h = d->h, g = d->g, E = d->E, k = d->k, T = d->T, EP = d->EP;
    memset(dwg, 0, sizeof(double) * (size_t)E * g * h);
    memset(dwu, 0, sizeof(double) * (size_t)E * g * h);
    memset(dwd, 0, sizeof(double) * (size_t)E * h * g);
    int64_t nq = EP * T * k;
    const int fed_gu = fed && fed->dgu_col_q, fed_aw = fed && fed->aw_col_q;
    int64_t* list = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nq > 0 ? nq : 1));
    double* Xb = (double*)malloc(sizeof(double) * (size_t)32 * (2 * h + 3 * g));
    if (!list || !Xb) { free(list); free(Xb); return 1; }
    double *Yb = Xb + 32 * h, *Gb = Yb + 32 * h, *Ub = Gb + 32 * g, *Ab = Ub + 32 * g;
    for (int32_t j = 0; j < C; j++) {
        int64_t t0 = oracle_chunk_begin(T, C, j), t1 = oracle_chunk_begin(T, C, j + 1);
        for (int32_t e = 0; e < E; e++) {
            int64_t n = 0;
            for (int64_t r = 0; r < EP; r++)
                for (int64_t t = t0; t < t1; t++)
                    for (int64_t sl = 0; sl < k; sl++) {
                        int64_t q = (r * T + t) * k + sl;
                        if (ids[q] == e) list[n++] = q;
                    }
            for (int64_t b0 = 0; b0 < n; b0 += 32) {
                int64_t nb = n - b0 < 32 ? n - b0 : 32;
                for (int64_t i = 0; i < 32; i++) {
                    int64_t q = i < nb ? list[b0 + i] : -1;
                    int64_t tok = q >= 0 ? q / k : 0;
                    for (int64_t c = 0; c < h; c++) {
                        Xb[i * h + c] = q >= 0 ? load(x, tok * h + c, d->in_dtype) : 0.0;
                        Yb[i * h + c] = q >= 0 ? load(dy, tok * h + c, d->in_dtype) : 0.0;
                    }
                    for (int64_t c = 0; c < g; c++) {
                        Gb[i * g + c] = q < 0 ? 0.0 : fed_gu ? fed->dgu_col_q[q * 2 * g + c] : dG_all[q * g + c];
                        Ub[i * g + c] = q < 0 ? 0.0 : fed_gu ? fed->dgu_col_q[q * 2 * g + g + c] : dU_all[q * g + c];
                        Ab[i * g + c] = q < 0 ? 0.0 : fed_aw ? fed->aw_col_q[q * g + c] : w[q] * a_all[q * g + c];
                    }
                }
                /* columnwise blocks: 32 rows of one column (stride = the row length) */
                for (int64_t c = 0; c < h; c++) { mx_qdq(Xb + c, 32, h, mode); mx_qdq(Yb + c, 32, h, mode); }
                for (int64_t c = 0; c < g; c++) {
                    if (!fed_gu) { mx_qdq(Gb + c, 32, g, mode); mx_qdq(Ub + c, 32, g, mode); }
                    if (!fed_aw) mx_qdq(Ab + c, 32, g, mode);
                }
                #pragma omp parallel for schedule(static)
                for (int64_t nn = 0; nn < g; nn++) {
                    double* rg = dwg + ((int64_t)e * g + nn) * h;
                    double* ru = dwu + ((int64_t)e * g + nn) * h;
                    for (int64_t i = 0; i < nb; i++) {
                        double gv = Gb[i * g + nn], uv = Ub[i * g + nn];
                        for (int64_t c = 0; c < h; c++) { rg[c] += gv * Xb[i * h + c]; ru[c] += uv * Xb[i * h + c]; }
                    }
                }
                #pragma omp parallel for schedule(static)
                for (int64_t m = 0; m < h; m++) {
                    double* rd = dwd + ((int64_t)e * h + m) * g;
                    for (int64_t i = 0; i < nb; i++) {
                        double yv = Yb[i * h + m];
                        for (int64_t c = 0; c < g; c++) rd[c] += yv * Ab[i * g + c];
                    }
                }
            }
        }
    }
    free(list); free(Xb);
    return 0;
}

/* MX variant of the whole layer: y, and (dy != NULL) dx, dscore and dW.  wgrad_C = 0: dW from
 * unquantised operands in the canonical copy order (accumulate_dw); wgrad_C >= 1: MXFP8
 * weight gradients over the chunk partition with C = wgrad_C (accumulate_dw_mx).  Outputs as
 * oracle_moe_forward / oracle_moe_backward.  wq from oracle_mx_weights with the same mode; wd the
 * unquantised W_down (in_dtype) for the dA step.  fed (nullable, members nullable): another
 * implementation's decisions, dequantised per copy q = (src*T + i)*k + slot; ex (nullable, members
 * nullable): the exact a, dG || dU, G || U and dA per copy (a and G || U also without dy). */
int32_t oracle_moe_mx(const oracle_dims* d, int32_t mode, const void* dy, const void* x, const int32_t* ids,
                      const double* w, double* const* wq, const void* wd, double* y, double* dx, double* dscore,
                      double* dwg, double* dwu, double* dwd, int32_t wgrad_C, const oracle_mx_fed* fed,
                      const oracle_mx_exact* ex)
{
    int64_t h = d->h, g = d->g, ntok = (int64_t)d->EP * d->T, nq = ntok * d->k;
    double *a_all = NULL, *dG_all = NULL, *dU_all = NULL, *dO_all = NULL;
    int64_t* order = NULL;
    if (dy) {
        a_all = (double*)malloc(sizeof(double) * (size_t)(nq > 0 ? nq : 1) * g);
        dG_all = (double*)malloc(sizeof(double) * (size_t)(nq > 0 ? nq : 1) * g);
        dU_all = (double*)malloc(sizeof(double) * (size_t)(nq > 0 ? nq : 1) * g);
        dO_all = (double*)malloc(sizeof(double) * (size_t)(nq > 0 ? nq : 1) * h);
        order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nq > 0 ? nq : 1));
        if (!a_all || !dG_all || !dU_all || !dO_all || !order) {
            free(a_all); free(dG_all); free(dU_all); free(dO_all); free(order);
            return 1;
        }
    }
    #pragma omp parallel
    {
        double* scratch = (double*)malloc(sizeof(double) * (size_t)(8 * g + 2 * h));
        double* O = (double*)malloc(sizeof(double) * (size_t)(2 * h + 3 * g + h));
        double *dxc = O + h, *a1 = dxc + h, *dG1 = a1 + g, *dU1 = dG1 + g, *dO1 = dU1 + g;
        #pragma omp for schedule(dynamic, 1)
        for (int64_t t = 0; t < ntok; t++) {
            for (int64_t c = 0; c < h; c++) { y[t * h + c] = 0.0; if (dy) dx[t * h + c] = 0.0; }
            for (int32_t s = 0; s < d->k; s++) {
                int64_t q = t * d->k + s;
                int32_t e = ids[q];
                if (dy) dscore[q] = 0.0;
                double *aq = dy ? a_all + q * g : a1, *dGq = dy ? dG_all + q * g : dG1;
                double *dUq = dy ? dU_all + q * g : dU1, *dOq = dy ? dO_all + q * h : dO1;
                if (e < 0 || e >= d->E) {
                    if (dy) {
                        memset(aq, 0, sizeof(double) * (size_t)g); memset(dGq, 0, sizeof(double) * (size_t)g);
                        memset(dUq, 0, sizeof(double) * (size_t)g); memset(dOq, 0, sizeof(double) * (size_t)h);
                    }
                    if (ex && ex->a) memset(ex->a + q * g, 0, sizeof(double) * (size_t)g);
                    if (ex && ex->dgu) memset(ex->dgu + q * 2 * g, 0, sizeof(double) * (size_t)(2 * g));
                    if (ex && ex->gu) memset(ex->gu + q * 2 * g, 0, sizeof(double) * (size_t)(2 * g));
                    if (ex && ex->da) memset(ex->da + q * g, 0, sizeof(double) * (size_t)g);
                    continue;
                }
                expert_mx(d, mode, x, t * h, dy, t * h, w[q], wq, e, wd, e, scratch, O, aq, dOq, dGq, dUq, dxc,
                          dy ? dscore + q : NULL, fed && fed->a_q ? fed->a_q + q * g : NULL,
                          fed && fed->dgu_q ? fed->dgu_q + q * 2 * g : NULL,
                          ex && ex->gu ? ex->gu + q * 2 * g : NULL, ex && ex->da && dy ? ex->da + q * g : NULL);
                if (ex && ex->a) memcpy(ex->a + q * g, aq, sizeof(double) * (size_t)g);
                if (ex && ex->dgu && dy) {
                    memcpy(ex->dgu + q * 2 * g, dGq, sizeof(double) * (size_t)g);
                    memcpy(ex->dgu + q * 2 * g + g, dUq, sizeof(double) * (size_t)g);
                }
                for (int64_t c = 0; c < h; c++) {
                    y[t * h + c] += w[q] * O[c];
                    if (dy) dx[t * h + c] += dxc[c];
                }
            }
        }
        free(scratch); free(O);
    }
    int32_t rc = 0;
    if (dy) {
        for (int64_t q = 0; q < nq; q++) order[q] = q;
        if (wgrad_C >= 1)
            rc = accumulate_dw_mx(d, mode, wgrad_C, x, dy, ids, w, a_all, dG_all, dU_all, fed, dwg, dwu, dwd);
        else
            accumulate_dw(d, x, ids, order, nq, a_all, dO_all, dG_all, dU_all, dwg, dwu, dwd);
        free(a_all); free(dG_all); free(dU_all); free(dO_all); free(order);
    }
    return rc;
}

/* MX layer on a token subset (full-size sampled parity): y, dx, dscore of tokens toks[0..ntok) exactly
 * as oracle_moe_mx computes them (the per-token terms do not depend on other tokens), with the
 * weights quantised one expert at a time (the five operand layouts of oracle_mx_weights), so the
 * dequantised copies of all experts never exist at once.  fed / ex as in oracle_moe_mx, indexed by
 * the sampled copy p*k + slot (a_q, dgu_q only; ex->a, ex->dgu). */
int32_t oracle_moe_mx_tokens(const oracle_dims* d, int32_t mode, int64_t ntok, const int64_t* toks, const void* dy,
                             const void* x, const int32_t* ids, const double* w, const void* wg, const void* wu,
                             const void* wd, double* y, double* dx, double* dscore, const oracle_mx_fed* fed,
                             const oracle_mx_exact* ex)
{
    int64_t h = d->h, g = d->g, k = d->k;
    double* wqe[5];
    for (int i = 0; i < 5; i++) wqe[i] = (double*)malloc(sizeof(double) * (size_t)g * h);
    double* scratch = (double*)malloc(sizeof(double) * (size_t)(8 * g + 2 * h));
    double* O = (double*)malloc(sizeof(double) * (size_t)(2 * h + 4 * g + h));
    int ok = scratch && O;
    for (int i = 0; i < 5; i++) ok = ok && wqe[i];
    if (!ok) {
        for (int i = 0; i < 5; i++) free(wqe[i]);
        free(scratch); free(O);
        return 1;
    }
    double *dxc = O + h, *a1 = dxc + h, *dG1 = a1 + g, *dU1 = dG1 + g, *dO1 = dU1 + g;
    for (int64_t i = 0; i < ntok * h; i++) { y[i] = 0.0; if (dy) dx[i] = 0.0; }
    for (int32_t e = 0; e < d->E; e++) {
        int used = 0;
        for (int64_t i = 0; i < ntok && !used; i++)
            for (int64_t sl = 0; sl < k; sl++) used |= ids[toks[i] * k + sl] == e;
        if (!used) continue;
        int64_t off = (int64_t)e * g * h;
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < g * h; i++) {
            wqe[0][i] = wqe[3][i] = load(wg, off + i, d->in_dtype);
            wqe[1][i] = wqe[4][i] = load(wu, off + i, d->in_dtype);
            wqe[2][i] = load(wd, off + i, d->in_dtype);
        }
        #pragma omp parallel for schedule(dynamic, 16)
        for (int64_t r = 0; r < g; r++) { mx_qdq(wqe[0] + r * h, h, 1, mode); mx_qdq(wqe[1] + r * h, h, 1, mode); }
        #pragma omp parallel for schedule(dynamic, 16)
        for (int64_t c = 0; c < h; c++) { mx_qdq(wqe[3] + c, g, h, mode); mx_qdq(wqe[4] + c, g, h, mode); }
        #pragma omp parallel for schedule(dynamic, 16)
        for (int64_t r = 0; r < h; r++) mx_qdq(wqe[2] + r * g, g, 1, mode);
        for (int64_t i = 0; i < ntok; i++) {
            int64_t t = toks[i];
            for (int64_t sl = 0; sl < k; sl++) {
                int64_t q = t * k + sl, p = i * k + sl;
                if (ids[q] != e) continue;
                expert_mx(d, mode, x, t * h, dy, t * h, w[q], wqe, 0, wd, e, scratch, O, a1, dO1, dG1, dU1, dxc,
                          dy ? dscore + p : NULL, fed && fed->a_q ? fed->a_q + p * g : NULL,
                          fed && fed->dgu_q ? fed->dgu_q + p * 2 * g : NULL,
                          ex && ex->gu ? ex->gu + p * 2 * g : NULL, ex && ex->da && dy ? ex->da + p * g : NULL);
                if (ex && ex->a) memcpy(ex->a + p * g, a1, sizeof(double) * (size_t)g);
                if (ex && ex->dgu && dy) {
                    memcpy(ex->dgu + p * 2 * g, dG1, sizeof(double) * (size_t)g);
                    memcpy(ex->dgu + p * 2 * g + g, dU1, sizeof(double) * (size_t)g);
                }
                for (int64_t c = 0; c < h; c++) {
                    y[i * h + c] += w[q] * O[c];
                    if (dy) dx[i * h + c] += dxc[c];
                }
            }
        }
    }
    for (int i = 0; i < 5; i++) free(wqe[i]);
    free(scratch); free(O);
    return 0;
}

/* Eq. 2's m_g (§3): "Generally, m_g = (v p + p - 2 r_pp - 1), and when full
 * recomputation is employed, then m_g = 1."  r_pp: the pipeline stage, 0-based (reading R29). */
int32_t oracle_m_g(int32_t v, int32_t p, int32_t r_pp, int32_t full_recompute)
{
    if (full_recompute) return 1;
    return v * p + p - 2 * r_pp - 1;
}

int32_t oracle_version(void) { return 1; }

#ifdef _OPENMP
#include <omp.h>
#endif
/* Threads the OpenMP loops above use (reported as cpu_baseline.cores). */
int32_t oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
