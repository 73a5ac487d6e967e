/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain loops, no BLAS, no blocking, no reordering beyond what the paper's
 * algorithms state.  Built with  gcc -O2 -fno-fast-math -ffp-contract=off.
 * Each function cites the passage of /root/reference/PAPER.md it follows.
 */
#include "oracle.h"
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define AT(a, i, j, ld) ((a)[(size_t)(i) + (size_t)(j) * (size_t)(ld)])

/* House(w): Alg. QR:qnxn line 4, with LAPACK dlarfg's sign choice
 * (reading R1) and the zero-tail rule of reading R2. */
void orc_house(int64_t len, double *x, double *tau, double *beta)
{
    double alpha = x[0];
    long double sigma2 = 0.0L;
    for (int64_t i = 1; i < len; ++i)
        sigma2 += (long double)x[i] * (long double)x[i];
    if (sigma2 == 0.0L) {           /* H = I: nothing to annihilate */
        *tau = 0.0;
        *beta = alpha;
        return;
    }
    long double norm = sqrtl((long double)alpha * (long double)alpha + sigma2);
    double b = (double)(alpha >= 0.0 ? -norm : norm);   /* beta = -sign(alpha)||w|| */
    *tau = (b - alpha) / b;
    double denom = alpha - b;                            /* v = (w - beta e0)/(alpha - beta) */
    for (int64_t i = 1; i < len; ++i)
        x[i] = x[i] / denom;
    *beta = b;
}

/* Unblocked Householder QR (DGEQR2): the local "sequential Householder QR" of
 * Alg. TSQR:par line 1; reflectors overwrite the lower trapezoid,
 * tau stored separately. */
void orc_hqr(int64_t m, int64_t n, double *A, int64_t lda, double *tau)
{
    for (int64_t j = 0; j < n; ++j) {
        double t, beta;
        orc_house(m - j, &AT(A, j, j, lda), &t, &beta);
        tau[j] = t;
        /* A(j:m, j+1:n) := (I - tau v v^T) A(j:m, j+1:n), v = [1; A(j+1:m, j)] */
        for (int64_t c = j + 1; c < n; ++c) {
            long double w = AT(A, j, c, lda);
            for (int64_t i = j + 1; i < m; ++i)
                w += (long double)AT(A, i, j, lda) * (long double)AT(A, i, c, lda);
            double tw = t * (double)w;
            AT(A, j, c, lda) -= tw;
            for (int64_t i = j + 1; i < m; ++i)
                AT(A, i, c, lda) -= AT(A, i, j, lda) * tw;
        }
        AT(A, j, j, lda) = beta;
    }
}

/* Rows of reflector j of chunk k of a tile's flat chain (orc_chain_qr): the
 * chunk is rows [r0, r0 + h).  j < r0: "structured" -- pivot row j (the
 * running R's row j, kept in place in the tile's head) and tail = the whole
 * chunk; r0 <= j < r0 + h: "dense" -- pivot row j inside the chunk, tail =
 * rows j+1 .. r0+h-1; otherwise no reflector.  Returns the tail length
 * (-1: no reflector) and the first tail row in *t0. */
static int64_t chain_rows(int64_t j, int64_t r0, int64_t h, int64_t *t0)
{
    if (j < r0) { *t0 = r0; return h; }
    if (j < r0 + h) { *t0 = j + 1; return r0 + h - j - 1; }
    return -1;
}

static int64_t chunks_of(int64_t rows, int64_t c)
{
    return c <= 0 ? 1 : (rows + c - 1) / c;
}

/* Flat-tree ("sequential") TSQR of one tile ([TR] Alg. sequential
 * TSQR P:1725-1753) over chunks of c consecutive rows: chunk k (rows
 * r0 = k c .. r0 + h - 1) is merged into the running R by qr([R; A_k]), one
 * Householder reflector per column j = 0..n-1 on the rows chain_rows gives
 * (the structure of [R; A_k]: R upper trapezoidal, its row j being the tile's
 * row j).  c <= 0 (or c >= rows): one chunk, i.e. orc_hqr.  On exit the tile
 * holds R in the upper triangle of its first n rows and every reflector's
 * tail below the diagonal (row > column) in place; tau[k*n + j] (0 for a
 * missing reflector). */
void orc_chain_qr(int64_t rows, int64_t n, double *A, int64_t lda, int64_t c, double *tau)
{
    const int64_t cc = c <= 0 ? rows : c;
    double *w = (double *)malloc((size_t)(cc + 1) * sizeof(double));
    for (int64_t k = 0, r0 = 0; r0 < rows; ++k, r0 += cc) {
        const int64_t h = rows - r0 < cc ? rows - r0 : cc;
        for (int64_t j = 0; j < n; ++j) {
            int64_t t0;
            const int64_t len = chain_rows(j, r0, h, &t0);
            if (len < 0) { tau[k * n + j] = 0.0; continue; }
            /* gather the pivot column (pivot row j, then the tail rows) */
            w[0] = AT(A, j, j, lda);
            for (int64_t i = 0; i < len; ++i) w[1 + i] = AT(A, t0 + i, j, lda);
            double t, beta;
            orc_house(len + 1, w, &t, &beta);
            for (int64_t col = j + 1; col < n; ++col) {
                long double d = AT(A, j, col, lda);
                for (int64_t i = 0; i < len; ++i)
                    d += (long double)w[1 + i] * (long double)AT(A, t0 + i, col, lda);
                double td = t * (double)d;
                AT(A, j, col, lda) -= td;
                for (int64_t i = 0; i < len; ++i) AT(A, t0 + i, col, lda) -= w[1 + i] * td;
            }
            AT(A, j, j, lda) = beta;
            for (int64_t i = 0; i < len; ++i) AT(A, t0 + i, j, lda) = w[1 + i];
            tau[k * n + j] = t;
        }
    }
    free(w);
}

/* Alg. QR:qnxn with q = 2: index set I_j = {j, n+1:n+j}
 * (P:1964-1965), i.e. row j of Ra and rows 0..j of Rb. */
void orc_combine(int64_t n, double *Ra, int64_t lda, double *Rb, int64_t ldb,
                 double *tau, double *flops)
{
    double fl = 0.0;
    double *w = (double *)malloc((size_t)(n + 1) * sizeof(double));
    for (int64_t j = 0; j < n; ++j) {
        /* w := A(I_j, j): gather the pivot column (line 3) */
        w[0] = AT(Ra, j, j, lda);
        for (int64_t i = 0; i <= j; ++i) w[1 + i] = AT(Rb, i, j, ldb);
        double t, beta;
        orc_house(j + 2, w, &t, &beta);                           /* line 4 */
        fl += 2.0 * (double)(j + 1) + 3.0 + (double)(j + 1);       /* norm, sqrt/div, scale */
        /* X := (I - tau v v^T) A(I_j, j+1:n)   (lines 5-6) */
        for (int64_t c = j + 1; c < n; ++c) {
            long double d = AT(Ra, j, c, lda);
            for (int64_t i = 0; i <= j; ++i)
                d += (long double)w[1 + i] * (long double)AT(Rb, i, c, ldb);
            double td = t * (double)d;
            AT(Ra, j, c, lda) -= td;
            for (int64_t i = 0; i <= j; ++i)
                AT(Rb, i, c, ldb) -= w[1 + i] * td;
            fl += 2.0 * (double)(j + 1) + 1.0 + 1.0 + 2.0 * (double)(j + 1) + 1.0;
        }
        /* scatter v(2:end) and the new diagonal (lines 7-8) */
        AT(Ra, j, j, lda) = beta;
        for (int64_t i = 0; i <= j; ++i) AT(Rb, i, j, ldb) = w[1 + i];
        tau[j] = t;
    }
    free(w);
    if (flops) *flops = fl;
}

/* dlarft-style T, LAPACK sign: Alg. YT:scaled computes
 * T' with T'(j,j) = -tau_j and rho_1...rho_n = I + Y T' Y^T; we store T = -T'
 * so that H_0...H_{k-1} = I - Y T Y^T (reading R3).  The recurrence is the
 * paper's line "z := -tau_j (T (Y^T v_j))" with that sign flip:
 *   T(0:j, j) = -tau_j * T(0:j, 0:j) * (Y(:,0:j)^T v_j),  T(j,j) = tau_j. */
static void build_t_from_gram(int64_t k, const long double *G, const double *tau,
                              double *T, int64_t ldt)
{
    /* G[i + j*k] = v_i^T v_j for i < j */
    for (int64_t j = 0; j < k; ++j) {
        for (int64_t i = 0; i < k; ++i) AT(T, i, j, ldt) = 0.0;
        for (int64_t i = 0; i < j; ++i) {
            long double s = 0.0L;
            for (int64_t l = i; l < j; ++l)
                s += (long double)AT(T, i, l, ldt) * G[l + j * k];
            AT(T, i, j, ldt) = (double)(-(long double)tau[j] * s);
        }
        AT(T, j, j, ldt) = tau[j];
    }
}

void orc_build_t(int64_t rows, int64_t k, const double *Y, int64_t ldy,
                 const double *tau, double *T, int64_t ldt)
{
    long double *G = (long double *)calloc((size_t)(k * k), sizeof(long double));
    for (int64_t j = 0; j < k; ++j)
        for (int64_t i = 0; i < j; ++i) {
            /* v_i = [0..0, 1 (row i), Y(i+1:, i)], v_j = [0..0, 1 (row j), Y(j+1:, j)] */
            long double s = (long double)AT(Y, j, i, ldy);          /* v_i(j) * v_j(j)=1 */
            for (int64_t r = j + 1; r < rows; ++r)
                s += (long double)AT(Y, r, i, ldy) * (long double)AT(Y, r, j, ldy);
            G[i + j * k] = s;
        }
    build_t_from_gram(k, G, tau, T, ldt);
    free(G);
}

void orc_build_t_node(int64_t n, const double *Y1, int64_t ldy, const double *tau,
                      double *T, int64_t ldt)
{
    long double *G = (long double *)calloc((size_t)(n * n), sizeof(long double));
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < j; ++i) {
            /* [e_i; y_i]^T [e_j; y_j] = y_i^T y_j, y_i nonzero in rows 0..i */
            long double s = 0.0L;
            for (int64_t r = 0; r <= i; ++r)
                s += (long double)AT(Y1, r, i, ldy) * (long double)AT(Y1, r, j, ldy);
            G[i + j * n] = s;
        }
    build_t_from_gram(n, G, tau, T, ldt);
    free(G);
}

/* ------------------------------- plan ------------------------------------ */

typedef struct {
    int64_t ntiles, nnodes;
    int64_t *tile_row0, *tile_rows, *tile_rank;
    int64_t *node_a, *node_b, *node_stage, *node_level;
    int count_only;
} plan_out;

static void emit_node(plan_out *p, int64_t a, int64_t b, int64_t stage, int64_t level)
{
    if (!p->count_only) {
        p->node_a[p->nnodes] = a;
        p->node_b[p->nnodes] = b;
        p->node_stage[p->nnodes] = stage;
        p->node_level[p->nnodes] = level;
    }
    p->nnodes++;
}

/* binary reduction of list[0..len) with pairing (2i, 2i+1) and the odd
 * trailing entry promoted unchanged (Alg. TSQR:par P:1693-1696; reading R5) */
static void reduce_binary(plan_out *p, int64_t *list, int64_t len, int64_t stage)
{
    int64_t level = 1;
    while (len > 1) {
        int64_t out = 0;
        for (int64_t i = 0; i < len; i += 2) {
            if (i + 1 < len) emit_node(p, list[i], list[i + 1], stage, level);
            list[out++] = list[i];
        }
        len = out;
        level++;
    }
}

static int build_plan(int64_t m, int64_t n, int64_t b, int64_t s, int64_t G, plan_out *p)
{
    if (n < 1 || m < n || b < 1 || s < 0 || G < 1) return -1;
    if ((G & (G - 1)) != 0) return -1;
    /* row blocks (reading R6) */
    int64_t nblk = m / b, rem = m - (m / b) * b;
    int64_t last_rows = b;
    if (nblk == 0) { nblk = 1; last_rows = m; }
    else if (rem >= n) { nblk += 1; last_rows = rem; }
    else if (rem > 0) { last_rows = b + rem; }
    if (nblk < G) return -1;
    int64_t *blk_row0 = (int64_t *)malloc((size_t)nblk * sizeof(int64_t));
    int64_t *blk_rows = (int64_t *)malloc((size_t)nblk * sizeof(int64_t));
    for (int64_t k = 0; k < nblk; ++k) {
        blk_row0[k] = k * b;
        blk_rows[k] = (k == nblk - 1) ? last_rows : b;
    }
    /* tiles */
    int64_t *blk_tile0 = (int64_t *)malloc((size_t)(nblk + 1) * sizeof(int64_t));
    int64_t nt = 0;
    for (int64_t k = 0; k < nblk; ++k) {
        blk_tile0[k] = nt;
        int64_t h = blk_rows[k];
        int64_t t = (s == 0) ? 1 : (h + s - 1) / s;   /* s = 0: one tile per block */
        if (t > h / n) t = h / n;                      /* never a tile shorter than n */
        if (t < 1) t = 1;
        /* near-equal tiles of EVEN height: the block's row pairs are split near-equally
         * (the first (h/2 mod t) tiles one pair taller), the last tile takes what is left
         * (one row more when h is odd); if that would leave a tile shorter than n, plain
         * near-equal heights (the first h mod t tiles one row taller) */
        int64_t base = h / t, extra = h - base * t;
        const int64_t pb = (h / 2) / t, pe = (h / 2) - pb * t;
        const int64_t last_even = h - 2 * (pb * (t - 1) + (pe < t - 1 ? pe : t - 1));
        const int even = t > 1 && 2 * pb >= n && last_even >= n;
        int64_t r0 = blk_row0[k];
        for (int64_t i = 0; i < t; ++i) {
            int64_t rows = base + (i < extra ? 1 : 0);
            if (even) rows = (i < t - 1) ? 2 * (pb + (i < pe ? 1 : 0)) : last_even;
            if (rows < n) { free(blk_row0); free(blk_rows); free(blk_tile0); return -1; }
            if (!p->count_only) { p->tile_row0[nt] = r0; p->tile_rows[nt] = rows; }
            r0 += rows;
            nt++;
        }
    }
    blk_tile0[nblk] = nt;
    p->ntiles = nt;
    /* ranks: contiguous runs of whole blocks */
    int64_t *rank_blk0 = (int64_t *)malloc((size_t)(G + 1) * sizeof(int64_t));
    {
        int64_t base = nblk / G, extra = nblk - base * G, k0 = 0;
        for (int64_t r = 0; r < G; ++r) {
            rank_blk0[r] = k0;
            k0 += base + (r < extra ? 1 : 0);
        }
        rank_blk0[G] = nblk;
    }
    if (!p->count_only)
        for (int64_t r = 0; r < G; ++r)
            for (int64_t k = rank_blk0[r]; k < rank_blk0[r + 1]; ++k)
                for (int64_t t = blk_tile0[k]; t < blk_tile0[k + 1]; ++t) p->tile_rank[t] = r;
    /* nodes */
    int64_t *list = (int64_t *)malloc((size_t)(nt + nblk + G + 1) * sizeof(int64_t));
    p->nnodes = 0;
    for (int64_t r = 0; r < G; ++r) {
        for (int64_t k = rank_blk0[r]; k < rank_blk0[r + 1]; ++k) {      /* stage 0 */
            int64_t len = 0;
            for (int64_t t = blk_tile0[k]; t < blk_tile0[k + 1]; ++t) list[len++] = t;
            reduce_binary(p, list, len, 0);
        }
        int64_t len = 0;                                                  /* stage 1 */
        for (int64_t k = rank_blk0[r]; k < rank_blk0[r + 1]; ++k) list[len++] = blk_tile0[k];
        reduce_binary(p, list, len, 1);
    }
    {
        int64_t len = 0;                                                  /* stage 2 */
        for (int64_t r = 0; r < G; ++r) list[len++] = blk_tile0[rank_blk0[r]];
        reduce_binary(p, list, len, 2);
    }
    free(list); free(rank_blk0); free(blk_tile0); free(blk_row0); free(blk_rows);
    return 0;
}

int orc_plan_count(int64_t m, int64_t n, int64_t b, int64_t s, int64_t G,
                   int64_t *ntiles, int64_t *nnodes)
{
    plan_out p;
    memset(&p, 0, sizeof(p));
    p.count_only = 1;
    int rc = build_plan(m, n, b, s, G, &p);
    *ntiles = p.ntiles;
    *nnodes = p.nnodes;
    return rc;
}

int orc_plan_fill(int64_t m, int64_t n, int64_t b, int64_t s, int64_t G,
                  int64_t *tile_row0, int64_t *tile_rows, int64_t *tile_rank,
                  int64_t *node_a, int64_t *node_b, int64_t *node_stage,
                  int64_t *node_level)
{
    plan_out p;
    memset(&p, 0, sizeof(p));
    p.tile_row0 = tile_row0; p.tile_rows = tile_rows; p.tile_rank = tile_rank;
    p.node_a = node_a; p.node_b = node_b; p.node_stage = node_stage; p.node_level = node_level;
    return build_plan(m, n, b, s, G, &p);
}

/* ------------------------------- TSQR ------------------------------------ */

/* Eqs. 1-4: every tile A_i = Q_i R_i, then stacked pairs of R's
 * are re-factored up the tree; the implicit Q is the tree of local factors. */
/* Eq. 1 for tiles [t0, t1): the leaf QRs, independent of one another. */
typedef struct {
    int64_t n, lda, c, t0, t1;
    double *A, *tau_tile, *Rsub;
    const int64_t *tile_row0, *tile_rows, *chunk0;
} leaf_job;

static void *leaf_range(void *arg)
{
    const leaf_job *J = (const leaf_job *)arg;
    const size_t nn = (size_t)(J->n * J->n);
    for (int64_t t = J->t0; t < J->t1; ++t) {
        double *At = J->A + J->tile_row0[t];
        orc_chain_qr(J->tile_rows[t], J->n, At, J->lda, J->c, J->tau_tile + J->chunk0[t] * J->n);
        for (int64_t j = 0; j < J->n; ++j)
            for (int64_t i = 0; i <= j; ++i) AT(J->Rsub + t * nn, i, j, J->n) = AT(At, i, j, J->lda);
    }
    return NULL;
}

void orc_tsqr_factor_mt(int64_t m, int64_t n, double *A, int64_t lda, int64_t c,
                        int64_t ntiles, const int64_t *tile_row0, const int64_t *tile_rows,
                        int64_t nnodes, const int64_t *node_a, const int64_t *node_b,
                        double *tau_tile, double *Y1, double *tau_node,
                        double *R, int64_t ldr, int64_t nthreads)
{
    (void)m;
    size_t nn = (size_t)(n * n);
    double *Rsub = (double *)calloc((size_t)ntiles * nn, sizeof(double));
    int64_t *chunk0 = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ntiles + 1));
    chunk0[0] = 0;
    for (int64_t t = 0; t < ntiles; ++t) chunk0[t + 1] = chunk0[t] + chunks_of(tile_rows[t], c);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > ntiles) nthreads = ntiles;
    leaf_job *jobs = (leaf_job *)malloc(sizeof(leaf_job) * (size_t)nthreads);
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int64_t w = 0; w < nthreads; ++w) {                     /* Eq. 1: contiguous runs of leaves */
        leaf_job J = {n, lda, c, ntiles * w / nthreads, ntiles * (w + 1) / nthreads,
                      A, tau_tile, Rsub, tile_row0, tile_rows, chunk0};
        jobs[w] = J;
    }
    for (int64_t w = 1; w < nthreads; ++w) pthread_create(&th[w], NULL, leaf_range, &jobs[w]);
    leaf_range(&jobs[0]);
    for (int64_t w = 1; w < nthreads; ++w) pthread_join(th[w], NULL);
    for (int64_t k = 0; k < nnodes; ++k) {                       /* Eqs. 2-3, in plan order */
        double *Ra = Rsub + node_a[k] * nn, *Rb = Rsub + node_b[k] * nn;
        orc_combine(n, Ra, n, Rb, n, tau_node + k * n, NULL);
        if (Y1) {
            double *Yk = Y1 + k * nn;
            for (int64_t j = 0; j < n; ++j)
                for (int64_t i = 0; i < n; ++i) AT(Yk, i, j, n) = (i <= j) ? AT(Rb, i, j, n) : 0.0;
        }
    }
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) AT(R, i, j, ldr) = (i <= j) ? AT(Rsub, i, j, n) : 0.0;
    free(th);
    free(jobs);
    free(chunk0);
    free(Rsub);
}

void orc_tsqr_factor(int64_t m, int64_t n, double *A, int64_t lda, int64_t c,
                     int64_t ntiles, const int64_t *tile_row0, const int64_t *tile_rows,
                     int64_t nnodes, const int64_t *node_a, const int64_t *node_b,
                     double *tau_tile, double *Y1, double *tau_node,
                     double *R, int64_t ldr)
{
    orc_tsqr_factor_mt(m, n, A, lda, c, ntiles, tile_row0, tile_rows, nnodes, node_a, node_b,
                       tau_tile, Y1, tau_node, R, ldr, 1);
}

/* reflector j of a tile chunk (rows from chain_rows, vector tail stored in
 * the tile below the diagonal) applied to the same rows of C: C -= tau v (v^T C) */
static void apply_chain_reflector(int64_t j, int64_t t0, int64_t len, const double *At, int64_t lda,
                                  double tau, double *Ct, int64_t ldc, int64_t k)
{
    if (tau == 0.0 || len < 0) return;
    for (int64_t c = 0; c < k; ++c) {
        long double w = AT(Ct, j, c, ldc);
        for (int64_t i = 0; i < len; ++i)
            w += (long double)AT(At, t0 + i, j, lda) * (long double)AT(Ct, t0 + i, c, ldc);
        double tw = tau * (double)w;
        AT(Ct, j, c, ldc) -= tw;
        for (int64_t i = 0; i < len; ++i) AT(Ct, t0 + i, c, ldc) -= AT(At, t0 + i, j, lda) * tw;
    }
}

/* Q_t^T C_t for one tile: chunks in order, reflectors j = 0..n-1 (forward), or
 * Q_t C_t: chunks and reflectors in reverse. */
static void apply_tile(int64_t rows, int64_t n, int64_t c, const double *At, int64_t lda,
                       const double *tau, double *Ct, int64_t ldc, int64_t k, int forward)
{
    const int64_t cc = c <= 0 ? rows : c;
    const int64_t nk = chunks_of(rows, c);
    for (int64_t kk = 0; kk < nk; ++kk) {
        const int64_t ck = forward ? kk : nk - 1 - kk;
        const int64_t r0 = ck * cc, h = rows - r0 < cc ? rows - r0 : cc;
        for (int64_t jj = 0; jj < n; ++jj) {
            const int64_t j = forward ? jj : n - 1 - jj;
            int64_t t0;
            const int64_t len = chain_rows(j, r0, h, &t0);
            apply_chain_reflector(j, t0, len, At, lda, tau[ck * n + j], Ct, ldc, k);
        }
    }
}

/* one node reflector j (vector [e_j; Y1(0:j, j)]) applied to the head rows
 * Ca (row j) and Cb (rows 0..j): eq. localQTupdate one column
 * of [I; Y1] at a time. */
static void apply_node_reflector(int64_t n, int64_t j, const double *Yk, double tau,
                                 double *Ca, double *Cb, int64_t ldc, int64_t k)
{
    (void)n;
    if (tau == 0.0) return;
    for (int64_t c = 0; c < k; ++c) {
        long double w = AT(Ca, j, c, ldc);
        for (int64_t i = 0; i <= j; ++i)
            w += (long double)AT(Yk, i, j, n) * (long double)AT(Cb, i, c, ldc);
        double tw = tau * (double)w;
        AT(Ca, j, c, ldc) -= tw;
        for (int64_t i = 0; i <= j; ++i) AT(Cb, i, c, ldc) -= AT(Yk, i, j, n) * tw;
    }
}

/* Q^T C: leaves first, then nodes bottom-up in factor order (Eq. 4 gives
 * A = Q_leaves Q_level1 ... Q_root R; reading R4). */
void orc_tsqr_apply_qt(int64_t m, int64_t n, const double *A, int64_t lda, int64_t c,
                       int64_t ntiles, const int64_t *tile_row0, const int64_t *tile_rows,
                       int64_t nnodes, const int64_t *node_a, const int64_t *node_b,
                       const double *tau_tile, const double *Y1, const double *tau_node,
                       double *C, int64_t ldc, int64_t k)
{
    (void)m;
    size_t nn = (size_t)(n * n);
    for (int64_t t = 0, ch0 = 0; t < ntiles; ch0 += chunks_of(tile_rows[t], c), ++t)
        apply_tile(tile_rows[t], n, c, A + tile_row0[t], lda, tau_tile + ch0 * n, C + tile_row0[t], ldc, k, 1);
    for (int64_t q = 0; q < nnodes; ++q)
        for (int64_t j = 0; j < n; ++j)
            apply_node_reflector(n, j, Y1 + q * nn, tau_node[q * n + j],
                                 C + tile_row0[node_a[q]], C + tile_row0[node_b[q]], ldc, k);
}

void orc_tsqr_apply_q(int64_t m, int64_t n, const double *A, int64_t lda, int64_t c,
                      int64_t ntiles, const int64_t *tile_row0, const int64_t *tile_rows,
                      int64_t nnodes, const int64_t *node_a, const int64_t *node_b,
                      const double *tau_tile, const double *Y1, const double *tau_node,
                      double *C, int64_t ldc, int64_t k)
{
    (void)m;
    size_t nn = (size_t)(n * n);
    for (int64_t q = nnodes - 1; q >= 0; --q)
        for (int64_t j = n - 1; j >= 0; --j)     /* Q_node = H_0 ... H_{n-1}: H_{n-1} first */
            apply_node_reflector(n, j, Y1 + q * nn, tau_node[q * n + j],
                                 C + tile_row0[node_a[q]], C + tile_row0[node_b[q]], ldc, k);
    for (int64_t t = 0, ch0 = 0; t < ntiles; ch0 += chunks_of(tile_rows[t], c), ++t)
        apply_tile(tile_rows[t], n, c, A + tile_row0[t], lda, tau_tile + ch0 * n, C + tile_row0[t], ldc, k, 0);
}

void orc_tsqr_form_q(int64_t m, int64_t n, const double *A, int64_t lda, int64_t c,
                     int64_t ntiles, const int64_t *tile_row0, const int64_t *tile_rows,
                     int64_t nnodes, const int64_t *node_a, const int64_t *node_b,
                     const double *tau_tile, const double *Y1, const double *tau_node,
                     double *Q, int64_t ldq)
{
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) AT(Q, i, j, ldq) = (i == j) ? 1.0 : 0.0;
    orc_tsqr_apply_q(m, n, A, lda, c, ntiles, tile_row0, tile_rows, nnodes, node_a, node_b,
                     tau_tile, Y1, tau_node, Q, ldq, n);
}

/* Modified Gram-Schmidt, every operation in long double. */
void orc_mgs_ld(int64_t m, int64_t n, const double *A, int64_t lda,
                double *Q, int64_t ldq, double *R, int64_t ldr)
{
    long double *V = (long double *)malloc((size_t)(m * n) * sizeof(long double));
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) V[i + j * m] = AT(A, i, j, lda);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) AT(R, i, j, ldr) = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        long double s = 0.0L;
        for (int64_t i = 0; i < m; ++i) s += V[i + j * m] * V[i + j * m];
        long double r = sqrtl(s);
        AT(R, j, j, ldr) = (double)r;
        for (int64_t i = 0; i < m; ++i) V[i + j * m] /= r;
        for (int64_t c = j + 1; c < n; ++c) {
            long double d = 0.0L;
            for (int64_t i = 0; i < m; ++i) d += V[i + j * m] * V[i + c * m];
            AT(R, j, c, ldr) = (double)d;
            for (int64_t i = 0; i < m; ++i) V[i + c * m] -= d * V[i + j * m];
        }
    }
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) AT(Q, i, j, ldq) = (double)V[i + j * m];
    free(V);
}

/* Alg. CholeskyQR ([TR] P:1410-1419), see oracle.h. */
int orc_cholqr(int64_t m, int64_t n, const double *A, int64_t lda, double *R, int64_t ldr,
               double *Q, int64_t ldq)
{
    /* line 1: W := A^T A */
    double *W = (double *)malloc((size_t)(n * n) * sizeof(double));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) {
            long double s = 0.0L;
            for (int64_t r = 0; r < m; ++r) s += (long double)AT(A, r, i, lda) * AT(A, r, j, lda);
            W[i + j * n] = (double)s;
        }
    /* line 2: W = R^T R, R upper triangular, row j from rows 0..j-1 */
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) AT(R, i, j, ldr) = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        long double d = W[j + j * n];
        for (int64_t k = 0; k < j; ++k) d -= (long double)AT(R, k, j, ldr) * AT(R, k, j, ldr);
        if (!(d > 0.0L)) { free(W); return (int)(j + 1); }
        const double rjj = (double)sqrtl(d);
        AT(R, j, j, ldr) = rjj;
        for (int64_t c = j + 1; c < n; ++c) {
            long double s = W[j + c * n];
            for (int64_t k = 0; k < j; ++k) s -= (long double)AT(R, k, j, ldr) * AT(R, k, c, ldr);
            AT(R, j, c, ldr) = (double)(s / rjj);
        }
    }
    free(W);
    /* line 3: Q := A R^{-1}, row by row (R^T q_i = a_i, forward substitution) */
    if (Q) {
        for (int64_t r = 0; r < m; ++r)
            for (int64_t j = 0; j < n; ++j) {
                long double s = AT(A, r, j, lda);
                for (int64_t l = 0; l < j; ++l) s -= (long double)AT(Q, r, l, ldq) * AT(R, l, j, ldr);
                AT(Q, r, j, ldq) = (double)(s / AT(R, j, j, ldr));
            }
    }
    return 0;
}
