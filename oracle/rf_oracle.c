/*
 * rf_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU oracle for the hot path of
 * arXiv 2001.07104 as scoped by SURVEY.md section 8: random-forest regression
 * (bootstrap, per-node random feature subsets, greedy CART variance-reduction
 * splits), prediction, and k-fold cross-validation scored with MAPE.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no source with the
 * CUDA path (paper_2001_07104_b200/csrc): it has its own Philox, its own
 * quantisation, its own tree growth.  Build: plain C11,
 * -O2 -ffp-contract=off (no FMA contraction, no fast-math), no threads.
 *
 * Citation notation: P:n = /root/reference/PAPER.md line n; DESIGN.md Rn =
 * reading n of the ambiguity ledger in DESIGN.md (paper silent/garbled).
 *
 *   - Random forest: trees whose nodes compare one feature with a threshold,
 *     leaves output a value; forest = mean of trees (sec. 2.2).
 *   - max_features = features considered when splitting a node.
 *   - split criterion MSE -> variance reduction, proxy
 *     G = SL^2/WL + SR^2/WR (R6).
 *   - MAPE, Eq. 1, reported in percent.
 *   - log transform of time targets.
 *   - k-fold CV with a fresh random split per iteration;
 *     custom split for time.
 *   - everything the paper leaves open (bootstrap, RNG addressing, exact
 *     sums, tie-break, thresholds, histogram cuts) follows DESIGN.md R1-R28.
 *   - split_mode 2: Extremely Randomized Trees, one uniform random
 *     threshold per drawn feature (R29).
 *
 * Parity status of each exported function is listed in DESIGN.md section 3.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <quadmath.h>

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Random123 constants), R14/R15             */
/* ------------------------------------------------------------------ */
#define OR_M0 0xD2511F53u
#define OR_M1 0xCD9E8D57u
#define OR_W0 0x9E3779B9u
#define OR_W1 0xBB67AE85u

enum { TAG_FOLD = 0xD0, TAG_STRATUM = 0xD1, TAG_KEYDERIV = 0x4B,
       TAG_BOOT = 0xB0, TAG_FEAT = 0xF0, TAG_THR = 0xE7 };

void or_philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t prod0 = (uint64_t)OR_M0 * (uint64_t)c0;
        uint64_t prod1 = (uint64_t)OR_M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(prod0 >> 32), lo0 = (uint32_t)prod0;
        uint32_t hi1 = (uint32_t)(prod1 >> 32), lo1 = (uint32_t)prod1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += OR_W0;
        k1 += OR_W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* draw(i) of stream (key; c1, c2, c3): block b = i/2 is Philox(ctr=(b,c1,c2,c3));
   even i -> (w1<<32)|w0, odd i -> (w3<<32)|w2. */
uint64_t or_draw(uint32_t k0, uint32_t k1, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t i)
{
    uint32_t ctr[4] = { (uint32_t)(i >> 1), c1, c2, c3 };
    uint32_t key[2] = { k0, k1 };
    uint32_t o[4];
    or_philox(ctr, key, o);
    if ((i & 1u) == 0) return ((uint64_t)o[1] << 32) | o[0];
    return ((uint64_t)o[3] << 32) | o[2];
}

/* floor(u * m / 2^64) */
uint64_t or_mulhi64(uint64_t u, uint64_t m)
{
    unsigned __int128 prod = (unsigned __int128)u * (unsigned __int128)m;
    return (uint64_t)(prod >> 64);
}

/* per-tree key k_t = lanes 0,1 of Philox(key=seed, ctr=(t, task, 0, KEYDERIV)) */
static void tree_key(uint64_t seed, uint32_t task, uint32_t t, uint32_t *k0, uint32_t *k1)
{
    uint32_t ctr[4] = { t, task, 0u, TAG_KEYDERIV };
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint32_t o[4];
    or_philox(ctr, key, o);
    *k0 = o[0];
    *k1 = o[1];
}

void or_tree_key(uint64_t seed, uint32_t task, uint32_t t, uint32_t out[2])
{
    tree_key(seed, task, t, &out[0], &out[1]);
}

/* ------------------------------------------------------------------ */
/* Target transform + quantisation (R7, R20)      */
/* ------------------------------------------------------------------ */
/* ln correctly rounded to binary64: evaluate in binary128 and round once. */
double or_ln(double y)
{
    return (double)logq((__float128)y);
}

static int ceil_log2_u64(uint64_t n)
{
    int c = 0;
    while (((uint64_t)1 << c) < n) ++c;
    return c;
}

/* smallest integer e with M <= 2^e, M > 0 */
static int exp_ceil(double M)
{
    int ex;
    double m = frexp(M, &ex); /* M = m * 2^ex, m in [0.5, 1) */
    if (m == 0.5) return ex - 1;
    return ex;
}

/* Returns 0 on success, 3 non-finite, 4 non-positive y with LOG.  guard: extra
   headroom bits (2 under the MAE criterion, R32: doubled medians and absolute-
   deviation costs stay below 2^63). */
static int quantize_g(const double *y, uint64_t n, int target, int guard, double *t_out, int64_t *tq,
                      int32_t *F_out);

int or_quantize(const double *y, uint64_t n, int target, double *t_out, int64_t *tq, int32_t *F_out)
{
    return quantize_g(y, n, target, 0, t_out, tq, F_out);
}

static int quantize_g(const double *y, uint64_t n, int target, int guard, double *t_out, int64_t *tq,
                      int32_t *F_out)
{
    double *t = t_out;
    double M = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        if (!isfinite(y[i])) return 3;
        if (target == 1 && !(y[i] > 0.0)) return 4;
        t[i] = (target == 1) ? or_ln(y[i]) : y[i];
        double a = fabs(t[i]);
        if (a > M) M = a;
    }
    int F = 0;
    if (M > 0.0) F = 62 - ceil_log2_u64(n) - exp_ceil(M) - guard;
    for (uint64_t i = 0; i < n; ++i) {
        double s = ldexp(t[i], F);
        double r = nearbyint(s); /* default rounding mode: half-to-even */
        tq[i] = (int64_t)r;
    }
    *F_out = F;
    return 0;
}

/* ------------------------------------------------------------------ */
/* Folds (R16, R17)                               */
/* ------------------------------------------------------------------ */
typedef struct { uint64_t key; uint64_t idx; } keyidx;

static int cmp_keyidx(const void *a, const void *b)
{
    const keyidx *x = (const keyidx *)a, *y = (const keyidx *)b;
    if (x->key < y->key) return -1;
    if (x->key > y->key) return 1;
    if (x->idx < y->idx) return -1;
    if (x->idx > y->idx) return 1;
    return 0;
}

typedef struct { double y; uint64_t idx; } yidx;

static int cmp_ydesc(const void *a, const void *b)
{
    const yidx *x = (const yidx *)a, *z = (const yidx *)b;
    if (x->y > z->y) return -1;
    if (x->y < z->y) return 1;
    if (x->idx < z->idx) return -1;
    if (x->idx > z->idx) return 1;
    return 0;
}

/* fold_ids[rep*n + i] in {-1, 0..k-1}.  Plain: rows ordered by Philox key
   (ties by index), contiguous blocks of floor(n/k) (+1 for the first n mod k
   folds).  Custom (time targets): the 5 largest y always train
   (-1); remaining rows stratified short (<1e3) / medium (<1e5) / long,
   each stratum ordered by its Philox keys, dealt round-robin over folds,
   the deal counter continuing across strata.
   Returns 0, 6 (too few). */
int or_make_folds(const double *y, uint64_t n, uint32_t k, uint32_t reps, uint64_t seed,
                  uint32_t custom, int32_t *fold_ids)
{
    uint32_t s0 = (uint32_t)seed, s1 = (uint32_t)(seed >> 32);
    if (k < 2) return 6;
    if (!custom && (uint64_t)k > n) return 6;
    if (custom && (n < 5 || n - 5 < (uint64_t)k)) return 6;
    keyidx *ki = (keyidx *)malloc(sizeof(keyidx) * (n ? n : 1));
    for (uint32_t rep = 0; rep < reps; ++rep) {
        int32_t *fid = fold_ids + (uint64_t)rep * n;
        if (!custom) {
            for (uint64_t i = 0; i < n; ++i) {
                ki[i].key = or_draw(s0, s1, rep, 0u, TAG_FOLD, i);
                ki[i].idx = i;
            }
            qsort(ki, n, sizeof(keyidx), cmp_keyidx);
            uint64_t pos = 0;
            for (uint32_t f = 0; f < k; ++f) {
                uint64_t size = n / k + ((uint64_t)f < n % k ? 1 : 0);
                for (uint64_t j = 0; j < size; ++j) fid[ki[pos + j].idx] = (int32_t)f;
                pos += size;
            }
        } else {
            yidx *yi = (yidx *)malloc(sizeof(yidx) * n);
            for (uint64_t i = 0; i < n; ++i) { yi[i].y = y[i]; yi[i].idx = i; }
            qsort(yi, n, sizeof(yidx), cmp_ydesc);
            for (uint64_t i = 0; i < n; ++i) fid[i] = -2; /* unassigned marker */
            for (int j = 0; j < 5; ++j) fid[yi[j].idx] = -1;
            free(yi);
            uint64_t deal = 0;
            for (uint32_t s = 0; s < 3; ++s) {
                uint64_t m = 0;
                for (uint64_t i = 0; i < n; ++i) {
                    if (fid[i] == -1) continue;
                    double v = y[i];
                    uint32_t st = (v < 1000.0) ? 0u : (v < 100000.0 ? 1u : 2u);
                    if (st != s) continue;
                    ki[m].key = or_draw(s0, s1, rep, s, TAG_STRATUM, i);
                    ki[m].idx = i;
                    ++m;
                }
                qsort(ki, m, sizeof(keyidx), cmp_keyidx);
                for (uint64_t j = 0; j < m; ++j) {
                    fid[ki[j].idx] = (int32_t)(deal % k);
                    ++deal;
                }
            }
        }
    }
    free(ki);
    return 0;
}

/* Folds of a row subset (nested CV, R31): for each rep, the rows
   with mask[rep*n + i] != 0 are split exactly like or_make_folds splits a
   dataset of those rows (Philox keys still indexed by the original row i,
   stream (seed; rep, ...)); rows outside the subset get -2 (excluded).
   Returns 0, 6 (a subset too small for k folds). */
int or_make_folds_masked(const double *y, uint64_t n, uint32_t k, uint32_t reps, uint64_t seed,
                         uint32_t custom, const uint8_t *mask, int32_t *fold_ids)
{
    uint32_t s0 = (uint32_t)seed, s1 = (uint32_t)(seed >> 32);
    if (k < 2) return 6;
    keyidx *ki = (keyidx *)malloc(sizeof(keyidx) * (n ? n : 1));
    yidx *yi = (yidx *)malloc(sizeof(yidx) * (n ? n : 1));
    int st = 0;
    for (uint32_t rep = 0; rep < reps && !st; ++rep) {
        int32_t *fid = fold_ids + (uint64_t)rep * n;
        const uint8_t *mk = mask + (uint64_t)rep * n;
        uint64_t na = 0;
        for (uint64_t i = 0; i < n; ++i) {
            fid[i] = -2;
            if (mk[i]) ++na;
        }
        if ((!custom && (uint64_t)k > na) || (custom && (na < 5 || na - 5 < (uint64_t)k))) { st = 6; break; }
        if (!custom) {
            uint64_t m = 0;
            for (uint64_t i = 0; i < n; ++i) {
                if (!mk[i]) continue;
                ki[m].key = or_draw(s0, s1, rep, 0u, TAG_FOLD, i);
                ki[m].idx = i;
                ++m;
            }
            qsort(ki, m, sizeof(keyidx), cmp_keyidx);
            uint64_t pos = 0;
            for (uint32_t f = 0; f < k; ++f) {
                uint64_t size = na / k + ((uint64_t)f < na % k ? 1 : 0);
                for (uint64_t j = 0; j < size; ++j) fid[ki[pos + j].idx] = (int32_t)f;
                pos += size;
            }
        } else {
            uint64_t m = 0;
            for (uint64_t i = 0; i < n; ++i)
                if (mk[i]) { yi[m].y = y[i]; yi[m].idx = i; ++m; }
            qsort(yi, m, sizeof(yidx), cmp_ydesc);
            int32_t *pin = (int32_t *)calloc(n ? n : 1, sizeof(int32_t));
            for (int j = 0; j < 5; ++j) pin[yi[j].idx] = 1;
            uint64_t deal = 0;
            for (uint32_t s = 0; s < 3; ++s) {
                uint64_t q = 0;
                for (uint64_t i = 0; i < n; ++i) {
                    if (!mk[i] || pin[i]) continue;
                    double v = y[i];
                    uint32_t sv = (v < 1000.0) ? 0u : (v < 100000.0 ? 1u : 2u);
                    if (sv != s) continue;
                    ki[q].key = or_draw(s0, s1, rep, s, TAG_STRATUM, i);
                    ki[q].idx = i;
                    ++q;
                }
                qsort(ki, q, sizeof(keyidx), cmp_keyidx);
                for (uint64_t j = 0; j < q; ++j) {
                    fid[ki[j].idx] = (int32_t)(deal % k);
                    ++deal;
                }
            }
            for (uint64_t i = 0; i < n; ++i) if (pin[i]) fid[i] = -1;
            free(pin);
        }
    }
    free(ki);
    free(yi);
    return st;
}

/* ------------------------------------------------------------------ */
/* Dense ranks and histogram cuts (R10, R23)                 */
/* ------------------------------------------------------------------ */
static int cmp_double(const void *a, const void *b)
{
    double x = *(const double *)a, y = *(const double *)b;
    return (x < y) ? -1 : (x > y ? 1 : 0);
}

/* distinct sorted values of column f over the given rows */
static double *distinct_values(const double *X, uint32_t p, uint32_t f, const uint64_t *rows,
                               uint64_t m, uint64_t *nd)
{
    double *v = (double *)malloc(sizeof(double) * (m ? m : 1));
    for (uint64_t i = 0; i < m; ++i) v[i] = X[rows[i] * p + f];
    qsort(v, m, sizeof(double), cmp_double);
    uint64_t d = 0;
    for (uint64_t i = 0; i < m; ++i)
        if (d == 0 || v[i] != v[d - 1]) v[d++] = v[i];
    *nd = d;
    return v;
}

/* index of x in sorted distinct array u (x must be present) */
static uint64_t find_index(const double *u, uint64_t nd, double x)
{
    uint64_t lo = 0, hi = nd;
    while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        if (u[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* histogram cuts per DESIGN.md R23 from the (task) training rows, unweighted */
static double *hist_cuts(const double *X, uint32_t p, uint32_t f, const uint64_t *rows, uint64_t m,
                         uint32_t *ncuts)
{
    double *s = (double *)malloc(sizeof(double) * (m ? m : 1));
    for (uint64_t i = 0; i < m; ++i) s[i] = X[rows[i] * p + f];
    qsort(s, m, sizeof(double), cmp_double);
    uint64_t D = 0;
    double umax = m ? s[m - 1] : 0.0;
    for (uint64_t i = 0; i < m; ++i)
        if (i == 0 || s[i] != s[i - 1]) ++D;
    double *cuts = (double *)malloc(sizeof(double) * 256);
    uint32_t c = 0;
    if (D <= 256) {
        for (uint64_t i = 0; i < m; ++i) {
            if (i == 0 || s[i] != s[i - 1]) {
                if (s[i] != umax) cuts[c++] = s[i];
            }
        }
    } else {
        for (uint64_t j = 1; j <= 255; ++j) {
            uint64_t q = (j * m + 255) / 256; /* ceil(j*m/256) */
            double v = s[q - 1];
            if (v == umax) continue;
            if (c > 0 && cuts[c - 1] == v) continue;
            cuts[c++] = v;
        }
    }
    free(s);
    *ncuts = c;
    return cuts;
}

/* ------------------------------------------------------------------ */
/* Tree growth (R2-R14)                                      */
/* ------------------------------------------------------------------ */
typedef struct {
    int32_t feature;     /* -1 leaf */
    uint32_t thr_index;
    double thr_value;
    uint32_t left;       /* BFS id of left child; right = left + 1 */
    double leaf_value;
} or_node;

typedef struct {
    uint64_t *rows;  /* distinct in-bag rows, ascending */
    uint64_t nrows;
    int64_t W, S;
    uint32_t depth;
    uint64_t heap;
} work_node;

typedef struct {
    or_node *nodes;
    uint64_t n, cap;
} or_tree;

static void tree_push(or_tree *t, or_node nd)
{
    if (t->n == t->cap) {
        t->cap = t->cap ? 2 * t->cap : 64;
        t->nodes = (or_node *)realloc(t->nodes, sizeof(or_node) * t->cap);
    }
    t->nodes[t->n++] = nd;
}

typedef struct { double x; uint64_t row; } xrow;

static int cmp_xrow(const void *a, const void *b)
{
    const xrow *u = (const xrow *)a, *v = (const xrow *)b;
    if (u->x < v->x) return -1;
    if (u->x > v->x) return 1;
    if (u->row < v->row) return -1;
    if (u->row > v->row) return 1;
    return 0;
}

typedef struct {
    const double *X;
    uint64_t n;
    uint32_t p;
    const int64_t *tq;
    int32_t F;
    /* exact mode: global distinct values per feature (for threshold index) */
    double **gdist;
    uint64_t *gnd;
    /* hist mode: cuts per feature for this task, bins per row (n x p) */
    int hist;
    /* ExtraTrees mode (split_mode 2): one random threshold per drawn feature (R29) */
    int extra;
    /* MAE criterion (R32): splits minimise the summed absolute deviations from the
       children's weighted medians; leaves hold the weighted median */
    int mae;
    /* tie-break among bitwise-equal scores (R9): 0 = lowest feature index, then lowest
       threshold (BASELINE.json north_star, the default); 1 = the feature drawn first at
       the node (lowest draw slot), then lowest threshold (scikit-learn's visiting order) */
    int tie_draw;
    double **cuts;
    uint32_t *ncuts;
    uint16_t *bins; /* [row*p + f] */
    uint32_t mtry, min_split;
    int32_t max_depth;
} grow_ctx;

/* G = fl(fl(fl(SL*SL)/WL) + fl(fl(SR*SR)/WR))  (R6, R28) */
static double gain(int64_t WL, int64_t SL, int64_t WR, int64_t SR)
{
    double dSL = (double)SL, dWL = (double)WL, dSR = (double)SR, dWR = (double)WR;
    double a = dSL * dSL;
    a = a / dWL;
    double b = dSR * dSR;
    b = b / dWR;
    return a + b;
}

/* ---- MAE criterion (T4/T5 P:858-861; R32) ---- */
typedef struct { int64_t t; uint64_t row; } trow;

static int cmp_trow(const void *a, const void *b)
{
    const trow *u = (const trow *)a, *v = (const trow *)b;
    if (u->t < v->t) return -1;
    if (u->t > v->t) return 1;
    if (u->row < v->row) return -1;
    if (u->row > v->row) return 1;
    return 0;
}

/* 2 x the weighted median of t_q over rows (scikit-learn's rule): values in
   ascending order, k = the first with 2 cum_k >= W; if 2 cum_k == W the median
   is (t_k + t_k+1) / 2, else t_k.  Doubling keeps it an exact integer. */
static int64_t median2(const uint64_t *rows, uint64_t m, const uint32_t *w, const int64_t *tq, trow *buf)
{
    int64_t W = 0;
    for (uint64_t i = 0; i < m; ++i) {
        buf[i].t = tq[rows[i]];
        buf[i].row = rows[i];
        W += (int64_t)w[rows[i]];
    }
    qsort(buf, m, sizeof(trow), cmp_trow);
    int64_t cum = 0;
    for (uint64_t i = 0; i < m; ++i) {
        cum += (int64_t)w[buf[i].row];
        if (2 * cum >= W) {
            if (2 * cum == W && i + 1 < m) return buf[i].t + buf[i + 1].t;
            return 2 * buf[i].t;
        }
    }
    return 0;
}

/* 2 x the sum of weighted absolute deviations from the median: sum w |2 t - m2| (exact) */
static unsigned __int128 sad2(const uint64_t *rows, uint64_t m, const uint32_t *w, const int64_t *tq,
                              int64_t m2)
{
    unsigned __int128 s = 0;
    for (uint64_t i = 0; i < m; ++i) {
        __int128 d = (__int128)2 * tq[rows[i]] - m2;
        if (d < 0) d = -d;
        s += (unsigned __int128)w[rows[i]] * (unsigned __int128)d;
    }
    return s;
}

static unsigned __int128 mae_cost(const uint64_t *rows, uint64_t m, const uint32_t *w, const int64_t *tq,
                                  trow *buf)
{
    return sad2(rows, m, w, tq, median2(rows, m, w, tq, buf));
}

/* Mean-decrease-in-impurity of one split (feature importance, SURVEY 8(f)
   NEXT-3; Table 6): W imp(node) - WL imp(L) - WR imp(R)
   with imp = weighted MSE; the sum-of-squares terms cancel, leaving
   SL^2/WL + SR^2/WR - S^2/W = (SL WR - SR WL)^2 / (W WL WR), in target units
   (x 2^-2F).  Evaluated exactly in __int128, then once in binary128. */
static double mdi_decrease(int64_t WL, int64_t SL, int64_t WR, int64_t SR, int32_t F)
{
    __int128 num = (__int128)SL * WR - (__int128)SR * WL;
    __float128 q = (__float128)num;
    q = q * q / ((__float128)(WL + WR) * (__float128)WL * (__float128)WR);
    return (double)ldexpq(q, -2 * F);
}

/* grows one tree; w[] = multiplicities per row (0 = out of bag);
   imp (or NULL): per-feature sums of split decreases, BFS order */
static void grow_tree(const grow_ctx *c, const uint32_t *w, uint32_t k0, uint32_t k1,
                      or_tree *out, int32_t *leaf_of_row, double *imp)
{
    const uint32_t p = c->p;
    /* root */
    uint64_t nr = 0;
    for (uint64_t i = 0; i < c->n; ++i) if (w[i] > 0) ++nr;
    work_node *q = (work_node *)malloc(sizeof(work_node) * 16);
    uint64_t qcap = 16, qn = 0;
    {
        work_node r;
        r.rows = (uint64_t *)malloc(sizeof(uint64_t) * (nr ? nr : 1));
        r.nrows = 0; r.W = 0; r.S = 0;
        for (uint64_t i = 0; i < c->n; ++i) if (w[i] > 0) {
            r.rows[r.nrows++] = i;
            r.W += (int64_t)w[i];
            r.S += (int64_t)w[i] * c->tq[i];
        }
        r.depth = 0; r.heap = 1;
        q[qn++] = r;
    }
    out->n = 0;
    uint32_t *perm = (uint32_t *)malloc(sizeof(uint32_t) * p);
    xrow *xr = (xrow *)malloc(sizeof(xrow) * (nr ? nr : 1));
    uint64_t *lr = (uint64_t *)malloc(sizeof(uint64_t) * (nr ? nr : 1)); /* MAE: child row sets */
    uint64_t *rr = (uint64_t *)malloc(sizeof(uint64_t) * (nr ? nr : 1));
    trow *tb = (trow *)malloc(sizeof(trow) * (nr ? nr : 1));
    unsigned __int128 bestD = 0;
    int64_t *hW = (int64_t *)malloc(sizeof(int64_t) * 257);
    int64_t *hS = (int64_t *)malloc(sizeof(int64_t) * 257);

    for (uint64_t qi = 0; qi < qn; ++qi) {
        work_node nd = q[qi];
        or_node rec;
        memset(&rec, 0, sizeof rec);
        rec.feature = -1;
        int is_leaf = 0;
        if (c->max_depth >= 0 && nd.depth >= (uint32_t)c->max_depth) is_leaf = 1;
        if (nd.nrows < c->min_split) is_leaf = 1;
        if (!is_leaf) {
            int64_t mn = c->tq[nd.rows[0]], mx = mn;
            for (uint64_t i = 1; i < nd.nrows; ++i) {
                int64_t v = c->tq[nd.rows[i]];
                if (v < mn) mn = v;
                if (v > mx) mx = v;
            }
            if (mn == mx) is_leaf = 1;
        }
        int found = 0;
        double bestG = 0.0;
        uint32_t bestF = 0;
        /* tie-break (R9): among bitwise-equal G the lowest tie key, then the lowest
           threshold rank; tie key = the feature index (north_star: "lowest feature then
           lowest threshold", default) or, with tie_draw, the draw slot (scikit-learn's
           splitter visits features in the random draw order and keeps the first best). */
        uint32_t bestTie = 0;
        uint64_t bestRank = 0; /* exact: rank_f(a) ; hist: cut index j */
        double bestA = 0.0, bestB = 0.0;
        if (!is_leaf) {
            /* draw m features: partial Fisher-Yates keyed by heap index (R4, R14) */
            for (uint32_t f = 0; f < p; ++f) perm[f] = f;
            uint32_t hlo = (uint32_t)nd.heap, hhi = (uint32_t)(nd.heap >> 32);
            for (uint32_t j = 0; j < c->mtry; ++j) {
                uint64_t u = or_draw(k0, k1, hlo, hhi, TAG_FEAT, j);
                uint32_t r = j + (uint32_t)or_mulhi64(u, (uint64_t)(p - j));
                uint32_t tmp = perm[j]; perm[j] = perm[r]; perm[r] = tmp;
            }
            for (uint32_t jj = 0; jj < c->mtry && c->mae; ++jj) {
                /* MAE criterion (R32): candidates as in R8 (exact) or R29 (ExtraTrees);
                   cost D = 2 (SAD_L + SAD_R), exact integers; best = lowest D, ties by
                   draw slot, then threshold rank (R9) */
                uint32_t f = perm[jj];
                uint32_t tk = c->tie_draw ? jj : f;
                for (uint64_t i = 0; i < nd.nrows; ++i) {
                    xr[i].row = nd.rows[i];
                    xr[i].x = c->X[nd.rows[i] * p + f];
                }
                qsort(xr, nd.nrows, sizeof(xrow), cmp_xrow);
                uint64_t i0 = 0, i1 = nd.nrows - 1; /* candidate boundaries i in [i0, i1) */
                double ethr = 0.0;
                if (c->extra) {
                    double lo = xr[0].x, hi = xr[nd.nrows - 1].x;
                    if (lo == hi) continue;
                    uint64_t ud = or_draw(k0, k1, hlo, hhi, TAG_THR, jj);
                    double u = (double)(ud >> 11) * 0x1p-53;
                    double span = hi - lo;
                    ethr = span * u;
                    ethr = ethr + lo;
                    if (!(ethr < hi)) ethr = lo;
                    uint64_t b = 0;
                    while (b + 1 < nd.nrows && xr[b + 1].x <= ethr) ++b;
                    i0 = b; i1 = b + 1;
                }
                for (uint64_t i = i0; i < i1; ++i) {
                    if (!(xr[i].x < xr[i + 1].x)) continue;
                    for (uint64_t a = 0; a <= i; ++a) lr[a] = xr[a].row;
                    for (uint64_t a = i + 1; a < nd.nrows; ++a) rr[a - i - 1] = xr[a].row;
                    unsigned __int128 D = mae_cost(lr, i + 1, w, c->tq, tb) +
                                          mae_cost(rr, nd.nrows - i - 1, w, c->tq, tb);
                    uint64_t rk = find_index(c->gdist[f], c->gnd[f], xr[i].x);
                    int better = 0;
                    if (!found) better = 1;
                    else if (D < bestD) better = 1;
                    else if (D == bestD) {
                        if (tk < bestTie) better = 1;
                        else if (tk == bestTie && rk < bestRank) better = 1;
                    }
                    if (better) {
                        found = 1; bestD = D; bestF = f; bestTie = tk; bestRank = rk;
                        bestA = c->extra ? ethr : xr[i].x;
                        bestB = c->extra ? 0.0 : xr[i + 1].x;
                    }
                }
            }
            for (uint32_t jj = 0; jj < c->mtry && !c->mae; ++jj) {
                uint32_t f = perm[jj];
                uint32_t tk = c->tie_draw ? jj : f;
                if (c->extra) {
                    /* Extremely Randomized Trees (R29):
                       thr uniform in [lo, hi) of the node's values of f,
                       thr = fl(fl(fl(hi - lo) * u) + lo), u = (draw >> 11) 2^-53,
                       replaced by lo if it does not fall below hi. */
                    double lo = c->X[nd.rows[0] * p + f], hi = lo;
                    for (uint64_t i = 1; i < nd.nrows; ++i) {
                        double x = c->X[nd.rows[i] * p + f];
                        if (x < lo) lo = x;
                        if (x > hi) hi = x;
                    }
                    if (lo == hi) continue; /* constant feature in this node */
                    uint64_t ud = or_draw(k0, k1, hlo, hhi, TAG_THR, jj);
                    double u = (double)(ud >> 11) * 0x1p-53;
                    double span = hi - lo;
                    double thr = span * u;
                    thr = thr + lo;
                    if (!(thr < hi)) thr = lo;
                    int64_t WL = 0, SL = 0;
                    double a = lo; /* largest node value <= thr */
                    for (uint64_t i = 0; i < nd.nrows; ++i) {
                        uint64_t r = nd.rows[i];
                        double x = c->X[r * p + f];
                        if (x <= thr) {
                            WL += (int64_t)w[r];
                            SL += (int64_t)w[r] * c->tq[r];
                            if (x > a) a = x;
                        }
                    }
                    double G = gain(WL, SL, nd.W - WL, nd.S - SL);
                    int better = 0;
                    if (!found) better = 1;
                    else if (G > bestG) better = 1;
                    else if (G == bestG && tk < bestTie) better = 1;
                    if (better) {
                        found = 1; bestG = G; bestF = f; bestTie = tk;
                        bestRank = find_index(c->gdist[f], c->gnd[f], a);
                        bestA = thr; bestB = 0.0;
                    }
                } else if (!c->hist) {
                    for (uint64_t i = 0; i < nd.nrows; ++i) {
                        xr[i].row = nd.rows[i];
                        xr[i].x = c->X[nd.rows[i] * p + f];
                    }
                    qsort(xr, nd.nrows, sizeof(xrow), cmp_xrow);
                    int64_t WL = 0, SL = 0;
                    for (uint64_t i = 0; i + 1 < nd.nrows; ++i) {
                        uint64_t r = xr[i].row;
                        WL += (int64_t)w[r];
                        SL += (int64_t)w[r] * c->tq[r];
                        if (!(xr[i].x < xr[i + 1].x)) continue;
                        double G = gain(WL, SL, nd.W - WL, nd.S - SL);
                        uint64_t rk = find_index(c->gdist[f], c->gnd[f], xr[i].x);
                        int better = 0;
                        if (!found) better = 1;
                        else if (G > bestG) better = 1;
                        else if (G == bestG) {
                            if (tk < bestTie) better = 1;
                            else if (tk == bestTie && rk < bestRank) better = 1;
                        }
                        if (better) {
                            found = 1; bestG = G; bestF = f; bestTie = tk; bestRank = rk;
                            bestA = xr[i].x; bestB = xr[i + 1].x;
                        }
                    }
                } else {
                    uint32_t nc = c->ncuts[f];
                    for (uint32_t b = 0; b <= nc; ++b) { hW[b] = 0; hS[b] = 0; }
                    for (uint64_t i = 0; i < nd.nrows; ++i) {
                        uint64_t r = nd.rows[i];
                        uint32_t b = c->bins[r * p + f];
                        hW[b] += (int64_t)w[r];
                        hS[b] += (int64_t)w[r] * c->tq[r];
                    }
                    int64_t WL = 0, SL = 0;
                    for (uint32_t j = 0; j < nc; ++j) {
                        WL += hW[j];
                        SL += hS[j];
                        int64_t WR = nd.W - WL;
                        if (WL <= 0 || WR <= 0) continue;
                        double G = gain(WL, SL, WR, nd.S - SL);
                        int better = 0;
                        if (!found) better = 1;
                        else if (G > bestG) better = 1;
                        else if (G == bestG) {
                            if (tk < bestTie) better = 1;
                            else if (tk == bestTie && j < bestRank) better = 1;
                        }
                        if (better) {
                            found = 1; bestG = G; bestF = f; bestTie = tk; bestRank = j;
                            bestA = c->cuts[f][j]; bestB = 0.0;
                        }
                    }
                }
            }
            if (!found) is_leaf = 1;
        }
        if (is_leaf) {
            rec.feature = -1;
            if (c->mae) /* weighted median (R32) */
                rec.leaf_value = ldexp((double)median2(nd.rows, nd.nrows, w, c->tq, tb), -c->F - 1);
            else
                rec.leaf_value = ldexp((double)nd.S / (double)nd.W, -c->F);
            if (leaf_of_row)
                for (uint64_t i = 0; i < nd.nrows; ++i) leaf_of_row[nd.rows[i]] = (int32_t)out->n;
            tree_push(out, rec);
            free(nd.rows);
            continue;
        }
        double thr;
        if (c->extra) {
            thr = bestA; /* the drawn threshold (R29) */
        } else if (!c->hist) {
            thr = bestA / 2.0 + bestB / 2.0; /* R8 */
            if (thr == bestB) thr = bestA;
        } else {
            thr = bestA; /* cut value c_j (R23) */
        }
        rec.feature = (int32_t)bestF;
        rec.thr_index = (uint32_t)bestRank;
        rec.thr_value = thr;
        /* children: BFS ids assigned in queue order */
        rec.left = (uint32_t)(qn);
        work_node L, R;
        L.rows = (uint64_t *)malloc(sizeof(uint64_t) * nd.nrows);
        R.rows = (uint64_t *)malloc(sizeof(uint64_t) * nd.nrows);
        L.nrows = R.nrows = 0; L.W = L.S = R.W = R.S = 0;
        for (uint64_t i = 0; i < nd.nrows; ++i) {
            uint64_t r = nd.rows[i];
            double x = c->X[r * p + bestF];
            if (x <= thr) {
                L.rows[L.nrows++] = r; L.W += (int64_t)w[r]; L.S += (int64_t)w[r] * c->tq[r];
            } else {
                R.rows[R.nrows++] = r; R.W += (int64_t)w[r]; R.S += (int64_t)w[r] * c->tq[r];
            }
        }
        if (imp && c->mae) /* (SAD_node - SAD_L - SAD_R) in target units (R30, R32) */
            imp[bestF] += ldexp((double)(mae_cost(nd.rows, nd.nrows, w, c->tq, tb) - bestD), -c->F - 1);
        else if (imp) imp[bestF] += mdi_decrease(L.W, L.S, R.W, R.S, c->F);
        L.depth = R.depth = nd.depth + 1;
        L.heap = 2 * nd.heap;       /* uint64 wrap-around (R14) */
        R.heap = 2 * nd.heap + 1;
        if (qn + 2 > qcap) {
            qcap *= 2;
            q = (work_node *)realloc(q, sizeof(work_node) * qcap);
        }
        q[qn++] = L;
        q[qn++] = R;
        tree_push(out, rec);
        free(nd.rows);
    }
    free(q); free(perm); free(xr); free(hW); free(hS); free(lr); free(rr); free(tb);
}

/* ------------------------------------------------------------------ */
/* Task setup shared by fit and CV                                    */
/* ------------------------------------------------------------------ */
typedef struct {
    grow_ctx g;
    double *t;
    int64_t *tq;
} data_ctx;

static int validate_X(const double *X, uint64_t n, uint32_t p, double *Xc)
{
    for (uint64_t i = 0; i < n * p; ++i) {
        if (!isfinite(X[i])) return 3;
        Xc[i] = (X[i] == 0.0) ? 0.0 : X[i]; /* -0.0 -> +0.0 (R22) */
    }
    return 0;
}

static void setup_exact(grow_ctx *g, const double *X, uint64_t n, uint32_t p)
{
    uint64_t *all = (uint64_t *)malloc(sizeof(uint64_t) * n);
    for (uint64_t i = 0; i < n; ++i) all[i] = i;
    g->gdist = (double **)malloc(sizeof(double *) * p);
    g->gnd = (uint64_t *)malloc(sizeof(uint64_t) * p);
    for (uint32_t f = 0; f < p; ++f) g->gdist[f] = distinct_values(X, p, f, all, n, &g->gnd[f]);
    free(all);
}

static void free_exact(grow_ctx *g, uint32_t p)
{
    for (uint32_t f = 0; f < p; ++f) free(g->gdist[f]);
    free(g->gdist); free(g->gnd);
}

static void setup_hist(grow_ctx *g, const double *X, uint64_t n, uint32_t p, const uint64_t *tr, uint64_t ntr)
{
    g->cuts = (double **)malloc(sizeof(double *) * p);
    g->ncuts = (uint32_t *)malloc(sizeof(uint32_t) * p);
    g->bins = (uint16_t *)malloc(sizeof(uint16_t) * n * p);
    for (uint32_t f = 0; f < p; ++f) {
        g->cuts[f] = hist_cuts(X, p, f, tr, ntr, &g->ncuts[f]);
        for (uint64_t i = 0; i < n; ++i) {
            double x = X[i * p + f];
            uint32_t b = 0;
            while (b < g->ncuts[f] && g->cuts[f][b] < x) ++b; /* bin(x) = #{c < x} */
            g->bins[i * p + f] = (uint16_t)b;
        }
    }
}

static void free_hist(grow_ctx *g, uint32_t p)
{
    for (uint32_t f = 0; f < p; ++f) free(g->cuts[f]);
    free(g->cuts); free(g->ncuts); free(g->bins);
}

/* bootstrap multiplicities over training rows tr[0..ntr) (R2) */
static void bootstrap(uint32_t k0, uint32_t k1, const uint64_t *tr, uint64_t ntr, uint64_t n,
                      int boot, uint32_t *w)
{
    for (uint64_t i = 0; i < n; ++i) w[i] = 0;
    if (!boot) {
        for (uint64_t j = 0; j < ntr; ++j) w[tr[j]] = 1;
        return;
    }
    for (uint64_t j = 0; j < ntr; ++j) {
        uint64_t u = or_draw(k0, k1, 0u, 0u, TAG_BOOT, j);
        w[tr[or_mulhi64(u, ntr)]] += 1;
    }
}

static double tree_predict(const or_tree *t, const double *x)
{
    uint64_t i = 0;
    while (t->nodes[i].feature >= 0) {
        const or_node *nd = &t->nodes[i];
        i = (x[nd->feature] <= nd->thr_value) ? nd->left : nd->left + 1;
    }
    return t->nodes[i].leaf_value;
}

/* ------------------------------------------------------------------ */
/* Public oracle entry points                                          */
/* ------------------------------------------------------------------ */

/* split_mode word of or_fit / or_cv_grid: bits 0-7 the split rule (0 exact, 1 hist,
   2 ExtraTrees), bit 8 the MAE criterion (R32; exact and ExtraTrees only), bit 9 the
   draw-order tie-break (R9; clear = lowest feature index, north_star) */
static int split_mode_ok(uint32_t split_mode)
{
    uint32_t rule = split_mode & 0xFFu, mae = (split_mode >> 8) & 1u;
    if (rule > 2 || (split_mode >> 10) != 0) return 0;
    if (rule == 1 && mae) return 0;
    return 1;
}

/* Fit trees [tree_begin, tree_end) of task 0 (all rows train).
   Outputs per tree (index t - tree_begin) with capacity cap nodes:
   n_nodes[T], feature/thr_index/thr_value/left/leaf_value [T][cap],
   leaf_of_row [T][n] (or NULL; -1 = out of bag), imp_raw [T][p] (or NULL):
   per tree and feature the sum of the MDI decreases of its splits (target
   units, see mdi_decrease). Returns status. */
int or_fit(const double *X, uint64_t n, uint32_t p, const double *y,
           uint32_t mtry, uint32_t min_split, int32_t max_depth, uint32_t boot,
           uint32_t split_mode, uint32_t target, uint64_t seed,
           uint32_t tree_begin, uint32_t tree_end, uint64_t cap,
           uint64_t *n_nodes, int32_t *feature, uint32_t *thr_index, double *thr_value,
           uint32_t *left, double *leaf_value, int32_t *leaf_of_row, int32_t *F_out,
           double *imp_raw)
{
    if (n == 0) return 2;
    if (p == 0 || mtry == 0 || mtry > p || min_split < 2 || !split_mode_ok(split_mode)) return 1;
    double *Xc = (double *)malloc(sizeof(double) * n * p);
    int st = validate_X(X, n, p, Xc);
    if (st) { free(Xc); return st; }
    double *t = (double *)malloc(sizeof(double) * n);
    int64_t *tq = (int64_t *)malloc(sizeof(int64_t) * n);
    int32_t F;
    st = quantize_g(y, n, (int)target, ((split_mode >> 8) & 1u) ? 2 : 0, t, tq, &F);
    if (st) { free(Xc); free(t); free(tq); return st; }
    if (F_out) *F_out = F;
    uint64_t *tr = (uint64_t *)malloc(sizeof(uint64_t) * n);
    for (uint64_t i = 0; i < n; ++i) tr[i] = i;
    grow_ctx g;
    memset(&g, 0, sizeof g);
    g.X = Xc; g.n = n; g.p = p; g.tq = tq; g.F = F;
    g.mtry = mtry; g.min_split = min_split; g.max_depth = max_depth;
    g.hist = ((split_mode & 0xFFu) == 1);
    g.extra = ((split_mode & 0xFFu) == 2);
    g.mae = (int)((split_mode >> 8) & 1u);
    g.tie_draw = (int)((split_mode >> 9) & 1u);
    if (g.hist) setup_hist(&g, Xc, n, p, tr, n); else setup_exact(&g, Xc, n, p);
    uint32_t *w = (uint32_t *)malloc(sizeof(uint32_t) * n);
    or_tree tree = { NULL, 0, 0 };
    for (uint32_t tt = tree_begin; tt < tree_end; ++tt) {
        uint32_t k0, k1;
        tree_key(seed, 0u, tt, &k0, &k1);
        bootstrap(k0, k1, tr, n, n, (int)boot, w);
        uint64_t o = tt - tree_begin;
        int32_t *lor = leaf_of_row ? leaf_of_row + o * n : NULL;
        if (lor) for (uint64_t i = 0; i < n; ++i) lor[i] = -1;
        double *imp = imp_raw ? imp_raw + o * p : NULL;
        if (imp) for (uint32_t f = 0; f < p; ++f) imp[f] = 0.0;
        grow_tree(&g, w, k0, k1, &tree, lor, imp);
        n_nodes[o] = tree.n;
        if (tree.n > cap) { st = 9; break; }
        for (uint64_t i = 0; i < tree.n; ++i) {
            feature[o * cap + i] = tree.nodes[i].feature;
            thr_index[o * cap + i] = tree.nodes[i].thr_index;
            thr_value[o * cap + i] = tree.nodes[i].thr_value;
            left[o * cap + i] = tree.nodes[i].left;
            leaf_value[o * cap + i] = tree.nodes[i].leaf_value;
        }
    }
    free(tree.nodes);
    if (g.hist) free_hist(&g, p); else free_exact(&g, p);
    free(w); free(tr); free(Xc); free(t); free(tq);
    return st;
}

/* Predict with a flattened forest: node arrays concatenated, tree_off[T+1].
   yhat[i] = (sum_t leaf_t(x_i)) / T summed in tree order; exp if LOG. */
int or_predict(const int32_t *feature, const double *thr_value, const uint32_t *left,
               const double *leaf_value, const uint64_t *tree_off, uint32_t T, uint32_t target,
               const double *Xq, uint64_t nq, uint32_t p, double *yhat)
{
    for (uint64_t r = 0; r < nq; ++r) {
        const double *x = Xq + r * p;
        double s = 0.0;
        for (uint32_t t = 0; t < T; ++t) {
            uint64_t base = tree_off[t], i = 0;
            while (feature[base + i] >= 0) {
                uint64_t j = base + i;
                i = (x[feature[j]] <= thr_value[j]) ? left[j] : left[j] + 1;
            }
            s += leaf_value[base + i];
        }
        s = s / (double)T;
        yhat[r] = (target == 1) ? exp(s) : s;
    }
    return 0;
}

/* MAPE in percent over the rows of one fold, ascending (Eq. 1) */
double or_mape(const double *y, const double *yhat, uint64_t m)
{
    double s = 0.0;
    for (uint64_t i = 0; i < m; ++i) s += fabs(y[i] - yhat[i]) / y[i];
    return 100.0 * s / (double)m;
}

/* Grid cross-validation (R16-R19).
   fold_ids: [reps][n] or NULL (plain folds from seed); -1 = always train,
   -2 = excluded from the task (neither trains nor tests; nested CV, R31).
   ntrees evaluated as prefixes of max(ntrees).  Outputs:
   fold_mape [n_mtry][n_ntree][reps][k];  pred (optional) [n_mtry][n_ntree][reps][n]
   = prediction of each row by the forest of its test fold (raw units; rows with
   fold -1 get NaN).  task range [task_begin, task_end) (0,0 = all): entries of
   other tasks are NaN.  Returns status. */
int or_cv_grid(const double *X, uint64_t n, uint32_t p, const double *y,
               uint32_t min_split, int32_t max_depth, uint32_t boot, uint32_t split_mode,
               uint32_t target, uint64_t seed, uint32_t k, uint32_t reps, const int32_t *fold_ids_in,
               const uint32_t *ntrees, uint32_t n_ntree, const uint32_t *mtrys, uint32_t n_mtry,
               uint32_t task_begin, uint32_t task_end,
               double *fold_mape, double *pred)
{
    if (n == 0) return 2;
    if (k < 2 || (uint64_t)k > n) return 6;
    if (p == 0 || min_split < 2 || n_ntree == 0 || n_mtry == 0 || (split_mode & 0xFFu) > 2 ||
        !split_mode_ok(split_mode)) return 1;
    for (uint32_t i = 0; i < n_mtry; ++i) if (mtrys[i] == 0 || mtrys[i] > p) return 1;
    for (uint32_t i = 0; i < n_ntree; ++i) if (ntrees[i] == 0) return 1;
    for (uint64_t i = 0; i < n; ++i) {
        if (!isfinite(y[i])) return 3;
        if (!(y[i] > 0.0)) return 4;
    }
    double *Xc = (double *)malloc(sizeof(double) * n * p);
    int st = validate_X(X, n, p, Xc);
    if (st) { free(Xc); return st; }
    double *t = (double *)malloc(sizeof(double) * n);
    int64_t *tq = (int64_t *)malloc(sizeof(int64_t) * n);
    int32_t F;
    st = quantize_g(y, n, (int)target, ((split_mode >> 8) & 1u) ? 2 : 0, t, tq, &F);
    if (st) { free(Xc); free(t); free(tq); return st; }
    int32_t *fid = (int32_t *)malloc(sizeof(int32_t) * n * reps);
    if (fold_ids_in) memcpy(fid, fold_ids_in, sizeof(int32_t) * n * reps);
    else {
        st = or_make_folds(y, n, k, reps, seed, 0u, fid);
        if (st) { free(Xc); free(t); free(tq); free(fid); return st; }
    }
    /* every fold must have a test row */
    for (uint32_t rep = 0; rep < reps; ++rep)
        for (uint32_t f = 0; f < k; ++f) {
            uint64_t c = 0;
            for (uint64_t i = 0; i < n; ++i) if (fid[(uint64_t)rep * n + i] == (int32_t)f) ++c;
            if (c == 0) { free(Xc); free(t); free(tq); free(fid); return 6; }
        }
    uint32_t Tmax = 0;
    for (uint32_t i = 0; i < n_ntree; ++i) if (ntrees[i] > Tmax) Tmax = ntrees[i];
    uint32_t ntask = reps * k;
    if (task_begin == 0 && task_end == 0) task_end = ntask;
    uint64_t nm = (uint64_t)n_mtry * n_ntree * reps * k;
    for (uint64_t i = 0; i < nm; ++i) fold_mape[i] = NAN;
    if (pred) for (uint64_t i = 0; i < (uint64_t)n_mtry * n_ntree * reps * n; ++i) pred[i] = NAN;

    grow_ctx g;
    memset(&g, 0, sizeof g);
    g.X = Xc; g.n = n; g.p = p; g.tq = tq; g.F = F;
    g.min_split = min_split; g.max_depth = max_depth;
    g.hist = ((split_mode & 0xFFu) == 1);
    g.extra = ((split_mode & 0xFFu) == 2);
    g.mae = (int)((split_mode >> 8) & 1u);
    g.tie_draw = (int)((split_mode >> 9) & 1u);
    if (!g.hist) setup_exact(&g, Xc, n, p);
    uint64_t *tr = (uint64_t *)malloc(sizeof(uint64_t) * n);
    uint64_t *te = (uint64_t *)malloc(sizeof(uint64_t) * n);
    uint32_t *w = (uint32_t *)malloc(sizeof(uint32_t) * n);
    double *sum = (double *)malloc(sizeof(double) * n);
    double *yh = (double *)malloc(sizeof(double) * n);
    double *yt = (double *)malloc(sizeof(double) * n);
    or_tree tree = { NULL, 0, 0 };

    for (uint32_t task = task_begin; task < task_end; ++task) {
        uint32_t rep = task / k, fold = task % k;
        const int32_t *fr = fid + (uint64_t)rep * n;
        uint64_t ntr = 0, nte = 0;
        for (uint64_t i = 0; i < n; ++i) {
            if (fr[i] == (int32_t)fold) te[nte++] = i;
            else if (fr[i] != -2) tr[ntr++] = i; /* -2: excluded row (nested CV, R31) */
        }
        if (g.hist) setup_hist(&g, Xc, n, p, tr, ntr);
        for (uint32_t mi = 0; mi < n_mtry; ++mi) {
            g.mtry = mtrys[mi];
            for (uint64_t i = 0; i < nte; ++i) sum[i] = 0.0;
            for (uint32_t tt = 0; tt < Tmax; ++tt) {
                uint32_t k0, k1;
                tree_key(seed, task, tt, &k0, &k1);
                bootstrap(k0, k1, tr, ntr, n, (int)boot, w);
                grow_tree(&g, w, k0, k1, &tree, NULL, NULL);
                for (uint64_t i = 0; i < nte; ++i) sum[i] += tree_predict(&tree, Xc + te[i] * p);
                for (uint32_t ni = 0; ni < n_ntree; ++ni) {
                    if (ntrees[ni] != tt + 1) continue;
                    for (uint64_t i = 0; i < nte; ++i) {
                        double s = sum[i] / (double)(tt + 1);
                        yh[i] = (target == 1) ? exp(s) : s;
                        yt[i] = y[te[i]];
                    }
                    uint64_t o = (((uint64_t)mi * n_ntree + ni) * reps + rep) * k + fold;
                    fold_mape[o] = or_mape(yt, yh, nte);
                    if (pred) {
                        double *pp = pred + (((uint64_t)mi * n_ntree + ni) * reps + rep) * n;
                        for (uint64_t i = 0; i < nte; ++i) pp[te[i]] = yh[i];
                    }
                }
            }
        }
        if (g.hist) free_hist(&g, p);
    }
    free(tree.nodes);
    if (!g.hist) free_exact(&g, p);
    free(tr); free(te); free(w); free(sum); free(yh); free(yt);
    free(Xc); free(t); free(tq); free(fid);
    return 0;
}
