/*
 * oracle/c0.c -- CPU ORACLE (test infrastructure only) for C0, the affinity
 * build of L-tsNET: partial-BFS kNN, perplexity calibration, symmetrisation.
 *
 * TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library.  It shares no code with the CUDA
 * path (paper_2509_19785_b200/csrc) and must never be called by it.
 *
 * Plain, slow, obviously-correct fp64 code.  Readings of the paper used here
 * (DESIGN.md "Readings"): R4 hash tie-break, R5 k = min(round(3u), n-1) with
 * short rows allowed, R6 unreachable perplexity -> beta = inf, R7 nats and a
 * 1e-13 bisection stop, R8 conditional rows sum to 1.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* SplitMix64 finaliser (counter-based generator implemented independently on
 * both sides, R4).  key(v,w) = SplitMix64(seed XOR (v<<32 | w)). */
uint64_t oracle_splitmix64(uint64_t x)
{
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t oracle_tie_key(uint64_t seed, int64_t v, int64_t w)
{
    return oracle_splitmix64(seed ^ (((uint64_t)v << 32) | (uint64_t)(uint32_t)w));
}

typedef struct { int32_t w; int32_t hop; uint64_t key; } cand_t;

static int cmp_key_w(const void* a, const void* b)
{
    const cand_t* x = (const cand_t*)a;
    const cand_t* y = (const cand_t*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return (x->w > y->w) - (x->w < y->w);
}

static int cmp_hop_w(const void* a, const void* b)
{
    const cand_t* x = (const cand_t*)a;
    const cand_t* y = (const cand_t*)b;
    if (x->hop != y->hop) return x->hop < y->hop ? -1 : 1;
    return (x->w > y->w) - (x->w < y->w);
}

/*
 * O1. Partial BFS from v (Alg. 3 l.388 "Run BFS starting at v until
 * k vertices are visited"; §3.1 l.270 "when multiple vertices are of the same
 * shortest path distance from v, ties are broken randomly").
 * Whole BFS levels are taken while the running count stays <= k; from the
 * first level that would overflow, the k - taken vertices with the smallest
 * (key(v,w), w) are taken.  Output sorted by (hop, w).  Returns row length.
 * dist[] must be all -1 on entry and is restored on exit.
 */
static int64_t partial_bfs(int64_t n, const int64_t* indptr, const int32_t* indices, int64_t v,
                           int64_t k, uint64_t seed, int32_t* dist, int32_t* out_w, int32_t* out_hop)
{
    (void)n;
    int64_t cap_f = 64, cap_n = 64, cap_t = 64;
    int32_t* frontier = (int32_t*)malloc(sizeof(int32_t) * cap_f);
    int32_t* next = (int32_t*)malloc(sizeof(int32_t) * cap_n);
    int32_t* touched = (int32_t*)malloc(sizeof(int32_t) * cap_t);
    cand_t* row = (cand_t*)malloc(sizeof(cand_t) * (k > 0 ? k : 1));
    int64_t nf = 1, nt = 1, taken = 0;
    int32_t d = 0;
    frontier[0] = (int32_t)v;
    touched[0] = (int32_t)v;
    dist[v] = 0;
    while (taken < k && nf > 0) {
        d += 1;
        int64_t nn = 0;
        for (int64_t a = 0; a < nf; ++a) {
            int32_t f = frontier[a];
            for (int64_t e = indptr[f]; e < indptr[f + 1]; ++e) {
                int32_t w = indices[e];
                if (dist[w] != -1) continue;
                dist[w] = d;
                if (nn == cap_n) { cap_n *= 2; next = (int32_t*)realloc(next, sizeof(int32_t) * cap_n); }
                next[nn++] = w;
                if (nt == cap_t) { cap_t *= 2; touched = (int32_t*)realloc(touched, sizeof(int32_t) * cap_t); }
                touched[nt++] = w;
            }
        }
        if (nn == 0) break;
        if (taken + nn <= k) {
            for (int64_t a = 0; a < nn; ++a) {
                row[taken].w = next[a];
                row[taken].hop = d;
                row[taken].key = 0;
                taken++;
            }
            int32_t* tmp = frontier; frontier = next; next = tmp;
            int64_t tc = cap_f; cap_f = cap_n; cap_n = tc;
            nf = nn;
        } else {
            /* the cap = k - taken smallest (key, w) of the level: a bounded
             * max-heap of size cap over the level, then sorted */
            const int64_t cap = k - taken;
            cand_t* heap = (cand_t*)malloc(sizeof(cand_t) * cap);
            int64_t hs = 0;
            for (int64_t a = 0; a < nn; ++a) {
                cand_t c = {next[a], d, oracle_tie_key(seed, v, next[a])};
                if (hs < cap) {                       /* push, sift up */
                    int64_t i = hs++;
                    while (i > 0 && cmp_key_w(&heap[(i - 1) / 2], &c) < 0) { heap[i] = heap[(i - 1) / 2]; i = (i - 1) / 2; }
                    heap[i] = c;
                } else if (cmp_key_w(&c, &heap[0]) < 0) { /* replace the max, sift down */
                    int64_t i = 0;
                    for (;;) {
                        int64_t l = 2 * i + 1, r = l + 1, m = i;
                        const cand_t* big = &c;
                        if (l < hs && cmp_key_w(&heap[l], big) > 0) { m = l; big = &heap[l]; }
                        if (r < hs && cmp_key_w(&heap[r], big) > 0) { m = r; }
                        if (m == i) break;
                        heap[i] = heap[m];
                        i = m;
                    }
                    heap[i] = c;
                }
            }
            qsort(heap, (size_t)hs, sizeof(cand_t), cmp_key_w);
            for (int64_t a = 0; a < hs; ++a) row[taken++] = heap[a];
            free(heap);
            break;
        }
    }
    for (int64_t a = 0; a < nt; ++a) dist[touched[a]] = -1;
    qsort(row, (size_t)taken, sizeof(cand_t), cmp_hop_w);
    for (int64_t a = 0; a < taken; ++a) { out_w[a] = row[a].w; out_hop[a] = row[a].hop; }
    free(frontier); free(next); free(touched); free(row);
    return taken;
}

/* O1 over all sources (or a list of sources).  Row r of the output holds the
 * kNN of src[r] (src == NULL means src[r] = r).  out_len[r] = row length. */
void oracle_knn(int64_t n, const int64_t* indptr, const int32_t* indices, int64_t k, uint64_t seed,
                int64_t nsrc, const int64_t* src, int32_t* out_idx, int32_t* out_hop, int32_t* out_len)
{
#pragma omp parallel if (nsrc > 256)
    {
        int32_t* dist = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
        for (int64_t i = 0; i < n; ++i) dist[i] = -1;
#pragma omp for schedule(dynamic, 64)
        for (int64_t r = 0; r < nsrc; ++r) {
            int64_t v = src ? src[r] : r;
            out_len[r] = (int32_t)partial_bfs(n, indptr, indices, v, k, seed, dist,
                                              out_idx + r * k, out_hop + r * k);
        }
        free(dist);
    }
}

/* Entropy (nats) of the row distribution p_j ∝ exp(-beta D_j), Eq. 3
 * (PAPER.md:109-115): H = ln S + beta * sum_j D_j p_j, S = sum_j exp(-beta D_j). */
static double row_entropy(const double* D, int64_t len, double beta)
{
    double S = 0.0, SD = 0.0;
    for (int64_t j = 0; j < len; ++j) {
        double e = exp(-beta * D[j]);
        S += e;
        SD += D[j] * e;
    }
    return log(S) + beta * SD / S;
}

/*
 * O2. Calibrate one conditional row (Eq. 3): find beta_i =
 * 1/(2 sigma_i^2) so that the perplexity 2^H2 equals u, i.e. H (nats) = ln u.
 * d_ij = hop distance.  D_j = d_j^2 - d_min^2 (shift leaves p unchanged).
 * Special cases: len <= u -> beta = 0 (uniform); c_min >= u -> beta = inf
 * (uniform on the min-distance set, R6).  Otherwise bisection:
 *   beta = 1, lo = 0, hi = inf; repeat (max 200):
 *     H = H(beta); if |H - ln u| <= 1e-13 stop;
 *     if H > ln u: lo = beta, beta = (hi == inf) ? 2 beta : (lo+hi)/2
 *     else:        hi = beta, beta = (lo+hi)/2
 *     stop if hi is finite and the bracket holds <= 2 ulp (next(next(lo)) >= hi).
 * p_j = exp(-beta D_j) / S at the final beta.  Returns beta.
 */
double oracle_calibrate_row(const int32_t* hop, int64_t len, double u, double* p)
{
    if (len <= 0) return 0.0;
    int32_t dmin = hop[0];
    for (int64_t j = 1; j < len; ++j) if (hop[j] < dmin) dmin = hop[j];
    int64_t cmin = 0;
    for (int64_t j = 0; j < len; ++j) if (hop[j] == dmin) cmin++;
    if ((double)len <= u) {
        for (int64_t j = 0; j < len; ++j) p[j] = 1.0 / (double)len;
        return 0.0;
    }
    if ((double)cmin >= u) {
        for (int64_t j = 0; j < len; ++j) p[j] = (hop[j] == dmin) ? 1.0 / (double)cmin : 0.0;
        return INFINITY;
    }
    double* D = (double*)malloc(sizeof(double) * (size_t)len);
    for (int64_t j = 0; j < len; ++j) D[j] = (double)hop[j] * hop[j] - (double)dmin * dmin;
    const double Hstar = log(u);
    double beta = 1.0, lo = 0.0, hi = INFINITY;
    for (int it = 0; it < 200; ++it) {
        double H = row_entropy(D, len, beta);
        double diff = H - Hstar;
        if (fabs(diff) <= 1e-13) break;
        if (diff > 0) {
            lo = beta;
            beta = isinf(hi) ? 2.0 * beta : 0.5 * (lo + hi);
        } else {
            hi = beta;
            beta = 0.5 * (lo + hi);
        }
        if (!isinf(hi) && nextafter(nextafter(lo, INFINITY), INFINITY) >= hi) break;
    }
    double S = 0.0;
    for (int64_t j = 0; j < len; ++j) S += exp(-beta * D[j]);
    for (int64_t j = 0; j < len; ++j) p[j] = exp(-beta * D[j]) / S;
    free(D);
    return beta;
}

void oracle_calibrate(int64_t nrows, int64_t k, const int32_t* knn_hop, const int32_t* knn_len,
                      double u, double* p_cond, double* beta)
{
#pragma omp parallel for schedule(dynamic, 256) if (nrows > 1024)
    for (int64_t r = 0; r < nrows; ++r)
        beta[r] = oracle_calibrate_row(knn_hop + r * k, knn_len[r], u, p_cond + r * k);
}

typedef struct { int32_t col; double val; } ent_t;

static int cmp_col(const void* a, const void* b)
{
    const ent_t* x = (const ent_t*)a;
    const ent_t* y = (const ent_t*)b;
    return (x->col > y->col) - (x->col < y->col);
}

/*
 * O3. Symmetrise (Eq. 2): p_ij = (p_j|i + p_i|j) / (2n),
 * with p_j|i = 0 when j is not in N_k(i).  Row i collects its own entries
 * (i, j, p_j|i) and the transposed ones (i, j', p_i|j') of every row j' that
 * lists i; entries with equal column are added; exact zeros dropped.
 * Output CSR (columns ascending), values fp64.  Capacity: 2 * sum(len).
 * Returns nnz.
 */
int64_t oracle_symmetrize(int64_t n, int64_t k, const int32_t* knn_idx, const int32_t* knn_len,
                          const double* p_cond, int64_t* out_indptr, int32_t* out_indices,
                          double* out_values)
{
    int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t t = 0; t < knn_len[i]; ++t) {
            cnt[i]++;
            cnt[knn_idx[i * k + t]]++;
        }
    int64_t* start = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
    start[0] = 0;
    for (int64_t i = 0; i < n; ++i) start[i + 1] = start[i] + cnt[i];
    ent_t* buf = (ent_t*)malloc(sizeof(ent_t) * (size_t)(start[n] > 0 ? start[n] : 1));
    int64_t* fill = (int64_t*)calloc((size_t)n, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t t = 0; t < knn_len[i]; ++t) {
            int32_t j = knn_idx[i * k + t];
            double p = p_cond[i * k + t];
            buf[start[i] + fill[i]++] = (ent_t){j, p};
            buf[start[j] + fill[j]++] = (ent_t){(int32_t)i, p};
        }
    const double two_n = 2.0 * (double)n;
    int64_t nnz = 0;
    out_indptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) {
        ent_t* r = buf + start[i];
        int64_t len = cnt[i];
        qsort(r, (size_t)len, sizeof(ent_t), cmp_col);
        for (int64_t a = 0; a < len;) {
            int64_t b = a + 1;
            double s = r[a].val;
            while (b < len && r[b].col == r[a].col) { s += r[b].val; b++; }
            double pij = s / two_n;
            if (pij != 0.0) {
                out_indices[nnz] = r[a].col;
                out_values[nnz] = pij;
                nnz++;
            }
            a = b;
        }
        out_indptr[i + 1] = nnz;
    }
    free(cnt); free(start); free(buf); free(fill);
    return nnz;
}
