/*
 * tsnet.h -- C-ABI of the B200-native L-tsNET gradient hot path
 *            (arXiv 2509.19785, "L-tsNET", Alg. 3).
 *
 * One shared library, libtsnet.so (paper_2509_19785_b200/), built for sm_100a.
 * Every entry point is extern "C", takes plain pointers and sizes, returns an
 * int status (tsnet_status) and never throws.  The library never allocates
 * device memory on the hot path: scratch space is the caller's workspace,
 * sized by the matching *_workspace_bytes query.  All pointers are DEVICE
 * pointers unless marked [host].  All work is enqueued on the caller's CUDA
 * stream `stream` (a cudaStream_t; NULL = legacy default stream); calls are
 * asynchronous unless marked BLOCKING.  Asynchronous CUDA errors surface on a
 * later call.  Calls are re-entrant given distinct workspaces.
 *
 * Notation: n vertices, X_i = (x_i, y_i) the 2-D layout,
 * Delta_ij = X_i - X_j, r2 = |Delta_ij|^2, w_ij = 1/(1 + r2),
 * Z = sum_{k != l} w_kl, K_e = 1/(eps + r2).
 *
 * Entry points: the iteration (tsnet_grad, tsnet_grad_parts, tsnet_attr,
 * tsnet_step, tsnet_step_host, tsnet_cost; the phases tsnet_field_local /
 * tsnet_step_finish and the NCCL communicator for row shards); its set-up
 * (tsnet_build_P = C0, tsnet_pmds = the Pivot MDS initial layout; the
 * column-blocked and sliced-ELL re-layouts of P); the paper's other two
 * algorithms (tsnet_grad_tree: BH-tsNET, FIt-tsNET; tsnet_move); the quality
 * metrics of its evaluation (tsnet_quality).
 *
 * Data layout:
 *   layout Y / velocity / gains / gradient : n x 2 fp32, interleaved (x, y)
 *   graph and P                            : CSR, int64 indptr[n+1],
 *                                            int32 indices[nnz] (ascending per row),
 *                                            fp32 values[nnz] (P only)
 */
#ifndef TSNET_H
#define TSNET_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define TSNET_API __attribute__((visibility("default")))
#else
#define TSNET_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* tsnet_stream_t; /* == cudaStream_t */

/* Status codes.  Every call returns one of these. */
typedef enum {
    TSNET_OK = 0,
    TSNET_E_ARG = 1,         /* invalid argument (message in tsnet_last_error)            */
    TSNET_E_CAPACITY = 2,    /* P capacity too small; P->nnz holds the required nnz        */
    TSNET_E_CUDA = 3,        /* a CUDA runtime error (message in tsnet_last_error)        */
    TSNET_E_NCCL = 4,        /* reserved: multi-GPU collectives                             */
    TSNET_E_NONFINITE = 5,   /* returned by tsnet_read_stats when a non-finite value was seen */
    TSNET_W_PERPLEXITY = 6   /* warning from tsnet_build_P: some rows could not reach the
                                perplexity (c_min >= u, reading R6); P is still valid       */
} tsnet_status;

/* Undirected input graph G = (V, E) ("Input: Graph G=(V,E)"):
 * symmetric adjacency, no self loops, no duplicates, rows ascending.
 * Connectivity is NOT required (rows of small components are short). */
typedef struct {
    int64_t n;
    const int64_t* indptr;   /* device, n+1 */
    const int32_t* indices;  /* device, indptr[n] */
} tsnet_graph;

/* Sparse symmetric affinity matrix P (Eq. 2) in CSR.
 * `capacity` = allocated length of indices/values (input to tsnet_build_P),
 * `nnz` = stored entries (output of tsnet_build_P, input elsewhere).
 * `plan` = optional re-laid-out copy of the same P (device, caller-owned;
 * NULL = none) of kind `plan_kind`: TSNET_PLAN_CB (column-blocked,
 * tsnet_plan_build; 0 also means this kind) or TSNET_PLAN_SELL (sliced ELL,
 * tsnet_sell_build).  When set, the attractive SpMV (step a6) reads the plan
 * instead of indices/values; the caller must rebuild it whenever P's pattern
 * or values change (the library cannot detect a stale plan). */
#define TSNET_PLAN_CB 1
#define TSNET_PLAN_SELL 2
typedef struct {
    int64_t n;
    int64_t nnz;
    int64_t capacity;
    int64_t* indptr;         /* device, n+1 */
    int32_t* indices;        /* device, capacity */
    float* values;           /* device, capacity */
    const void* plan;        /* device, tsnet_plan_build / tsnet_sell_build output, or NULL */
    int32_t plan_kind;       /* TSNET_PLAN_CB (or 0) / TSNET_PLAN_SELL; ignored without a plan */
    int64_t plan_row_begin;  /* the rows [plan_row_begin, plan_row_end) the plan was built for (its
                                shard; [0, n) without one); a call whose rows differ fails with
                                TSNET_E_ARG.  Set by the caller with P->plan; ignored without a plan */
    int64_t plan_row_end;
} tsnet_csr;

/* Cost multipliers and interpolation grid policy.
 *   lambda_kl, lambda_c, lambda_r : Eq. 1 multipliers
 *   eps                           : entropy regulariser, 1/20 in the paper
 *   interp_P                      : interpolation points per interval ("P");
 *                                   only 3 is supported (TSNET_E_ARG otherwise)
 *   h_max, I_min, I_max           : grid policy of reading R9: per axis
 *                                   I = clamp(ceil(S/h_max), I_min, I_max) intervals over
 *                                   the bounding-box span S, rounded up to 2^a 3^b 5^c
 *                                   ("# of intervals I"); 1 <= I_min <= I_max
 *                                   <= TSNET_I_MAX_LIMIT. */
typedef struct {
    float lambda_kl, lambda_c, lambda_r, eps;
    int32_t interp_P;
    float h_max;
    int32_t I_min, I_max;
    int32_t spread;          /* how steps a1-a2 (the spread of the charges onto the grid,
                                PAPER.md:187-188) visit the points; the result is the same sum
                                (up to fp32 rounding order):
                                TSNET_SPREAD_AUTO (0): decided on the device every iteration
                                  (below);
                                TSNET_SPREAD_SORT (1): counting sort of the points by box (the
                                  box order is recorded in the workspace), then one pass over
                                  the points in that order, summed in registers while the box
                                  stays the same;
                                TSNET_SPREAD_RUNS (2): the same pass over the last recorded
                                  box order, without the sort (index order when none is
                                  recorded for this n); points that left their box since are
                                  summed one by one;
                                AUTO sorts on a fresh workspace, then runs over the recorded
                                order until a run averages fewer than 16 points (the points
                                moved across boxes since the sort), then sorts again.  Other
                                values: TSNET_E_ARG. */
} tsnet_grad_params;
#define TSNET_SPREAD_AUTO 0
#define TSNET_SPREAD_SORT 1
#define TSNET_SPREAD_RUNS 2

/* I <= 1024 (reading R9; N = 3 I <= 3072 nodes, FFT size M = 6 I <= 6144).
 * Workspace grid buffers are sized by the call's I_max (tsnet_workspace_bytes):
 * ~2.3 GB at I_max = 1024, ~150 MB at 256. */
#define TSNET_I_MAX_LIMIT 1024

/* Momentum/gains update (reading R12; the paper only says "Move each vertex v
 * in the direction of dC/dv"):
 *   gains <- max(gain_min, sign(g) != sign(v) ? gains + gain_inc : gain_dec * gains)
 *   v     <- momentum * v - eta * gains * g ;   Y <- Y + v ;   if recenter: Y <- Y - mean(Y) */
typedef struct {
    float eta, momentum, gain_inc, gain_dec, gain_min;
    int32_t recenter;
} tsnet_step_params;

/* Row shard for multi-GPU runs.  One process per GPU; rank
 * `rank` of `world` owns the contiguous rows [row_begin, row_end) of P, of the
 * gradient and of the state (vel, gains).  Y is REPLICATED: every rank holds
 * all n x 2 positions; each iteration the ranks
 *   - derive the same grid geometry from the full Y (no collective),
 *   - spread their own points (step a2) and sum the charge grid over the ranks
 *     (peer-memory all-reduce of the live cells, tsnet_comm_init),
 *   - convolve the reduced grid (replicated FFT), run the attractive SpMV and
 *     the gather/move for their own rows,
 *   - exchange Y -- tsnet_step only: pushed by the move into every rank's copy
 *     when Y is the communicator's layout buffer (tsnet_comm_layout), else
 *     all-gathered (equal padded slices, one ncclAllGather).
 * comm   : communicator from tsnet_comm_init (NULL only for the phase calls
 *          tsnet_field_local / tsnet_step_finish, which do no communication).
 * bounds : [host] world + 1 row offsets, bounds[r] .. bounds[r+1] = rank r's rows
 *          (tsnet_shard_rows); row_begin/row_end must equal bounds[rank], bounds[rank+1].
 * NULL shard, or world == 1 with rows [0, n), = one GPU, all rows.
 * With a plan (P->plan), it must have been built for the same rows
 * (tsnet_plan_build with this shard); recentring is not supported across
 * ranks (TSNET_E_ARG). */
typedef struct {
    int32_t rank, world;
    int64_t row_begin, row_end;
    void* comm;
    const int64_t* bounds;
} tsnet_shard;

#define TSNET_COMM_ID_BYTES 128

/* Per-call statistics kept in the workspace (read with tsnet_read_stats). */
typedef struct {
    double Z;                /* normaliser of the last gradient evaluation              */
    double lo_x, lo_y, S;    /* bounding box origin and span of the last evaluation     */
    double h_b;              /* interval (box) width                                    */
    int32_t I, N, M;         /* intervals per axis, nodes per axis (3I), FFT size (6I)   */
    int32_t nonfinite;       /* 1 if a non-finite coordinate/gradient was produced       */
    int32_t spread;          /* spread path of the last evaluation: TSNET_SPREAD_SORT / _RUNS */
    int64_t spread_points;   /* runs path: points of the last evaluation (0 after a sort)   */
    int64_t spread_flushes;  /* runs path: box runs it summed (flushes to the grid)         */
} tsnet_stats;

/* ---------------------------------------------------------------- C0 (set-up) */

/* k = round(3u) ("k = 3u"; half rounds up) when k_req <= 0, else
 * k_req; capped at n-1 (reading R5).  [host, pure] */
TSNET_API int32_t tsnet_resolve_k(int64_t n, double perplexity_u, int32_t k_req);

/* ------------------------------------------------ Pivot MDS initial layout */

/*
 * Alg. 3 line 2, "Compute initial layout D of G using Pivot MDS" (
 * tsNET* = tsNET with a PMDS initialisation).  Set-up,
 * outside the iteration loop.  Readings (R20-R22; the paper gives no
 * parameters):
 *   pivots: farthest-first -- the first is splitmix64(seed) mod n, each next
 *           maximises the hop distance to the chosen set (ties: smallest id);
 *           unreachable vertices count as distance n;
 *   layout: D2 = hop^2 (n x p), C = -1/2 (D2 - row means - column means +
 *           grand mean), v1, v2 = top-2 eigenvectors of C^T C (power
 *           iteration from splitmix64 start vectors, <= 1000 iterations,
 *           stop at |v' - v| < 1e-10; each flipped so its largest-magnitude
 *           entry is positive), Y = C [v1 v2] (zero mean by construction);
 *           a second eigenvalue <= 1e-12 of the first gives Y[:, 1] = 0.
 * g       : graph (device CSR), 1 <= n < 2^31 - 1.
 * pivots  : p, 1 <= p <= min(n, 1024) (SPEC default min(n, 250)).
 * Y       : out, device, n x 2 fp32 interleaved.
 * pivots_out (device int32[p]), hops_out (device int32[p][n], pivot-major),
 * eig_out (device fp64[2]: the two eigenvalues): optional outputs, NULL = skip.
 * ws      : device scratch of tsnet_pmds_workspace_bytes(n, p) bytes
 *           (~4 n p bytes for the hop matrix).
 * BLOCKING (one host round trip per BFS level).  TSNET_E_ARG on bad sizes.
 */
TSNET_API size_t tsnet_pmds_workspace_bytes(int64_t n, int32_t pivots);
TSNET_API int tsnet_pmds(const tsnet_graph* g, int32_t pivots, uint64_t seed, float* Y, int32_t* pivots_out,
                         int32_t* hops_out, double* eig_out, void* ws, size_t ws_bytes, tsnet_stream_t stream);

/* Device scratch bytes tsnet_build_P needs for n vertices and k neighbours. [host] */
TSNET_API size_t tsnet_build_P_workspace_bytes(int64_t n, int32_t k);

/*
 * C0: build P from G (Alg. 3 l.385-394), on the GPU.
 *  (1) partial BFS from every v until k vertices are visited (PAPER.md:388,
 *      §3.1 l.270): whole BFS levels while the count stays <= k; at the first
 *      overflowing level the k - taken vertices with the smallest
 *      (SplitMix64(seed ^ (v<<32 | w)), w) are taken (reading R4: "ties are
 *      broken randomly" made reproducible);
 *  (2) per row, beta_i = 1/(2 sigma_i^2) so that the perplexity of
 *      p_j|i ∝ exp(-beta_i d_ij^2) equals u (Eq. 3), d_ij =
 *      hop distance; bisection to |H - ln u| <= 1e-13 (R7); beta = 0 when the
 *      row has <= u entries, beta = inf (uniform on the nearest hop level)
 *      when that level alone has >= u entries (R6, counted -> TSNET_W_PERPLEXITY);
 *  (3) p_ij = (p_j|i + p_i|j) / (2n) (Eq. 2), computed in fp64, exact zeros
 *      dropped, rounded to fp32, columns ascending.
 * Outputs: knn_idx / knn_hop [n * k] (row v = its kNN sorted by (hop, w),
 * entries >= knn_len[v] are -1), knn_len [n], beta [n] (fp64; may be NULL),
 * P (indptr/indices/values, P->nnz).  If P->capacity < nnz the call returns
 * TSNET_E_CAPACITY with P->nnz = the required nnz (2 n k always suffices).
 * BLOCKING: synchronises `stream` (it returns nnz on the host).
 */
TSNET_API int tsnet_build_P(const tsnet_graph* g, double perplexity_u, int32_t k, uint64_t seed,
                  tsnet_csr* P, int32_t* knn_idx, int32_t* knn_hop, int32_t* knn_len, double* beta,
                  void* ws, size_t ws_bytes, tsnet_stream_t stream);

/* ------------------------------------------------------- the per-iteration path */

/* Device workspace bytes for tsnet_grad / tsnet_grad_parts / tsnet_step /
 * tsnet_cost on n vertices and nnz entries of P. [host] */
TSNET_API size_t tsnet_workspace_bytes(int64_t n, int64_t nnz, const tsnet_grad_params* gp, const tsnet_shard* shard);

/*
 * Gradient of C = C_KL + C_CMP + C_ENT at layout Y (one L-tsNET iteration,
 * Alg. 3 l.396-404):
 *   grad_i = 4 lambda_kl (F_attr,i - F_rep,i) + (lambda_c / n) X_i + lambda_r g_ent,i
 *   F_attr,i = sum_j p_ij w_ij Delta_ij                (Eq. 6 term 1, exact sparse SpMV)
 *   F_rep,i  ~ sum_j w_ij^2 Delta_ij / Z,  Z ~ sum_{k!=l} w_kl   (Eq. 6 term 2, FIt-SNE
 *              interpolation)
 *   g_ent,i  ~ -(1/n^2) sum_j Delta_ij / (eps + r2)    (Eq. 8)
 * The two interpolated sums use P=3 Lagrange nodes per interval on an
 * I x I-interval grid, convolved by FFT (local-moment form).
 * grad: (row_end - row_begin) x 2 fp32 (device; n x 2 without a shard), row q
 * = vertex row_begin + q.  Z: device fp64 scalar (may be NULL).  Sharded:
 * all-reduces the charge grid over shard->comm.
 */
TSNET_API int tsnet_grad(const tsnet_csr* P, const float* Y, const tsnet_grad_params* gp, const tsnet_shard* shard,
               float* grad, double* Z, void* ws, size_t ws_bytes, tsnet_stream_t stream);

/* The attractive term alone (step a6, Eq. 6 first term):
 *   f_attr,i = sum_{j in row i} p_ij w_ij Delta_ij
 * for the rows [row_begin, row_end) of `shard` (all n rows if NULL; only the row
 * range of the shard is used): f_attr is (row_end - row_begin) x 2 fp32
 * (device), row q = vertex row_begin + q.  Y is the full n x 2 layout.  Uses
 * P->plan when set (its rows must be the shard's), else the row-wise CSR
 * kernel.  Needs no workspace.  Async.  (Also the kernel bench.py times for the
 * roofline.) */
TSNET_API int tsnet_attr(const tsnet_csr* P, const float* Y, const tsnet_shard* shard, float* f_attr,
                         tsnet_stream_t stream);

/* Same evaluation, returning the parts separately (diagnostics / parity):
 *   f_attr  = F_attr (n x 2), f_field = -4 lambda_kl F_rep + lambda_r g_ent (n x 2),
 * so that grad = 4 lambda_kl f_attr + f_field + (lambda_c / n) Y.  Any output may be NULL. */
TSNET_API int tsnet_grad_parts(const tsnet_csr* P, const float* Y, const tsnet_grad_params* gp,
                     const tsnet_shard* shard, float* f_attr, float* f_field, double* Z,
                     void* ws, size_t ws_bytes, tsnet_stream_t stream);

/*
 * One full iteration: gradient at Y (as tsnet_grad) followed by the
 * momentum/gains move ("Move each vertex v in the direction of
 * dC/dv"; reading R12), in place on Y, vel, gains (n x 2 fp32 each).
 * Sharded: rows [row_begin, row_end) of vel/gains are updated, and every
 * rank's new rows reach every rank's Y: on the communicator's layout buffer
 * (tsnet_comm_layout) the move stores them into the peers' copies and the next
 * tsnet_step waits until every peer's have landed (tsnet_comm_layout_sync
 * before reading Y outside tsnet_step); on any other Y they are all-gathered
 * over shard->comm before the call returns (stream order).
 */
TSNET_API int tsnet_step(const tsnet_csr* P, float* Y, float* vel, float* gains, const tsnet_grad_params* gp,
               const tsnet_step_params* sp, const tsnet_shard* shard, void* ws, size_t ws_bytes,
               tsnet_stream_t stream);

/*
 * Same as tsnet_step with HOST state buffers (pinned host memory recommended):
 * copies Y, vel, gains host -> device into the workspace, runs one iteration
 * and copies them back device -> host.  P stays on the device.  BLOCKING
 * (returns after the results are in the host buffers; work is ordered after
 * earlier work on `stream`).  Used for the end-to-end measurement of the
 * host-facing API.
 * Without recentring, shards or a plan (and n >= 4 * 16384), the rows are
 * processed in 4 row chunks so that the download
 * of a moved chunk overlaps the attractive SpMV of the next ones; the new
 * positions go to a separate workspace buffer until every chunk's SpMV has
 * read the old ones.  Results equal tsnet_step's up to fp32 summation order
 * of rows split across warps.
 */
TSNET_API int tsnet_step_host(const tsnet_csr* P, float* Y_host, float* vel_host, float* gains_host,
                    const tsnet_grad_params* gp, const tsnet_step_params* sp, const tsnet_shard* shard,
                    void* ws, size_t ws_bytes, tsnet_stream_t stream);

/*
 * Cost C = (C_KL, C_CMP, C_ENT*) written to out3 (device, 3 doubles):
 *   C_KL  = lambda_kl sum_{p_ij > 0} p_ij ln(p_ij Z / w_ij)    (Eq. 1/4, natural log, R14)
 *   C_CMP = lambda_c / (2n) sum_i |X_i|^2                       (Eq. 1)
 *   C_ENT* = -lambda_r / (4 n^2) sum_{i != j} ln(eps + r2_ij)   (reading R1 of PAPER.md:90)
 * mode 0: exact (Z and C_ENT* by O(n^2) tiles, fp64 accumulation);
 * mode 1: O(n) -- Z and sum_{i != j} ln(eps + r2) from the interpolation grid
 *         (Parseval sums of the spread W1 against K1 and ln(eps + d^2)).
 */
TSNET_API int tsnet_cost(const tsnet_csr* P, const float* Y, const tsnet_grad_params* gp, int32_t mode,
               const tsnet_shard* shard, double* out3, void* ws, size_t ws_bytes, tsnet_stream_t stream);

/* ------------------------------------- quadtree variants (BH-/FIt-tsNET) */

/*
 * The gradient of the paper's other two algorithms (NEXT-3), on one GPU:
 * BH-tsNET (variant 0, Alg. 2): KL repulsion
 * (Eq. 6 second term, Z summed the same way) and the entropy gradient of Eq. 7
 * (read with R2/R3) by a Barnes-Hut walk of a quadtree of Y
 * (PAPER.md:172-173); FIt-tsNET (variant 1): the repulsion
 * from the interpolation grid (as tsnet_grad with lambda_r = 0) and only the
 * entropy from the quadtree.  Attraction: the same SpMV as tsnet_grad.
 * Tree (R23): root = square of the bounding box, depth 16, nodes = runs of
 * the Morton-sorted points; a node of > 1 point summarises for X_i when
 * side^2 < theta^2 |X_i - com|^2 (fp64).  theta in [0, 0.7); theta = 0 gives
 * the exact O(n^2) gradient.
 * grad  : out, device n x 2 fp32 (the full gradient, as tsnet_grad).
 * Z_out : optional device fp64: Z of the tree (variant 0) or of the grid (1).
 * ws    : the tsnet_workspace_bytes workspace; tree_ws: device scratch of
 *         tsnet_tree_workspace_bytes(n) bytes.  Single GPU, n < 2^26.
 */
TSNET_API size_t tsnet_tree_workspace_bytes(int64_t n);
TSNET_API int tsnet_grad_tree(const tsnet_csr* P, const float* Y, const tsnet_grad_params* gp, double theta,
                              int32_t variant, float* grad, double* Z_out, void* ws, size_t ws_bytes, void* tree_ws,
                              size_t tree_ws_bytes, tsnet_stream_t stream);

/* ----------------------------------------- drawing quality; stand-alone move */

/*
 * Quality metrics of §4.3 (NEXT-4) of a drawing Y (device n x 2 fp32) of g:
 * out2[0] = neighbourhood preservation NP (mean over v of the
 * Jaccard index of the r-hop neighbourhood and the same number of nearest
 * drawn vertices, fp64 squared distances, ties by smaller id; r = 2 in the
 * paper), out2[1] = aggregated stress with the optimal scale (PAPER.md:607-611,
 * SPEC stress; NaN on a disconnected graph).  Readings R25-R26.  out2: device
 * fp64[2].  2 <= n <= 24576 (an evaluation of small drawings: a CTA per vertex,
 * O(n (n + m)) work).  ws: device scratch of tsnet_quality_workspace_bytes(n).
 */
TSNET_API size_t tsnet_quality_workspace_bytes(int64_t n);
TSNET_API int tsnet_quality(const tsnet_graph* g, const float* Y, int32_t r, double* out2, void* ws, size_t ws_bytes,
                            tsnet_stream_t stream);

/*
 * The gains/momentum move of step a7 (reading R12) for a
 * gradient computed elsewhere (e.g. tsnet_grad_tree): in place on Y, vel,
 * gains (device n x 2 fp32 each); grad device n x 2 fp32.  No recentring.
 */
TSNET_API int tsnet_move(float* Y, float* vel, float* gains, const float* grad, int64_t n,
                         const tsnet_step_params* sp, tsnet_stream_t stream);

/* ------------------------------------------- column-blocked layout of P (a6) */

/*
 * The attractive SpMV (Eq. 6 first term) gathers Y_j for every
 * stored entry of P.  On graphs without locality (config 4) those gathers, not
 * HBM, bound a row-wise CSR kernel (the L1->L2 request path: about one random
 * gather per SM-cycle).  A plan is P re-laid out for a kernel that reads Y_j
 * from shared memory instead:
 *   panels  : the rows of `shard` (all rows if NULL) dealt to P = 148 k panels
 *             (k = ceil(rows / (148 * 8192))) by longest-processing-time on
 *             (entries + 8), at most 8192 rows each; one CTA per panel keeps
 *             Y_i and the partial F_i of its rows in shared memory;
 *   blocks  : columns in blocks of 4096 points, streamed through a shared
 *             ring by TMA bulk copies;
 *   tiles   : per (panel, block) the entries sorted by (row, column) and cut
 *             into 512 equal contiguous chunks, one per lane; slot (step k,
 *             lane L) = k-th entry of chunk L as (column in block | local row
 *             << 12 | run flags, p_ij fp32), tiles padded to whole steps with
 *             (0, +0.0) slots.
 * The plan holds the values: the kernel that uses it reads no CSR array.
 * Results equal the CSR kernel's up to fp32 summation order.
 *
 * tsnet_plan_query : bytes of the plan (an upper bound) and of the build
 *                    workspace for this P and shard.  BLOCKING (reads
 *                    P->indptr to cut the rows).
 * tsnet_plan_build : writes the plan into `plan` (device, 256-byte aligned,
 *                    >= plan_bytes) using `ws` as scratch (~24 bytes per
 *                    stored entry; CUB radix sort).  BLOCKING.  Set P->plan =
 *                    plan and P->plan_kind = TSNET_PLAN_CB afterwards.  Needs
 *                    fewer than 2^32 entries in the shard and n < 2^31
 *                    (TSNET_E_ARG otherwise).
 * tsnet_plan_partition : the host cut alone (for tests): rows [row_begin,
 *                    row_end) of the HOST indptr into P = groups * k panels of
 *                    at most rows_cap rows.  Per row q (shard-local):
 *                    row_panel[q], row_local[q] (its index inside the panel,
 *                    rows ascending); panel_off[P + 1] = exclusive scan of
 *                    the panel sizes; panel_rows[panel_off[p] + l] = the row
 *                    of panel p with local index l.  Returns P (<= max_panels),
 *                    or -1.  [host, pure]
 */
TSNET_API int tsnet_plan_query(const tsnet_csr* P, const tsnet_shard* shard, size_t* plan_bytes, size_t* ws_bytes,
                               tsnet_stream_t stream);
TSNET_API int tsnet_plan_build(const tsnet_csr* P, const tsnet_shard* shard, void* plan, size_t plan_bytes, void* ws,
                               size_t ws_bytes, tsnet_stream_t stream);
TSNET_API int32_t tsnet_plan_partition(const int64_t* indptr_host, int64_t row_begin, int64_t row_end,
                                       int32_t groups, int32_t rows_cap, int32_t* row_panel, int32_t* row_local,
                                       int32_t* panel_off, int32_t* panel_rows, int64_t max_panels);
/* ------------------------------------------------- sliced-ELL layout of P (a6) */

/*
 * Same product as the CSR SpMV (Eq. 6 first term), P re-laid
 * out for graphs whose consecutive vertices have similar neighbourhoods
 * (meshes, config 5): rows of `shard` (all rows if NULL) in slices of 32
 * consecutive rows; a lane owns a row, a warp a slice; slot (slice s, step k,
 * lane) = (column, p_ij) of the k-th stored entry of row 32 s + lane (CSR
 * order), at base[s] + 32 k + lane, base = exclusive scan of 32 * (longest row
 * of the slice); missing entries = (own row, 0.0), which add exactly 0.
 * Result identical to the CSR kernel's up to fp32 summation order.
 *
 * tsnet_sell_query : bytes of the plan, and slots per stored entry (>= 1; the
 *                    padding; large on power-law graphs, where the CSR kernel
 *                    is the better choice).  BLOCKING (reads P->indptr).
 * tsnet_sell_build : writes the plan into `plan` (device, 256-byte aligned,
 *                    >= plan_bytes).  BLOCKING.  Then set P->plan = plan and
 *                    P->plan_kind = TSNET_PLAN_SELL.  Needs n < 2^31.
 */
TSNET_API int tsnet_sell_query(const tsnet_csr* P, const tsnet_shard* shard, size_t* plan_bytes,
                               double* slots_per_nnz, tsnet_stream_t stream);
TSNET_API int tsnet_sell_build(const tsnet_csr* P, const tsnet_shard* shard, void* plan, size_t plan_bytes,
                               tsnet_stream_t stream);


/* ------------------------------------------------------------- multi-GPU (§8(e)) */

/* Communicator (NCCL is loaded at run time; TSNET_E_ARG if it cannot be).
 * tsnet_comm_unique_id : on one rank, write the 128-byte id to share with the
 *                        others (e.g. through torch.distributed). [host]
 * tsnet_comm_init      : every rank, collectively: communicator of `world`
 *                        (<= 64) ranks on the calling thread's current device.
 *                        It allocates a peer-exchange buffer for charge grids of
 *                        up to 3 I_max nodes per axis (2 x 16 (3 I_max)^2 bytes +
 *                        256) and maps every peer's buffer (CUDA IPC); when all
 *                        ranks sit on distinct, peer-accessible devices, the
 *                        charge-grid sum of each step is a peer-memory
 *                        all-reduce of the live N x N cells (device-side flag
 *                        handshake, loads over NVLink), else an ncclAllReduce
 *                        of the whole (3 I_max)^2 grid.  BLOCKING.
 * tsnet_comm_peer_reduce : 1 if the communicator uses the peer-memory grid
 *                        all-reduce, else 0. [host]
 * tsnet_comm_destroy   : release it (synchronises the device). */
TSNET_API int tsnet_comm_unique_id(uint8_t* id_out);
TSNET_API int tsnet_comm_init(const uint8_t* id, int32_t world, int32_t rank, int32_t I_max, void** comm);
TSNET_API int tsnet_comm_peer_reduce(const void* comm);

/* The replicated layout Y owned by the communicator (SURVEY.md §8(e) "fused
 * all-gather"; the move, Alg. 3 l.405 PAPER.md:405, writes its new positions
 * straight into every rank's copy).
 * tsnet_comm_layout      : every rank, collectively (same n): allocate this
 *                          rank's n x 2 fp32 device buffer (owned and freed by
 *                          the communicator; *Y_out stays valid until
 *                          tsnet_comm_destroy) and map every peer's buffer.  A
 *                          second call with the same n returns the same buffer.
 *                          When every peer is mapped (tsnet_comm_layout_push),
 *                          tsnet_step called with Y == this buffer skips the
 *                          all-gather: k_update stores each moved position into
 *                          all ranks' buffers over NVLink, after a device-side
 *                          wait until every peer has finished reading Y for the
 *                          iteration, and the next tsnet_step waits until every
 *                          peer's move has landed.  Any other Y: the all-gather
 *                          of tsnet_step.
 * tsnet_comm_layout_push : 1 if the push is in use.
 * tsnet_comm_layout_sync : enqueue on `stream` a wait until every peer's move of
 *                          every iteration this rank has completed has landed in
 *                          this rank's buffer (before the caller reads or
 *                          overwrites Y outside tsnet_step). */
TSNET_API int tsnet_comm_layout(void* comm, int64_t n, float** Y_out);
TSNET_API int tsnet_comm_layout_push(const void* comm);
TSNET_API int tsnet_comm_layout_sync(void* comm, tsnet_stream_t stream);
TSNET_API int tsnet_comm_destroy(void* comm);

/* The charge-grid sum of `count` workspaces on the calling device (shards run
 * on one device, and the single-device emulation of several ranks): after
 * tsnet_field_local on each, every workspace's live grid becomes the sum of all
 * (the same N, from the first workspace's geometry).  n, nnz, gp: as for
 * tsnet_workspace_bytes.  BLOCKING. */
TSNET_API int tsnet_grids_sum(int32_t count, void* const* ws_list, size_t ws_bytes, int64_t n, int64_t nnz,
                              const tsnet_grad_params* gp, tsnet_stream_t stream);

/* Row shards: bounds[0..world] (host) cutting rows [0, n) of the HOST indptr
 * into `world` contiguous ranges balanced on nnz + rows (the per-rank bytes of
 * steps a6/a7).  Returns world, or -1 on bad arguments.  [host, pure] */
TSNET_API int32_t tsnet_shard_rows(const int64_t* indptr_host, int64_t n, int32_t world, int64_t* bounds);

/* The two halves of tsnet_step around its collectives, for callers that run
 * their own communication (and for single-GPU emulation of several ranks):
 * tsnet_field_local : steps a0-a2 -- geometry from the full Y, box sort and
 *                     spread of the shard's own rows into the charge grid in ws.
 * tsnet_ws_grid     : where that grid lives: byte offset into ws and its
 *                     length in floats (the buffer tsnet_step all-reduces). [host]
 * tsnet_step_finish : steps a3-a7 from the (summed) grid in ws: convolution, Z,
 *                     attractive SpMV and gather + move of the own rows of Y,
 *                     vel, gains (full n x 2 arrays).  No communication.
 * tsnet_step = field_local + all-reduce(grid) + step_finish + exchange of Y. */
TSNET_API int tsnet_field_local(const tsnet_csr* P, const float* Y, const tsnet_grad_params* gp,
                                const tsnet_shard* shard, void* ws, size_t ws_bytes, tsnet_stream_t stream);
TSNET_API int tsnet_ws_grid(int64_t n, int64_t nnz, const tsnet_grad_params* gp, size_t* offset_bytes,
                            size_t* count_floats);
TSNET_API int tsnet_step_finish(const tsnet_csr* P, float* Y, float* vel, float* gains, const tsnet_grad_params* gp,
                                const tsnet_step_params* sp, const tsnet_shard* shard, void* ws, size_t ws_bytes,
                                tsnet_stream_t stream);

/* Copy the statistics of the last evaluation from the workspace. BLOCKING. [host out] */
TSNET_API int tsnet_read_stats(const void* ws, tsnet_stats* out, tsnet_stream_t stream);

/* Thread-local message describing the last error of this thread. [host] */
TSNET_API const char* tsnet_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* TSNET_H */
