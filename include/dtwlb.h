/*
 * dtwlb.h -- C ABI of the B200-native two-pass DTW k-NN library (libdtwlb.so).
 *
 * Method: D. Lemire, "Faster Retrieval with a Two-Pass Dynamic-Time-Warping
 * Lower Bound" (arXiv:0811.3301).  "P:n" = line n of the paper's LaTeX source
 * (PAPER.md), with the section / equation / algorithm named alongside.
 *
 * Conventions for every entry point
 * ---------------------------------
 * - Series are float32, row-major [count][n] (n contiguous), indexed 0..n-1
 *   (the paper indexes 1..n).  x is the candidate (database row),
 *   y the query (Alg. 3).
 * - Pointers are CUDA DEVICE pointers unless a function says otherwise;
 *   nn_search additionally accepts host pointers (see there).
 * - The caller owns all memory.  The library never frees a caller pointer and
 *   keeps none after return (it caches its own device workspace, one per CUDA
 *   device ordinal: calls on different devices never share scratch memory; calls
 *   are serialised by a process-wide lock).
 * - Calls run on the CUDA device current on the calling thread, which must be an
 *   sm_100 device (checked once per device).
 * - `stream` is a cudaStream_t (NULL = legacy default stream).  The per-kernel
 *   entry points are stream-ordered and asynchronous; nn_search returns when
 *   its outputs are complete.
 * - p is the exponent of DTW_p / LB_p: 1 or 2 (DTW_p of P:193-201).  The
 *   locality constraint w (Sakoe-Chiba band |i-j| <= w) may be any
 *   w >= 0; w >= n is clamped to n-1 (the window saturates).
 * - Return value: DTWLB_OK (0) or a dtwlb_status.  dtwlb_last_error() returns a
 *   thread-local message describing the last failure.  No C++ exception ever
 *   crosses this boundary; there is no CPU fallback: without a usable sm_100
 *   device every call returns DTWLB_ECUDA.
 * - Distances/bounds returned are ROOTED (DTW_p = q_{1,1}^(1/p));
 *   internally everything is accumulated in p-th-power space.
 */
#ifndef DTWLB_H
#define DTWLB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum dtwlb_status {
    DTWLB_OK = 0,
    DTWLB_EINVAL = 1,       /* bad size / pointer / argument combination      */
    DTWLB_EUNSUPPORTED = 2, /* p not in {1,2}; k above DTWLB_MAX_K             */
    DTWLB_ENOMEM = 3,       /* device workspace allocation failed              */
    DTWLB_ECUDA = 4,        /* CUDA runtime error or no sm_100 device          */
    DTWLB_ENCCL = 5         /* NCCL error in the sharded path                  */
} dtwlb_status;

#define DTWLB_MAX_K 1024

/* Warping envelope (section "Computing Lower Bounds on the DTW"):
 *   U_i = max{x_k : |k-i| <= w},  L_i = min{x_k : |k-i| <= w},
 * window clipped to [0, n-1].  x, U, L: device [count][n].  Exact (min/max
 * do not round), so results are bit-identical to the definition.
 * Errors: EINVAL if n < 1, w < 0, count < 0, or a NULL pointer with count > 0. */
int lb_envelope(const float *x, int32_t n, int32_t w, float *U, float *L, int64_t count,
                void *stream);

/* LB_Keogh_p (section "LB_Keogh"; Alg. 2 lines P:507-514):
 *   out[q][c] = ( sum_i d(x_c,i , [L_q,i , U_q,i])^p )^(1/p)
 * = ||x_c - H(x_c, y_q)||_p with H the projection of Eq. (1).
 * q_env: device [2][Q][n] (the U block of all Q queries, then the L block), as
 * written by lb_envelope into a contiguous buffer.  db: device [N][n].
 * out: device [Q][N] float32.  This is the dense (test / inspection) form of
 * the bound pass that nn_search fuses.  Q <= 8 (n % 4 == 0, 16-byte aligned db)
 * runs the streaming kernel nn_search uses for few queries, else the tiled one.
 * Errors: EINVAL (sizes, NULL, n < 1), EUNSUPPORTED (p not 1 or 2). */
int lb_keogh(const float *q_env, const float *db, int64_t Q, int64_t N, int32_t n, int32_t p,
             float *out, void *stream);

/* Piecewise-sum lower bound (section "Using a multidimensional
 * indexing structure"), the cascade's pre-filter:
 *   out[q][c]^p = sum_j d(P(x_c)_j, [P(L_q)_j, P(U_q)_j])^p * (p == 2 ? 1/s : 1)
 * with P(v)_j = sum_{i in C_j} v_i over the cover C_j = [j*s, min((j+1)*s, n)),
 * s = 8.  p = 1 is the paper's bound (<= LB_Keogh_1); p = 2 adds
 * the per-segment Cauchy-Schwarz step (sum_{C_j} d_i^2 >= (sum_{C_j} d_i)^2/|C_j|,
 * |C_j| <= s; reading c18).  Evaluated with outward rounding, so the
 * returned value never exceeds the exact bound (hence never exceeds LB_Keogh_p
 * or DTW_p).  q_env, db, out and errors as lb_keogh. */
int lb_piecewise(const float *q_env, const float *db, int64_t Q, int64_t N, int32_t n, int32_t p,
                 float *out, void *stream);

/* Symmetric piecewise-sum bound, the gate nn_search runs over every pair
 * (reading c20):
 *   out[q][c] = max(lb_piecewise(x_c | envelope of y_q), lb_piecewise(y_q | envelope of x_c))
 * The second term is the piecewise-sum bound with the roles of query and
 * candidate exchanged -- a lower bound of LB_Keogh_p(y, x) <= DTW_p(y, x), and
 * DTW_p is symmetric -- so the maximum is a lower bound of DTW_p(x, y).
 * Both terms outward-rounded as lb_piecewise.  q: device [Q][n] queries; q_env:
 * device [2][Q][n] envelope of q with locality w; db: device [N][n]; the
 * candidates' envelopes (same w) are computed inside.  out: device [Q][N] rooted.
 * Errors: as lb_keogh, plus EINVAL for w < 0. */
int lb_piecewise_sym(const float *q, const float *q_env, const float *db, int64_t Q, int64_t N,
                     int32_t n, int32_t w, int32_t p, float *out, void *stream);

/* LB_Improved_p (section "LB_Improved"; Alg. 3 lines P:587-606):
 *   out[q][c]^p = LB_Keogh_p(x_c, y_q)^p + LB_Keogh_p(y_q, H(x_c, y_q))^p,
 * i.e. the first pass plus the distance of y to the envelope of the
 * projection H, both with locality constraint w.  q: device [Q][n] queries;
 * q_env: device [2][Q][n] envelope of q with the same w; db: device [N][n];
 * out: device [Q][N].  Dense form; nn_search evaluates it only on LB_Keogh
 * survivors.  Any n: n <= 1024 runs the survivor kernel (a pair's n samples in one
 * warp's registers, at most 32 per lane), longer series a warp-per-pair kernel with
 * the same closed form.  Errors: as lb_keogh, plus EINVAL for w < 0. */
int lb_improved(const float *q, const float *q_env, const float *db, int64_t Q, int64_t N,
                int32_t n, int32_t w, int32_t p, float *out, void *stream);

/* Banded DTW_p of row pairs (section "Dynamic Time Warping"):
 *   out[r] = DTW_p(x[r], y[r]) with the band |i-j| <= w, rooted.
 * p = 0 encodes p = infinity: DTW_inf, the max instead of the sum along the path
 * (P:211-214); exact in fp32 (only |x_i - y_j| rounds).  p = 4 is DTW_4, the third
 * member of the Appendix C comparison.  w >= n-1 is the unconstrained DTW
 * (Appendix B workload).
 * x, y: device [count][n]; out: device [count].
 * Errors: EINVAL (sizes, NULL, n < 1, w < 0, count > 2^31 - 1), EUNSUPPORTED (p not 0, 1,
 * 2 or 4). */
int dtw_band(const float *x, const float *y, int32_t n, int32_t w, int32_t p, float *out,
             int64_t count, void *stream);

/* Options of nn_search (all fields optional: pass NULL for defaults). */
typedef struct nn_opts {
    float eps;             /* prune iff bound > tau*(1+eps), tau = current k-th best
                              (p-th-power space); default 1e-3 (reading c13) */
    int64_t index_base;    /* added to every returned index (database shards)        */
    int32_t query_block;   /* queries per pipeline block; 0 = automatic              */
    int32_t flags;         /* DTWLB_KEOGH_ONLY: skip the LB_Improved pass (Alg. 2);
                              DTWLB_NO_PREFILTER: LB_Keogh over every pair (Alg. 3
                              literally) instead of the piecewise-sum pre-filter;
                              DTWLB_NO_CASCADE, DTWLB_NO_STREAM, DTWLB_NO_ABANDON: see below */
    /* Database-sharded search: called once per query block after the
     * first (best-first) range, with thr = DEVICE pointer to the block's count
     * thresholds tau_q^p (1+eps) (+inf until k results), stream-ordered on `stream`.
     * The callee may lower them in place, e.g. to the minimum over all shards
     * (an all-reduce MIN): a shard's k-th best is >= the global k-th best, so any
     * shard's threshold is safe for every shard.  All ranks must use the same
     * query_block so that the calls match.  NULL = no exchange. */
    void (*exchange)(float *thr, int64_t count, void *user);
    void *exchange_user;
    /* Optional database index (the query-independent part of the cascade, built once for
     * a database that is searched many times -- the paper's setting): DEVICE
     * [2][N][n], the envelope U(x) block then L(x) block of every database row with THIS
     * call's w, exactly as lb_envelope(db, n, w, U, L, N) writes it.  NULL = computed
     * inside the call.  A wrong index gives wrong bounds (not checked). */
    const float *db_env;
    /* Database-sharded search: the number of shards G whose thresholds the exchange combines
     * (0 or 1 = unsharded).  The best-first seed range -- the candidates searched first, whose
     * k-th best DTW seeds the threshold -- is sized for the WHOLE database and split among the
     * shards (each shard seeds from 1/G of it), so G shards together do the seed work of one
     * search instead of G times it.  Affects speed only, never the result. */
    int32_t shards;
    /* Further exchanges inside the LAST range's DTW walk, when the thresholds tighten fastest:
     * the exchange is also called after that walk's rounds 2, 4, ..., 2*exchange_walk
     * (0 <= exchange_walk <= 3; rounds a shard does not run still call it, with its final
     * thresholds), so a block makes exactly 1 + exchange_walk calls on every shard.  Speed
     * only (each call may only lower thresholds to values >= the global k-th best). */
    int32_t exchange_walk;
    /* The library's own threshold exchange (alternative to `exchange`, used when `exchange` is
     * NULL): an NCCL communicator from dtwlb_comm_init; at every exchange point the block's
     * thresholds are min-reduced in place with ONE ncclAllReduce(ncclMin) on `stream` -- no host
     * callback.  Same call schedule as `exchange` (1 + exchange_walk per block, equal
     * query_block on every rank).  NULL = no exchange. */
    void *nccl_comm;
} nn_opts;

#define DTWLB_KEOGH_ONLY 1
#define DTWLB_NO_PREFILTER 2
#define DTWLB_NO_CASCADE 4   /* DTW abandons on the row minimum alone (no LB_Keogh suffix) */
#define DTWLB_NO_STREAM 8    /* Q <= 8: use the tiled bound pass instead of the streaming one */
#define DTWLB_NO_ABANDON 16  /* no early abandon inside DTW: every pair the bounds pass runs to its last row
                                (the pruning by LB_Keogh / LB_Improved before DTW is unchanged); same k-NN */

/* Counters of one nn_search call (host struct, filled on return). */
typedef struct nn_stats {
    int64_t pairs;            /* Q*N query-candidate pairs                            */
    int64_t keogh_evaluated;  /* LB_Keogh evaluations (= pairs without the pre-filter) */
    int64_t improved_evaluated; /* LB_Improved evaluations (LB_Keogh survivors seen)  */
    int64_t dtw_evaluated;    /* DTW evaluations started                              */
    int64_t dtw_abandoned;    /* ... of which early-abandoned                         */
    int64_t dtw_cells_nominal;  /* band cells of every evaluated pair                 */
    int64_t dtw_cells_computed; /* cells actually executed (early abandon)            */
    double ms_envelope, ms_keogh, ms_select, ms_improved, ms_dtw, ms_total;
    int64_t kernel_launches;    /* kernels this call launched                         */
    int64_t range1_improved, range1_dtw, range1_cells; /* ... of the above, in the first
                                   (best-first seed) range of candidates               */
    int64_t walk_rounds;        /* DTW walk rounds (plan -> DTW -> merge)              */
    int64_t prefilter_evaluated; /* piecewise-sum bound evaluations (pairs, or 0)      */
    int32_t prefilter_segment;   /* segment length s of the pre-filter (0 = off)       */
    int32_t reserved_;
    double ms_survivor_kernel;   /* device time of the survivor-pass kernels (LB_Keogh /
                                    LB_Improved on sparse pairs), part of ms_improved   */
    double ms_dtw_kernel;        /* device time of the banded-DTW kernel launches of the
                                    walk, part of ms_dtw                                */
    int64_t survivor_entries;    /* (query, 64-candidate tile) entries the survivor kernel walked */
} nn_stats;

/* Exact k-nearest-neighbour search under banded DTW_p: for each query y_q,
 * the k database rows with the smallest (DTW_p(y_q, x_c), c) in lexicographic
 * order (ties to the smaller index), by the paper's cascade (Alg. 3,
 * P:578-620, generalised to p in {1,2}, k >= 1 and many queries): query
 * envelope -> [piecewise-sum bound over the whole database ->]
 * LB_Keogh -> LB_Improved on survivors -> banded DTW on what remains, each gate
 * pruning only when the bound exceeds the current k-th best times (1+eps).
 * Without the pre-filter (DTWLB_NO_PREFILTER) LB_Keogh runs over the whole
 * database, as Alg. 3 is printed.  With few queries (Q <= 8, n % 4 == 0) the bound
 * pass is memory-bound: LB_Keogh then runs as ONE streaming pass over the database
 * for all Q queries (no pre-filter; DTWLB_NO_STREAM disables this mode).  n > 1024:
 * Alg. 2 (LB_Keogh over every pair, then DTW; no LB_Improved pass) -- still exact.
 *   queries: [Q][n] float32, db: [N][n] float32 -- device OR host pointers
 *            (host buffers are staged to the device inside the call);
 *   out_idx: [Q][k] int64 (index_base + row), out_dist: [Q][k] float32 rooted
 *            DTW_p, ascending -- device or host pointers.
 * Errors: EINVAL (n < 1, w < 0, k < 1, Q < 0, N < 1, k > N, N > 2^32 - 1, NULL
 * pointers, an output overlapping an input or the other output), EUNSUPPORTED
 * (p not 1 or 2, k > DTWLB_MAX_K), ENOMEM (also: a query block whose key lists do
 * not fit even as single queries, or with a threshold exchange), ECUDA, ENCCL.
 * Q == 0 is a no-op.  Synchronous with respect to `stream`. */
int nn_search(const float *queries, int64_t Q, const float *db, int64_t N, int32_t n, int32_t w,
              int32_t p, int32_t k, int64_t *out_idx, float *out_dist, const nn_opts *opts,
              nn_stats *stats, void *stream);

/* Merge G per-shard k-NN lists into the global k-NN (sharded search, SURVEY
 * 8(e)): in_idx/in_dist are device [G][Q][k] (shard lists, global indices,
 * padded with (+inf, -1)); out_* device [Q][k].  The k smallest by
 * (dist, idx) of the G*k entries per query.  Stream-ordered. */
int nn_merge(const int64_t *in_idx, const float *in_dist, int32_t G, int64_t Q, int32_t k,
             int64_t *out_idx, float *out_dist, void *stream);

/* Last error message of the calling thread ("" if none). */
const char *dtwlb_last_error(void);

/* Multi-GPU bootstrap of the library's communicator (database-sharded search,
 * one process per GPU).  Rank 0 calls dtwlb_get_unique_id and broadcasts the 128 bytes (e.g.
 * with torch.distributed); every rank then calls dtwlb_comm_init with its rank on its current
 * device and passes the communicator as nn_opts.nccl_comm.  NCCL is loaded at run time
 * (libnccl.so.2).  Errors: EINVAL (NULL pointers, rank outside [0, nranks)), ECUDA (no sm_100
 * device), ENCCL (NCCL not loadable or failing).  dtwlb_comm_destroy(NULL) is a no-op. */
int dtwlb_get_unique_id(void *out128);
int dtwlb_comm_init(const void *id128, int32_t nranks, int32_t rank, void **comm);
int dtwlb_comm_destroy(void *comm);

/* Release the library's cached device workspace (optional). */
void dtwlb_release_workspace(void);

#ifdef __cplusplus
}
#endif

#endif /* DTWLB_H */
