// kernels.cuh -- internal launchers of libdtwlb (not part of the C ABI).
#pragma once

#include <algorithm>
#include <cstdlib>

#include <cuda_fp16.h>

#include "common.cuh"

namespace dtwlb {

// a1: envelope U, L of `count` rows.  Exact.
int launch_envelope(const float *x, int n, int w, float *U, float *L, int64_t count, cudaStream_t st);

// a2: LB_Keogh tile pass.  out[q*ldo + c] = sum_i d(x_c,i, [L_q,i, U_q,i])^p, rooted if `rooted`.
// U, L: [Q][n] with row pitch n; db: [N][n].  Q, N arbitrary.
int launch_keogh(const float *U, const float *L, const float *db, int64_t Q, int64_t N, int n, int p,
                 bool rooted, float *out, int64_t ldo, cudaStream_t st);

// Piecewise-sum pre-filter (section "Using a multidimensional indexing
// structure"): segment sums over C_j = [j*s, min((j+1)*s, n)), s = kSeg, D = ceil(n/s)
// segments padded to Dp = round_up(D, 4) columns.  Outward-rounded (fp64 directed
// sums, then directed conversion), so the fp32 bound is provably <= the exact one.
constexpr int kSeg = 8;
__host__ __device__ inline int paa_dims(int n) { return (n + kSeg - 1) / kSeg; }
__host__ __device__ inline int paa_pitch(int n) { return (paa_dims(n) + 3) / 4 * 4; }
// rows [count][n] -> lo/hi sums [count][Dp] (pad columns 0) (database side)
int launch_paa_sums(const float *x, int64_t count, int n, float *lo, float *hi, cudaStream_t st);
// query envelope U, L [count][n] -> Uhi (sums rounded up, pad +inf), Llo (rounded down, pad -inf)
int launch_paa_env_sums(const float *U, const float *L, int64_t count, int n, float *Uhi, float *Llo,
                        cudaStream_t st);
// beta0[q][c] = sum_j d(X_c,j, [Llo_q,j, Uhi_q,j])^p * (p == 2 ? 1/s : 1), directed rounding
// (a lower bound of LB_Keogh^p, hence of DTW_p^p).  rooted: float out (C-ABI lb_piecewise);
// else __half out rounded down (nn_search's gate block).
int launch_paa_bound(const float *Uhi, const float *Llo, const float *Xlo, const float *Xhi, int64_t Q,
                     int64_t N, int n, int p, bool rooted, void *out, int64_t ldo, cudaStream_t st);
// Midpoint-radius segment sums [count][Dp] (the fused gate's operands, outward-rounded):
// box = false: point sums of the rows lo_src (= hi_src); box = true: the boxes [P(L), P(U)] of
// envelopes lo_src = L, hi_src = U (padding segments: radius FLT_MAX).
int launch_paa_mid(const float *lo_src, const float *hi_src, int64_t count, int n, float *m, float *r, bool box,
                   cudaStream_t st);
// Both terms in one pass: out[q][c] = max(forward, reverse) over midpoint-radius operands
// (launch_paa_mid): Qm/Qr the query envelope boxes, Ym/Yr the query sums [Q][Dp]; Xm/Xr the
// candidate sums, Bm/Br the candidate envelope boxes [N][Dp].  Directed rounding: never above
// the exact max of the two piecewise-sum bounds (readings c18, c20).
int launch_paa_bound_sym(const float *Qm, const float *Qr, const float *Ym, const float *Yr, const float *Xm,
                         const float *Xr, const float *Bm, const float *Br, int64_t Q, int64_t N, int n, int p,
                         bool rooted, void *out, int64_t ldo, cudaStream_t st);

// LB_Keogh^p of Q <= kStreamMaxQ queries against every database row in ONE streaming pass
// (stream.cu; TMA bulk copies, thread per candidate): out[q*ldo + c] = beta1 (rooted if `rooted`).
// Requires n % 4 == 0 and a 16-byte aligned db (keogh_stream_ok).
constexpr int kStreamMaxQ = 8;
bool keogh_stream_ok(int64_t Q, int n, const void *db);
int launch_keogh_stream(const float *U, const float *L, const float *db, int64_t Q, int64_t N, int n, int p,
                        bool rooted, float *out, int64_t ldo, cudaStream_t st);

// Arguments of the survivor passes (improved.cu).  Padded per-query arrays:
//   yq, LUq, ULq: [Q][npadE] (npadE = 32 * epl), zero padded;
//   Uq, Lq: [Q][npadE] query envelope padded with +inf / -inf (phase 1 only).
// Candidate side: Ux, Lx: [N][n] envelopes of the database rows; xdb: the rows.
struct ImprovedArgs {
    const float *yq, *LUq, *ULq;  // [Qb][npadE]
    const float *Uq, *Lq;         // [Qb][npadE] (xdb != NULL)
    const float *Ux, *Lx;         // [N][n]
    const float *xdb;             // [N][n]: if set, beta1 (LB_Keogh^p) is computed in-kernel
                                  // from x (pre-filtered cascade); else read from `gate`
    const void *gate;             // [Qb][ldb] dense gate bound: beta0 = piecewise-sum bound as
                                  // __half (xdb != NULL), or beta1 = LB_Keogh^p as float
    bool gate_half;               // gate element type (__half iff the pre-filter runs)
    __half *gate_w;               // = gate (LIST mode with xdb): slots of the pairs whose beta1
                                  // passed are overwritten with -rd(beta1) (for the DTW walk)
    int64_t ldb;
    int64_t Qb, N;
    int n, npadE;
    const float *lo, *hi;          // per query: gate survivors satisfy lo < gate <= min(hi, thr)
    const float *thr;              // per query: tau^p (1+eps)  (may be NULL = +inf)
    // LIST mode outputs
    unsigned long long *list;      // keys (beta_lb bits << 32 | c): query q's at list[loff[q] ..
                                   // loff[q + 1]) (loff set), else at list[q * cap ..)
    int64_t cap;
    const int64_t *loff;           // [Qb + 1] per-query list offsets (exact-count lists), or NULL
    int *list_len;                 // [Qb]
    // LIST mode with xdb, n <= 256 (reading c22): if set, the key query q appends at position
    // j of its list gets the column part of its DTW abandon schedule at rec[32 (rec_off[q] + j)
    // ..) (32 fp16: the column suffix from 4 rec_c0b rounded down, then 31 sums of 8 columns
    // rounded up; rec_off: per-query offsets of capacity >= the list's); rec_c0b = ceil(w / 4)
    __half *rec;
    const int64_t *rec_off;
    int rec_c0b;
    int *q_count;                 // [Qb] select: gate survivors of the range per query (or NULL)
    // DENSE mode output
    float *dense;                  // [Qb][ldd], rooted
    int64_t ldd;
    unsigned long long *n_eval;        // stats: LB_Improved (phase-2) evaluations (may be NULL)
    unsigned long long *n_eval_keogh;  // stats: in-kernel LB_Keogh evaluations (may be NULL)
    unsigned long long *n_entries;     // stats: (query, 64-candidate tile) entries walked (may be NULL)
    // scratch: per 64-candidate tile, the list of (query, survivor mask) entries
    unsigned long long *tile_m;    // [ceil(N/64)][Qb]
    int *tile_q;                   // [ceil(N/64)][Qb]
    int *tile_cnt;                 // [ceil(N/64)]
    cudaEvent_t ev0, ev1;          // optional: recorded around the survivor kernel (timing)
};
size_t improved_scratch_bytes(int64_t Qb, int64_t N);
void improved_scratch_bind(ImprovedArgs &a, void *p);
int launch_improved(const ImprovedArgs &a, int p, bool keogh_only, bool dense, cudaStream_t st);
// the two halves of launch_improved: the range's (query, survivor mask) tile lists (and the
// per-query survivor counts when a.q_count is set), then the survivor kernel
int launch_select(const ImprovedArgs &a, bool dense, cudaStream_t st);
int launch_survivor(const ImprovedArgs &a, int p, bool keogh_only, bool dense, cudaStream_t st);
int improved_epl(int n);  // elements per lane (4, 8, 16, 32); 0 if n > 1024 (unsupported fast path)
// dense LB_Improved for any n: rooted(beta1 + beta2) per pair, beta1 dense [Q][ldb] (p-th power)
int launch_improved_generic(const float *y, const float *LU, const float *UL, const float *Ux, const float *Lx,
                            const float *beta1, int64_t ldb, int64_t Q, int64_t N, int n, int p, float *out,
                            int64_t ldd, cudaStream_t st);

// Banded DTW (a5).
struct DtwArgs {
    // query side: 4 shifted copies of the +inf-padded query rows, [4][Qy][LP]
    const float *ysh;
    int64_t ysh_stride_s;  // elements between shifted copies
    int LP;                // padded row length
    const float *db;       // candidate rows [*][n]
    int64_t Ndb;           // rows of db (bounds checks of the debug build)
    int n, w;
    // PAIRS mode: item t -> candidate row t, query row t, no pruning
    // WALK mode: item t -> per-query sorted list entry
    const int *item_off;   // [Qb+1] prefix offsets of this round's items per query
    const int *chunk_off;  // [Qb+1] prefix offsets of this round's warp chunks per query
    int64_t nchunks;       // WALK: number of warp chunks (kDtwIpw items of one query each)
    const int *pos;        // [Qb] list position of the query's first item this round
    const unsigned long long *list;  // query q's keys at list[loff[q] ..) (loff set) or list[q * cap ..)
    int64_t cap;
    const int64_t *loff;
    int Qb;
    float *thr;            // [Qb] tau^p (1+eps); WALK: lowered by walk_result as the top-k fills
    int64_t total;         // number of items (WALK with dev_total: an upper bound, see below)
    const int *dev_total;  // WALK, w <= 32 kernel: if set, the round's item count is read here
                           // (written by the plan kernel: no host round trip per walk round)
    float *res;            // [total] DTW^p, +inf if pruned/abandoned (PAIRS: rooted)
    unsigned long long *cells;  // stats: computed cells (may be NULL)
    unsigned long long *abandoned;  // stats (may be NULL)
    unsigned long long *started;    // stats: pairs whose DTW started (may be NULL)
    unsigned *queue;                 // work-queue counter (scratch, 4 bytes) for the w <= 32 kernel
    // WALK, cascading abandon (b1 and b1h NULL = off): |b1[q*ldb + c]| (float) or |b1h[...]|
    // (__half, rounded down) = LB_Keogh^p of the pair, Uq/Lq [Qb][n] the query envelopes;
    // abandon once rowmin + (terms of rows left) > thr
    const float *b1;
    const __half *b1h;
    int64_t ldb;
    const float *Uq, *Lq;
    // row+column cascade (reading c21; dtw4_kernel, col_c0 > 0, with b1h): besides the rows'
    // LB_Keogh terms, rest holds the LB_Improved column terms beta2_j of the columns the
    // remaining rows must still visit; their total is key - next_up(|b1h|) (a lower bound of
    // beta2), the columns [0, C(i)), C(i) = min(n, i + col_c0), col_c0 = round_up(w, 4),
    // are subtracted (up to 16 per 8-row step; the column part joins the abandon test once
    // caught up).  yq, LUq, ULq: [Qb][n] y, U(L(y)), L(U(y)); Uxdb, Lxdb: [N][n] U(x), L(x).
    int col_c0;
    const float *yq, *LUq, *ULq, *Uxdb, *Lxdb;
    // WALK, dtw4_kernel with the row cascade (b1h), n % 4 == 0 (reading c22): if set, the
    // column schedules the survivor kernel wrote (ImprovedArgs::rec / rec_off); the key at
    // sorted list position j of query q was appended at position (j & ~kKeyPosMask) +
    // key_pos(key) (runs of 2^kKeyPosBits keys are sorted in place).  Exclusive with col_c0
    const __half *rec;
    const int64_t *rec_off;
    // WALK: no early abandon (nn_opts DTWLB_NO_ABANDON): every started pair runs to its last row
    bool no_abandon;
    // WALK: completed pairs are merged into the query's top-k (keys (DTW^p bits << 32 | c),
    // ascending, [Qb][k]) under a per-query lock, and thr[q] follows the k-th key
    unsigned long long *topk;
    int *topk_lock;
    int k;
    float eps;
    // WALK: completed pairs of the round (appended by the DTW kernels, merged by launch_topk_merge)
    unsigned long long *rkey;   // [rcap] (DTW^p bits << 32 | c)
    int *rq;                    // [rcap] query
    unsigned *rcount;           // appended so far (reset before each round)
    int64_t rcap;
};
int launch_topk_merge(const DtwArgs &a, cudaStream_t st);
constexpr int kYPadL = 64;
constexpr int kDtwIpw = 64;  // items per warp chunk of the DTW walk  // left padding of query rows (>= largest register band)
int dtw_padded_len(int n);
int launch_dtw(const DtwArgs &a, int p, bool walk, cudaStream_t st);
// w > 64: does the generic kernel need a global band scratch of (2w+2) floats per item?
bool dtw_generic_needs_scratch(int w);
// Wide bands (dtw_wide.cu, four lanes per pair): dtw_wide_plan returns 1 (column coordinates,
// w >= n-1, n <= 256), 2 (band coordinates, instantiated S) or 0 (no wide kernel: generic);
// the query rows are padded to LPW = dtw_wide_padded(n, w, S, &padL) floats (+inf outside).
int dtw_wide_plan(int n, int w, int *S);
int dtw_wide_padded(int n, int w, int S, int *padL);
int launch_build_ywide(const float *y, int64_t rows, int n, float *yp, int LPW, int padL, cudaStream_t st);
int launch_dtw_wide(const DtwArgs &a, const float *yp, int LPW, int padL, int p, bool walk, cudaStream_t st);
// Build the 4 shifted, +inf-padded copies of `rows` query rows.
int launch_build_ysh(const float *y, int64_t rows, int n, float *ysh, int LP, cudaStream_t st);

}  // namespace dtwlb
