// kernels.cuh -- internal launchers of libdtwlb (not part of the C ABI).
#pragma once

#include <algorithm>

#include "common.cuh"

namespace dtwlb {

// a1: envelope U, L of `count` rows.  Exact.
int launch_envelope(const float *x, int n, int w, float *U, float *L, int64_t count, cudaStream_t st);

// a2: LB_Keogh tile pass.  out[q*ldo + c] = sum_i d(x_c,i, [L_q,i, U_q,i])^p, rooted if `rooted`.
// U, L: [Q][n] with row pitch n; db: [N][n].  Q, N arbitrary.
int launch_keogh(const float *U, const float *L, const float *db, int64_t Q, int64_t N, int n, int p,
                 bool rooted, float *out, int64_t ldo, cudaStream_t st);

// Padded per-query arrays used by the LB_Improved survivor kernel:
//   yq, LUq, ULq: [Q][npadE] (npadE = 32 * epl), zero padded.
// Candidate envelopes of the database: Ux, Lx: [N][n].
struct ImprovedArgs {
    const float *yq, *LUq, *ULq;  // [Qb][npadE]
    const float *Ux, *Lx;         // [N][n]
    const float *beta1;           // [Qb][ldb] LB_Keogh^p
    int64_t ldb;
    int64_t Qb, N;
    int n, npadE;
    const float *lo, *hi;          // per query: survivors satisfy lo < beta1 <= min(hi, thr)
    const float *thr;              // per query: tau^p (1+eps)  (may be NULL = +inf)
    // LIST mode outputs
    unsigned long long *list;      // [Qb][cap] keys (beta_lb bits << 32 | c)
    int64_t cap;
    int *list_len;                 // [Qb]
    // DENSE mode output
    float *dense;                  // [Qb][ldd], rooted
    int64_t ldd;
    unsigned long long *n_eval;    // stats: survivors evaluated (may be NULL)
    // scratch: per 64-candidate tile, the list of (query, survivor mask) entries
    unsigned long long *tile_m;    // [ceil(N/64)][Qb]
    int *tile_q;                   // [ceil(N/64)][Qb]
    int *tile_cnt;                 // [ceil(N/64)]
};
size_t improved_scratch_bytes(int64_t Qb, int64_t N);
void improved_scratch_bind(ImprovedArgs &a, void *p);
int launch_improved(const ImprovedArgs &a, int p, bool keogh_only, bool dense, cudaStream_t st);
int improved_epl(int n);  // elements per lane (4, 8, 16, 32); 0 if n > 1024 (unsupported fast path)

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
    const unsigned long long *list;  // [Qb][cap]
    int64_t cap;
    int Qb;
    const float *thr;      // [Qb] tau^p (1+eps)
    int64_t total;         // number of items
    float *res;            // [total] DTW^p, +inf if pruned/abandoned (PAIRS: rooted)
    unsigned long long *cells;  // stats: computed cells (may be NULL)
    unsigned long long *abandoned;  // stats (may be NULL)
    unsigned long long *started;    // stats: pairs whose DTW started (may be NULL)
    unsigned *queue;                 // work-queue counter (scratch, 4 bytes) for the w <= 32 kernel
};
constexpr int kYPadL = 64;
constexpr int kDtwIpw = 64;  // items per warp chunk of the DTW walk  // left padding of query rows (>= largest register band)
int dtw_padded_len(int n);
int launch_dtw(const DtwArgs &a, int p, bool walk, cudaStream_t st);
// Build the 4 shifted, +inf-padded copies of `rows` query rows.
int launch_build_ysh(const float *y, int64_t rows, int n, float *ysh, int LP, cudaStream_t st);

}  // namespace dtwlb
