// dtw.cu -- banded DTW_p (a5): the recursion of P:199-210 (section "Dynamic Time
// Warping") evaluated in its forward (prefix) form, which equals the suffix form
// by reversing both series:
//
//   D(i,j) = |x_i - y_j|^p + min(D(i-1,j), D(i,j-1), D(i-1,j-1)),  |i-j| <= w,
//   D(-1,-1) = 0, everything else outside the band = +inf;  DTW_p^p = D(n-1,n-1).
//
// B200 design (w <= 64, dtw4_kernel): thread-per-pair with the 2w+1-wide band held
// in REGISTERS (template WB >= w, exact instantiations for the configs' w), so each
// cell is the minimal 3-op SASS sequence FADD (x-y), FMNMX3, FADD|abs| / FFMA.  Four
// rows are advanced per pass, skewed by two cells, so every step holds four
// independent dependency chains; the query window lives in registers (w <= 32) or
// is read from shared memory / L1 (32 < w <= 64).  Early abandoning (not in the
// paper, readings c15, c19): every path crosses every row and costs are
// >= 0, so once a row's minimum plus the LB_Keogh terms of the rows not yet computed
// exceeds tau^p(1+eps) the pair cannot enter the top-k.  Lanes are desynchronised
// and refilled from a work queue through a cp.async pipeline, so one long pair does
// not idle the other 31 lanes.  w > 64: dtw_generic_kernel (one thread per pair,
// band in shared memory).
#include "kernels.cuh"

namespace dtwlb {

int dtw_padded_len(int n) { return ((n + kYPadL + 2 * 64 + 8) + 3) & ~3; }

namespace {

constexpr int NT = 128;

template <int P>
__device__ __forceinline__ float cell(float m, float t) {
    if constexpr (P == 1) return m + fabsf(t);
    else if constexpr (P == 0) return fmaxf(m, fabsf(t));  // DTW_inf: max, exact
    else if constexpr (P == 4) { const float t2 = t * t; return fmaf(t2, t2, m); }  // DTW_4
    else return fmaf(t, t, m);
}

// In-band cells of rows 0 .. r-1 of the n x n table: sum_i (min(n-1, i+w) - max(0, i-w) + 1)
// = r(2w+1) - (left clip) - (right clip); band_cells(n, n, w) = n(2w+1) - w(w+1).  (w <= n-1)
__device__ __forceinline__ unsigned long long band_cells(int r, int n, int w) {
    const long long m = r < w ? r : w;                        // rows i < w lose w - i cells
    const long long a = n - w;                                 // rows i >= n - w lose i + w - n + 1
    const long long t = r > a ? r - a : 0;
    return (unsigned long long)((long long)r * (2 * w + 1) - (m * w - m * (m - 1) / 2) - t * (t + 1) / 2);
}

template <int P>
__device__ __forceinline__ float col_lb(float y, float ux, float lx, float lu, float ul) {
    // LB_Improved column term d(y_j, [L(H)_j, U(H)_j])^p by the closed form (improved.cu)
    const float d = max3f(y - fmaxf(ux, lu), fminf(lx, ul) - y, 0.f);
    return P == 1 ? d : d * d;
}

// LB_Keogh term of row i: d(x_i, [L(y)_i, U(y)_i])^p.  Every banded path visits row i in some
// column j with |i-j| <= w, at cost |x_i - y_j|^p >= this term, so the sum of the terms of the
// rows not yet computed bounds what the path still has to pay (cascading abandon, DESIGN.md
// reading c19); the pair's total (+-beta1) comes from the gate slot the survivor kernel wrote.
template <int P>
__device__ __forceinline__ float row_lb(float x, float u, float l) {
    const float d = max3f(x - u, l - x, 0.f);
    return P == 1 ? d : d * d;
}

// cp.async of r[i0 .. i0+7] (zero beyond n) into dst[0..8) (16-byte copies when aligned)
__device__ __forceinline__ void stage_rows8(float *dst, const float *r, int i0, int n) {
    if (((n & 3) == 0)) {
        const bool ok0 = i0 + 4 <= n, ok1 = i0 + 8 <= n;
        cp_async16(dst, ok0 ? r + i0 : r, ok0 ? 16 : 0);
        cp_async16(dst + 4, ok1 ? r + i0 + 4 : r, ok1 ? 16 : 0);
    } else {
#pragma unroll
        for (int t = 0; t < 8; ++t) cp_async4(dst + t, i0 + t < n ? r + i0 + t : r, i0 + t < n ? 4 : 0);
    }
}

template <int WB>
__device__ __forceinline__ float band_min(const float (&B)[2 * WB + 2]) {
    float m = B[0];
#pragma unroll
    for (int d = 1; d + 1 < 2 * WB + 1; d += 2) m = min3f(m, B[d], B[d + 1]);
    if ((2 * WB + 1) % 2 == 0) m = fminf(m, B[2 * WB]);
    return m;
}

// Merge a completed pair (key = DTW^p bits << 32 | c) into query q's top-k -- the k
// smallest keys (float bits of r << 32 | c), ascending (reading c4: ties to the smaller
// index) -- and lower thr[q] to (k-th distance)(1+eps) once k results exist.  Taken under
// the query's lock; keys and thr are read/written through L2 (volatile), so every other
// warp's next refill or abandon test sees the tightened threshold.  Independent-thread-
// scheduling safe: the lane that wins the lock does the work inside the same iteration.
__device__ __forceinline__ void walk_result(const DtwArgs &a, int64_t q, unsigned long long key) {
    volatile float *thr = a.thr + q;
    if (!(__uint_as_float((uint32_t)(key >> 32)) <= *thr)) return;  // cannot enter the top-k
    volatile unsigned long long *tk = a.topk + q * a.k;
    int *lock = a.topk_lock + q;
    bool done = false;
    while (!done) {
        // re-test against the threshold while waiting: in a walk's first round (tau = +inf) a
        // query's ~128 completed pairs contend for its lock, and once k of them are in, most
        // of the rest can no longer enter -- they leave without taking the lock
        if (!(__uint_as_float((uint32_t)(key >> 32)) <= *thr)) return;
        if (atomicCAS(lock, 0, 1) == 0) {
            __threadfence();
            if (key < tk[a.k - 1]) {
                int j = a.k - 1;
                while (j > 0 && tk[j - 1] > key) {
                    tk[j] = tk[j - 1];
                    --j;
                }
                tk[j] = key;
                const unsigned long long kth = tk[a.k - 1];
                // thresholds only decrease (a shard exchange may have lowered thr below
                // this shard's own k-th best)
                if (kth != ~0ull) *thr = fminf(*thr, __uint_as_float((uint32_t)(kth >> 32)) * (1.0f + a.eps));
            }
            __threadfence();
            atomicExch(lock, 0);
            done = true;
        }
    }
}

// WALK: the lanes with has_res append their completed pair (query q, key (DTW^p, c)) to
// the round's result buffer (one warp-aggregated atomic); topk_merge_kernel merges the
// buffer into the top-k after the launch, so the DTW kernels carry no lock/insert code.
__device__ __forceinline__ void walk_results_warp(const DtwArgs &a, bool has_res, int q, uint32_t c, float r,
                                                  int lane) {
    const unsigned m = __ballot_sync(0xffffffffu, has_res);
    if (!m) return;
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(a.rcount, (unsigned)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (has_res) {
        const unsigned pos = base + __popc(m & ((1u << lane) - 1u));
        DCHECK(pos < a.rcap, "result buffer overflow pos=%u cap=%lld", pos, (long long)a.rcap);
        a.rkey[pos] = pack_key(r, c);
        a.rq[pos] = q;
    }
}

// After a walk round: merge the round's completed pairs (few: most pairs are abandoned)
// into the per-query top-k (grid-stride, one result per thread).
__global__ void __launch_bounds__(256) topk_merge_kernel(DtwArgs a) {
    const unsigned cnt = *a.rcount;
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x)
        walk_result(a, a.rq[t], a.rkey[t]);
}

// ---------------------------------------------------------------------------
// dtw4_kernel (w <= 32): four rows per pass and the y window in REGISTERS.
// Row r of the block (r = 0..3) computes its cell d-r at step d, so all four rows
// use the same y value y[i + d - w] at step d and form four independent dependency
// chains (ILP 4).  The window Y[0..2WB+3] = y[i-w .. i+w+3] shifts by four per
// block (one aligned 16-byte load of the next four values from the pre-shifted
// copy whose alignment matches (i - w) mod 4, fixed per item), so the cell loop
// touches no memory at all and lanes may work on pairs of different queries.
// Work distribution: a global queue of 256-item chunks of the flattened round
// (items of consecutive queries); lanes refill one item at a time from the warp's
// chunk, so a few long (non-abandoned) pairs do not idle the rest of the warp.
constexpr int kChunk4 = 256;

template <int WB, int P, bool EXACT>
__device__ __forceinline__ void four_rows(float (&B)[2 * WB + 2], const float2 (&Y2)[(2 * WB + 4 + 3) / 4 * 2],
                                          const float (&x)[4], int w2) {
    constexpr int NB = 2 * WB + 1;
    // skew 2: at step d, row r computes band cell e = d - 2r.  Its up (row r-1, cell e+1)
    // and diagonal (row r-1, cell e) neighbours came out of row r-1 one and two steps
    // earlier (h1, h2), its left neighbour is its own previous cell (pl); y index e + r = d - r.
    // The four rows of a step read the consecutive y[d - 3 .. d]; on odd steps (y[d-1], y[d]) and
    // (y[d-3], y[d-2]) are register pairs of the window Y2[k] = (Y[2k], Y[2k+1]), so the differences
    // of rows (1, 0) and (3, 2) issue as two packed FADD2 against the x pairs (x0, x1), (x2, x3)
    // read swapped (same IEEE operation per component); even steps stay scalar (their pairs
    // would need a misaligned (x2, x1)): 3 instead of 4 issue slots per four differences.
    const float2 x01 = make_float2(x[0], x[1]), x23 = make_float2(x[2], x[3]);
    float pl0 = kInf, pl1 = kInf, pl2 = kInf, pl3 = kInf;
    float h1_0 = kInf, h2_0 = kInf, h1_1 = kInf, h2_1 = kInf, h1_2 = kInf, h2_2 = kInf;
#pragma unroll
    for (int d = 0; d < NB + 6; ++d) {
        const bool a0 = d < NB, a1 = d >= 2 && d - 2 < NB, a2 = d >= 4 && d - 4 < NB, a3 = d >= 6;
        float t0 = 0.f, t1 = 0.f, t2 = 0.f, t3 = 0.f;
        if (d & 1) {
            if (a0 || a1) {  // (x0 - y[d], x1 - y[d-1])
                const float2 v = Y2[(d - 1) / 2];
                const float2 r = __fadd2_rn(x01, make_float2(-v.y, -v.x));
                t0 = r.x; t1 = r.y;
            }
            if ((a2 || a3) && d >= 3) {  // (x2 - y[d-2], x3 - y[d-3])
                const float2 v = Y2[(d - 3) / 2];
                const float2 r = __fadd2_rn(x23, make_float2(-v.y, -v.x));
                t2 = r.x; t3 = r.y;
            }
        } else {
            if (a0) t0 = x[0] - Y2[d / 2].x;
            if (a1) t1 = x[1] - Y2[(d - 2) / 2].y;
            if (a2) t2 = x[2] - Y2[(d - 2) / 2].x;
            if (a3) t3 = x[3] - Y2[(d - 4) / 2].y;
        }
        float c0 = kInf, c1 = kInf, c2 = kInf;
        if (a0) {  // row 0, cell d: up = B[d+1], diag = B[d]
            c0 = cell<P>(min3f(B[d], B[d + 1], pl0), t0);
            if (!EXACT && d > w2) c0 = kInf;
            pl0 = c0;
        }
        if (a1) {  // row 1, cell d-2
            c1 = cell<P>(min3f(h2_0, h1_0, pl1), t1);
            if (!EXACT && d - 2 > w2) c1 = kInf;
            pl1 = c1;
        }
        if (a2) {  // row 2, cell d-4
            c2 = cell<P>(min3f(h2_1, h1_1, pl2), t2);
            if (!EXACT && d - 4 > w2) c2 = kInf;
            pl2 = c2;
        }
        if (a3) {  // row 3, cell d-6 (stored: B becomes row i+3)
            float c3 = cell<P>(min3f(h2_2, h1_2, pl3), t3);
            if (!EXACT && d - 6 > w2) c3 = kInf;
            pl3 = c3;
            B[d - 6] = c3;
        }
        h2_0 = h1_0; h1_0 = c0;
        h2_1 = h1_1; h1_1 = c1;
        h2_2 = h1_2; h1_2 = c2;
    }
}

// four_rows with the y window read from global memory (L1: the lanes of a warp mostly walk
// the same query) instead of registers: frees 2w+4 registers (w up to 64 fits; more warps
// per SM) and removes the per-block window shift; yb[k] = y[i - w + k] (+inf padded).
template <int WB, int P, bool EXACT>
__device__ __forceinline__ void four_rows_g(float (&B)[2 * WB + 2], const float *yb,
                                            const float (&x)[4], int w2) {
    constexpr int NB = 2 * WB + 1;
    float yy[NB + 3];
    float pl0 = kInf, pl1 = kInf, pl2 = kInf, pl3 = kInf;
    float h1_0 = kInf, h2_0 = kInf, h1_1 = kInf, h2_1 = kInf, h1_2 = kInf, h2_2 = kInf;
#pragma unroll
    for (int d = 0; d < NB + 6; ++d) {
        if (d < NB + 3) yy[d] = yb[d];  // (generic load: shared or global)
        float c0 = kInf, c1 = kInf, c2 = kInf;
        if (d < NB) {
            c0 = cell<P>(min3f(B[d], B[d + 1], pl0), x[0] - yy[d]);
            if (!EXACT && d > w2) c0 = kInf;
            pl0 = c0;
        }
        if (d >= 2 && d - 2 < NB) {
            c1 = cell<P>(min3f(h2_0, h1_0, pl1), x[1] - yy[d - 1]);
            if (!EXACT && d - 2 > w2) c1 = kInf;
            pl1 = c1;
        }
        if (d >= 4 && d - 4 < NB) {
            c2 = cell<P>(min3f(h2_1, h1_1, pl2), x[2] - yy[d - 2]);
            if (!EXACT && d - 4 > w2) c2 = kInf;
            pl2 = c2;
        }
        if (d >= 6) {
            float c3 = cell<P>(min3f(h2_2, h1_2, pl3), x[3] - yy[d - 3]);
            if (!EXACT && d - 6 > w2) c3 = kInf;
            pl3 = c3;
            B[d - 6] = c3;
        }
        h2_0 = h1_0; h1_0 = c0;
        h2_1 = h1_1; h1_1 = c1;
        h2_2 = h1_2; h1_2 = c2;
    }
}

// Per-lane staging slot of the pipelined refill: the y window (NY floats), x[0..7] and
// the query envelope U[0..3], L[0..3] of the lane's next pair, written by cp.async while
// the lane still waits one step; +4 floats of padding rotate the banks between lanes.
template <int WB, bool YG = false>
struct Dtw4Cfg {
    static constexpr int NY = YG ? 0 : (2 * WB + 4 + 3) / 4 * 4;  // (YG: no y window in the slot)
    // [0, NY) the y window and [NY] the gate word (refill, read at activation); while the lane
    // is active [0, 40) stages the row+column cascade's column data (reading c21);
    // [XA, XA + 8) x and [XA + 8, XA + 24) U(y), L(y) of the next step's 8 rows (written by
    // the refill for rows 0..7, then one step ahead); [SL - 2, SL) the pair's (q, c)
    static constexpr int XA = NY + 4 > 40 ? NY + 4 : 40;  // (YG: the gate word sits at [0])
    static constexpr int SL = XA + 28;
    // per warp chunk: keys, schedule indices (reading c22), queries
    static constexpr size_t smem = (size_t)NT * SL * sizeof(float) +
                                   (size_t)(NT / 32) * kChunk4 * (2 * sizeof(unsigned long long) + sizeof(int));
};

// Lane states of dtw4_kernel
constexpr int kFree = 0, kPending = 1, kActive = 2;

template <int WB, bool YG>
constexpr int dtw4_min_blocks() { return YG ? (WB <= 32 ? 4 : 3) : (WB <= 25 ? 3 : 2); }

template <int WB, int P, bool EXACT, bool WALK, bool YG>
__global__ void __launch_bounds__(NT, (dtw4_min_blocks<WB, YG>()))
dtw4_kernel(DtwArgs a) {
    constexpr int NB = 2 * WB + 1;
    constexpr int NY = Dtw4Cfg<WB, YG>::NY;  // window length, a multiple of 4 (aligned refills)
    constexpr int SL = Dtw4Cfg<WB, YG>::SL;
    constexpr int XA = Dtw4Cfg<WB, YG>::XA;
    extern __shared__ __align__(16) float dsm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float *slot = dsm + (size_t)threadIdx.x * SL;  // this lane's staging slot
    unsigned long long *ckey = reinterpret_cast<unsigned long long *>(dsm + (size_t)NT * SL) + wid * kChunk4;
    long long *crec = reinterpret_cast<long long *>(dsm + (size_t)NT * SL) + (NT / 32) * kChunk4 + wid * kChunk4;
    int *cq = reinterpret_cast<int *>(reinterpret_cast<unsigned long long *>(dsm + (size_t)NT * SL) +
                                      2 * (NT / 32) * kChunk4) + wid * kChunk4;
    const int n = a.n, w = EXACT ? WB : a.w, w2 = 2 * w;
    const int sh = (kYPadL - w) & 3;  // alignment class of (i - w) for i % 4 == 0
    // YG, WALK: the padded row of the query of the warp's current chunk staged in shared
    // memory (lanes on that query read their y values there, others from global/L1)
    float *wrow = reinterpret_cast<float *>(reinterpret_cast<int *>(reinterpret_cast<unsigned long long *>(
                      dsm + (size_t)NT * SL) + 2 * (NT / 32) * kChunk4) + (NT / 32) * kChunk4) + (size_t)wid * a.LP;
    int staged_q = -1;
    bool ysm = false;           // this lane's y row is the staged one
    const float *ybase = nullptr;  // YG: start of this lane's padded y row (shared or global)
    const int64_t total = (WALK && a.dev_total) ? (int64_t)*a.dev_total : a.total;
    // chunk size: kChunk4 items per warp grab, smaller (down to 32) when the round is too
    // small to give every resident warp a few chunks (few long pairs: C3, C4)
    const int64_t nwarps = (int64_t)gridDim.x * (NT / 32);
    const int64_t chunk_w = (total / (4 * nwarps) + 31) / 32 * 32;
    const int chunk = (int)(chunk_w > kChunk4 ? kChunk4 : (chunk_w < 32 ? 32 : chunk_w));
    const int64_t nchunks = (total + chunk - 1) / chunk;
    if (total == 0) return;
    const unsigned lt = (1u << lane) - 1u;

    int cbeg = 0, cend = 0, cursor = 0;  // item indices (< 2^31: one walk round)
    int st = kFree;
    int item = 0;
    const float *xr = nullptr, *yr = nullptr;
    float thr = kInf, beta_n = 0.f;
    int i = 0;
    float B[NB + 1];
    float2 Y2[YG ? 1 : NY / 2];  // the y window as register pairs: Y2[k] = (Y[2k], Y[2k+1])
    float xv[8];  // x of rows i .. i+7 (staged in the slot one 8-row step ahead)
    // cascading abandon: rest = LB_Keogh^p terms of the rows not yet computed
    const bool casc = WALK && (a.b1 != nullptr || a.b1h != nullptr);
    // column schedule (reading c22, with the row cascade): the pair's 32 fp16 words written by
    // the survivor kernel, copied into the slot's [0, 16) (the y window / gate word, free once
    // the lane is active) at activation: word 0 joins rest at the first test, word k is
    // subtracted at the test after 8k rows
    const bool recm = casc && a.rec != nullptr;
    // row+column cascade (reading c21): the gate word holds rest0 = LB_Improved^p minus the
    // column terms of [0, col_c0) (rest0_kernel); each step subtracts its rows' LB_Keogh terms
    // and the column terms of [C(i0), C(i0 + 8)), C(i) = i + col_c0
    // (col_c0 > 0 requires n % 4 == 0 and the __half gate block)
    const bool casc2 = casc && a.col_c0 > 0 && a.b1h != nullptr;
    float rest = 0.f, rest_n = 0.f;
    const float *ur = nullptr, *lr = nullptr;
    unsigned long long cells_done = 0;  // in-band cells of this lane's finished / abandoned pairs
    unsigned n_abandon = 0, n_started = 0;  // per-lane counters

    while (true) {
        // ---- (a) activate the lanes whose refill copies were issued one step ago ----
        if (__any_sync(0xffffffffu, st == kPending)) {
            cp_wait<0>();
            if (st == kPending) {
                const float thr_n = slot[NY + 1];
                if (beta_n > thr_n) {
                    if constexpr (!WALK) a.res[item] = kInf;  // (WALK: pruned by its bound)
                    st = kFree;
                } else {
                    if constexpr (!YG) {
#pragma unroll
                        for (int d = 0; d < NY; d += 4) {
                            const float4 v = *reinterpret_cast<const float4 *>(slot + d);
                            Y2[d / 2] = make_float2(v.x, v.y);
                            Y2[d / 2 + 1] = make_float2(v.z, v.w);
                        }
                    }
                    const float4 x0 = *reinterpret_cast<const float4 *>(slot + XA);
                    const float4 x1 = *reinterpret_cast<const float4 *>(slot + XA + 4);
                    xv[0] = x0.x; xv[1] = x0.y; xv[2] = x0.z; xv[3] = x0.w;
                    xv[4] = x1.x; xv[5] = x1.y; xv[6] = x1.z; xv[7] = x1.w;
                    thr = thr_n;
                    if (casc) {
                        // the pair's gate word, copied with the refill (no register wait on a
                        // random HBM gather): +-beta1 / rest0, fp32 or the __half at c & 1
                        const uint32_t wv = reinterpret_cast<const uint32_t *>(slot)[NY];
                        const uint32_t c = reinterpret_cast<const uint32_t *>(slot)[SL - 1];
                        const unsigned short hb = (unsigned short)((c & 1u) ? wv >> 16 : wv & 0xffffu);
                        rest_n = a.b1 ? __uint_as_float(wv) : __half2float(__ushort_as_half(hb));
                    }
                    rest = fabsf(rest_n);
                    if (recm) {
                        const __half *rp = a.rec + crec[item - cbeg] * 32;
#pragma unroll
                        for (int m = 0; m < 4; ++m) cp_async16(slot + 4 * m, rp + 8 * m, 16);
                    }
                    st = kActive;
                    ++n_started;
                }
            }
        }
        // ---- (b) refill free lanes: claim the next items of the warp's chunk and issue
        //      their copies (y window, x[0..7]) into the lane's slot; active next step ----
        const unsigned need = __ballot_sync(0xffffffffu, st == kFree);
        if (need && cursor >= cend) {  // the warp's chunk is exhausted: grab the next one
            int64_t c = 0;
            if (lane == 0) c = atomicAdd(a.queue, 1u);
            c = __shfl_sync(0xffffffffu, c, 0);
            if (c < nchunks) {
                cbeg = (int)c * chunk;
                cend = (int)(cbeg + chunk < total ? cbeg + chunk : total);
                cursor = cbeg;
                if constexpr (WALK) {
                    // stage the chunk's keys and queries: items are in query order, each
                    // lane walks its 8 items (cbeg + lane + 32 t) forward from the chunk's first query
                    int lo = 0, hi = a.Qb;  // item_off[lo] <= cbeg < item_off[hi]
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if (a.item_off[mid] <= cbeg) lo = mid; else hi = mid;
                    }
                    if constexpr (YG) {
                        if (lo != staged_q) {  // restage: lanes still on the old row read it from global
                            if (ysm) { ybase = a.ysh + (int64_t)reinterpret_cast<const int *>(slot)[SL - 2] * a.LP; ysm = false; }
                            __syncwarp();
                            const float *src = a.ysh + (int64_t)lo * a.LP;
                            for (int u = lane; u < a.LP; u += 32) wrow[u] = __ldg(src + u);
                            staged_q = lo;
                        }
                    }
                    int q = lo;
                    for (int t = 0; t < chunk / 32; ++t) {
                        const int it = cbeg + lane + 32 * t;
                        if (it < cend) {
                            while (it >= a.item_off[q + 1]) ++q;
                            const int64_t j = a.pos[q] + (it - a.item_off[q]);
                            DCHECK(j >= 0 && (a.loff ? a.loff[q] + j < a.loff[q + 1] : j < a.cap), "dtw4 item %lld q=%d j=%lld",
                                   (long long)it, q, (long long)j);
                            const int64_t lb = list_base(a.loff, a.cap, q);
                            const unsigned long long key = a.list[lb + j];
                            ckey[lane + 32 * t] = key;
                            if (recm) crec[lane + 32 * t] = __ldg(a.rec_off + q) + (j & ~(int64_t)kKeyPosMask) + key_pos(key);
                            cq[lane + 32 * t] = q;
                        }
                    }
                }
                __syncwarp();
            }
        }
        if (need && cursor < cend) {
            const int mine = cursor + __popc(need & lt);
            cursor += __popc(need);
            if (st == kFree && mine < cend) {
                item = mine;
                int64_t c, qy;
                if constexpr (WALK) {
                    const unsigned long long key = ckey[item - cbeg];
                    qy = cq[item - cbeg];
                    c = (int64_t)(key & 0xffffffffu);
                    // the pair's (query, candidate), read back at completion (smem: no registers)
                    reinterpret_cast<int *>(slot)[SL - 2] = (int)qy;
                    reinterpret_cast<uint32_t *>(slot)[SL - 1] = (uint32_t)c;
                    DCHECK(c < a.Ndb, "dtw4 key c=%lld q=%lld", (long long)c, (long long)qy);
                    beta_n = key_bound(key);
                    // tau of the pair's query: copied into the slot's padding word [NY + 1] with the
                    // refill (as a register load its address pair was overwritten right after it, and
                    // that IMAD held 6.4 % of the stall samples waiting on the load's operand read,
                    // `profiles/r02zl_C5_dtw4_kernel_10_sass_top.txt`; in the walk tau changes only
                    // between launches, and a stale tau is larger, never wrong)
                    cp_async4(slot + NY + 1, a.thr + qy, 4);
                    if (casc) {
                        // +-beta1: the 4-byte word holding it -> slot[NY]
                        const int64_t gi = qy * a.ldb + c;
                        if (a.b1) cp_async4(slot + NY, a.b1 + gi, 4);
                        else cp_async4(slot + NY, reinterpret_cast<const float *>(a.b1h + (gi & ~(int64_t)1)), 4);
                        ur = a.Uq + qy * n;
                        lr = a.Lq + qy * n;
                    }
                } else {
                    c = qy = item;
                    beta_n = 0.f;
                    slot[NY + 1] = kInf;
                }
                xr = a.db + c * n;
                yr = a.ysh + (int64_t)sh * a.ysh_stride_s + qy * a.LP;
                if constexpr (YG) {
                    ysm = WALK && qy == staged_q;
                    ybase = ysm ? wrow : a.ysh + qy * a.LP;  // (shift-0 copy: no alignment needed)
                }
                // Y[d] = ypad[-w + kYPadL + d]; the copy `sh` makes base (kYPadL - w - sh) aligned
                const float *ys = yr + (kYPadL - w - sh);
                if constexpr (!YG) {
#pragma unroll
                    for (int d = 0; d < NY; d += 4) cp_async16(slot + d, ys + d, 16);
                }
                stage_rows8(slot + XA, xr, 0, n);
                if (casc) {
                    stage_rows8(slot + XA + 8, ur, 0, n);
                    stage_rows8(slot + XA + 16, lr, 0, n);
                }
                cp_commit();
#pragma unroll
                for (int d = 0; d <= NB; ++d) B[d] = kInf;
#pragma unroll
                for (int d = 0; d < NB; ++d)
                    if (d == w) B[d] = 0.f;  // virtual D(-1,-1) = 0 sits on the diagonal
                i = 0;
                st = kPending;
            }
        }
        if (!__any_sync(0xffffffffu, st != kFree)) {
            // no lane has work: done when the queue is exhausted
            bool more = cursor < cend;
            if (!more) {
                int64_t peek = 0;
                if (lane == 0) peek = *reinterpret_cast<volatile unsigned *>(a.queue);
                peek = __shfl_sync(0xffffffffu, peek, 0);
                more = peek < nchunks;
            }
            if (!more) break;
            continue;
        }
        // ---- (c) advance the active lanes by up to 8 rows ----
        bool has_res = false;
        float res_v = 0.f;
        if (st == kActive) {
            const int i0 = i;
            if (casc) {
                // LB_Keogh terms of this step's rows (their envelope was staged one step ahead)
                const float4 u0 = *reinterpret_cast<const float4 *>(slot + XA + 8);
                const float4 u1 = *reinterpret_cast<const float4 *>(slot + XA + 12);
                const float4 l0 = *reinterpret_cast<const float4 *>(slot + XA + 16);
                const float4 l1 = *reinterpret_cast<const float4 *>(slot + XA + 20);
                const float uu[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
                const float ll[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
                float rs = 0.f;
#pragma unroll
                for (int t = 0; t < 8; ++t) rs += i0 + t < n ? row_lb<P>(xv[t], uu[t], ll[t]) : 0.f;
                rest -= rs;  // (rs consumed before the slot is overwritten below)
            }
            // x (and the envelope) of the next step's rows into the slot: the gathers of a
            // candidate row miss L1 and their latency hides behind this step's cells
            stage_rows8(slot + XA, xr, i0 + 8, n);
            if (casc) {
                stage_rows8(slot + XA + 8, ur, i0 + 8, n);
                stage_rows8(slot + XA + 16, lr, i0 + 8, n);
            }
            // row+column cascade: the column terms of [C(i0), C(i0) + 8) (y, U(L(y)), L(U(y))
            // of the query, U(x), L(x) of the candidate) are copied into the lane's slot (free
            // while the lane is active) and subtracted at the end of the step
            if (casc2) {
                const int qy = reinterpret_cast<const int *>(slot)[SL - 2];
                const int64_t cx = (int64_t)reinterpret_cast<const uint32_t *>(slot)[SL - 1];
                const int cc = i0 + a.col_c0;
                stage_rows8(slot, a.yq + (int64_t)qy * n, cc, n);
                stage_rows8(slot + 8, a.LUq + (int64_t)qy * n, cc, n);
                stage_rows8(slot + 16, a.ULq + (int64_t)qy * n, cc, n);
                stage_rows8(slot + 24, a.Uxdb + cx * n, cc, n);
                stage_rows8(slot + 32, a.Lxdb + cx * n, cc, n);
            }
            cp_commit();
            // up to two blocks of four rows, then the abandon test
#pragma unroll 1
            for (int blk = 0; blk < 2; ++blk) {
                if (i + 4 > n) break;
                const float x4[4] = {xv[0], xv[1], xv[2], xv[3]};
                if constexpr (YG) {
                    four_rows_g<WB, P, EXACT>(B, ybase + (kYPadL - w) + i, x4, w2);
                    i += 4;
#pragma unroll
                    for (int t = 0; t < 4; ++t) xv[t] = xv[t + 4];
                } else {
                    four_rows<WB, P, EXACT>(B, Y2, x4, w2);
                    i += 4;
#pragma unroll
                    for (int t = 0; t < 4; ++t) xv[t] = xv[t + 4];
                    // shift the y window by four and append y[i + w + 1 .. i + w + 4] (next block)
#pragma unroll
                    for (int k = 0; k + 2 < NY / 2; ++k) Y2[k] = Y2[k + 2];
                    const float4 v = __ldg(reinterpret_cast<const float4 *>(yr + (kYPadL - w - sh) + i + NY - 4));
                    Y2[NY / 2 - 2] = make_float2(v.x, v.y);
                    Y2[NY / 2 - 1] = make_float2(v.z, v.w);
                }
            }
            if (i + 4 > n && i < n && i - i0 < 8) {  // tail rows (n % 4 != 0): one row at a time
                while (i < n) {
                    float prev = kInf;
#pragma unroll
                    for (int d = 0; d < NB; ++d) {
                        const float yd = YG ? ybase[(kYPadL - w) + i + d] : ((d & 1) ? Y2[YG ? 0 : d >> 1].y : Y2[YG ? 0 : d >> 1].x);
                        float c = cell<P>(min3f(B[d], B[d + 1], prev), __ldg(xr + i) - yd);
                        if (!EXACT && d > w2) c = kInf;
                        B[d] = c;
                        prev = c;
                    }
                    ++i;
                    if constexpr (!YG) {
#pragma unroll
                        for (int k = 0; k + 1 < NY / 2; ++k) Y2[k] = make_float2(Y2[k].y, Y2[k + 1].x);
                        Y2[NY / 2 - 1] = make_float2(Y2[NY / 2 - 1].y, __ldg(yr + (kYPadL - w - sh) + i + NY - 1));
                    }
                }
            }
            cp_wait<0>();
            {
                const float4 x0 = *reinterpret_cast<const float4 *>(slot + XA);
                const float4 x1 = *reinterpret_cast<const float4 *>(slot + XA + 4);
                xv[0] = x0.x; xv[1] = x0.y; xv[2] = x0.z; xv[3] = x0.w;
                xv[4] = x1.x; xv[5] = x1.y; xv[6] = x1.z; xv[7] = x1.w;
            }
            if (casc2) {
                // the columns [C(i0), C(i)) may have been visited by the rows just computed; the
                // columns >= C(i) only by rows >= i (reading c21)
                const int ncol = i - i0;  // 4 or 8 (n % 4 == 0)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (4 * h < ncol) {
                        const float4 yv = *reinterpret_cast<const float4 *>(slot + 4 * h);
                        const float4 lu = *reinterpret_cast<const float4 *>(slot + 8 + 4 * h);
                        const float4 ul = *reinterpret_cast<const float4 *>(slot + 16 + 4 * h);
                        const float4 ux = *reinterpret_cast<const float4 *>(slot + 24 + 4 * h);
                        const float4 lx = *reinterpret_cast<const float4 *>(slot + 32 + 4 * h);
                        rest -= col_lb<P>(yv.x, ux.x, lx.x, lu.x, ul.x) + col_lb<P>(yv.y, ux.y, lx.y, lu.y, ul.y) +
                                col_lb<P>(yv.z, ux.z, lx.z, lu.z, ul.z) + col_lb<P>(yv.w, ux.w, lx.w, lu.w, ul.w);
                    }
                }
            }
            // ---- (d) finished or abandoned lanes become free ----
            if (i >= n) {
                cells_done += band_cells(n, n, w);
                float r = B[WB];
                if constexpr (!EXACT) {
#pragma unroll
                    for (int d = 0; d < NB; ++d)
                        if (d == w) r = B[d];
                }
                if constexpr (WALK) { has_res = r <= thr; res_v = r; }
                else a.res[item] = rootp<P>(r);
                st = kFree;
            } else {
                if (recm) {  // (n % 4 == 0: i = i0 + 8 here)
                    const __half *hs = reinterpret_cast<const __half *>(slot);
                    if (i == 8) rest += __half2float(hs[0]);
                    rest -= __half2float(hs[i >> 3]);
                }
                if (!a.no_abandon && band_min<WB>(B) + rest > thr) {
                    if constexpr (!WALK) a.res[item] = kInf;
                    cells_done += band_cells(i, n, w);
                    ++n_abandon;  // early abandon (readings c15, c19, c21)
                    st = kFree;
                }
            }
        }
        if constexpr (WALK) {
            if (__any_sync(0xffffffffu, has_res))
                walk_results_warp(a, has_res, reinterpret_cast<const int *>(slot)[SL - 2],
                                  reinterpret_cast<const uint32_t *>(slot)[SL - 1], res_v, lane);
        }
    }
    if (a.cells) {
        unsigned long long cells = cells_done;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cells += __shfl_xor_sync(0xffffffffu, cells, o);
        if (lane == 0) atomicAdd(a.cells, cells);
    }
    if (a.started) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) n_started += __shfl_xor_sync(0xffffffffu, n_started, o);
        if (lane == 0 && n_started) atomicAdd(a.started, (unsigned long long)n_started);
    }
    if (a.abandoned) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) n_abandon += __shfl_xor_sync(0xffffffffu, n_abandon, o);
        if (lane == 0 && n_abandon) atomicAdd(a.abandoned, (unsigned long long)n_abandon);
    }
}

// Generic fallback for w > 64: one thread per pair, band kept in global scratch.
template <int P, bool WALK>
__global__ void dtw_generic_kernel(DtwArgs a, const float *__restrict__ yraw, float *__restrict__ scratch,
                                   int smem_pitch) {
    extern __shared__ float gband[];  // smem_pitch > 0: each thread's band in shared memory
    const int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= a.total) return;
    const int n = a.n, w = a.w, nb = 2 * w + 1;
    const float *xr, *yr;
    float thr = kInf;
    int lo = 0;
    uint32_t cand = 0;
    if constexpr (WALK) {
        int hi = a.Qb;
        while (hi - lo > 1) { int mid = (lo + hi) >> 1; if (a.item_off[mid] <= item) lo = mid; else hi = mid; }
        const int64_t j = a.pos[lo] + (item - a.item_off[lo]);
        const unsigned long long key = a.list[list_base(a.loff, a.cap, lo) + j];
        cand = (uint32_t)(key & 0xffffffffu);
        const float beta = key_bound(key);
        thr = *reinterpret_cast<volatile float *>(a.thr + lo);
        if (beta > thr) return;
        if (a.started) atomicAdd(a.started, 1ull);
        xr = a.db + (int64_t)(key & 0xffffffffu) * n;
        yr = yraw + (int64_t)lo * n;
    } else {
        xr = a.db + item * n;
        yr = yraw + item * n;
    }
    float *B = smem_pitch > 0 ? gband + threadIdx.x * smem_pitch : scratch + item * (int64_t)(nb + 1);
    for (int d = 0; d <= nb; ++d) B[d] = kInf;
    B[w] = 0.f;
    for (int i = 0; i < n; ++i) {
        const float xv = xr[i];
        float prev = kInf, rmin = kInf;
        for (int d = 0; d < nb; ++d) {
            const int j = i + d - w;
            float v = kInf;
            if (j >= 0 && j < n) v = cell<P>(min3f(B[d], B[d + 1], prev), xv - yr[j]);
            B[d] = v;
            prev = v;
            rmin = fminf(rmin, v);
        }
        if (!a.no_abandon && rmin > thr) {
            if constexpr (!WALK) a.res[item] = kInf;
            if (a.cells) atomicAdd(a.cells, band_cells(i + 1, n, w));
            if (a.abandoned) atomicAdd(a.abandoned, 1ull);
            return;
        }
    }
    if (a.cells) atomicAdd(a.cells, band_cells(n, n, w));
    if constexpr (WALK) {
        if (B[w] <= thr) {
            const unsigned pos = atomicAdd(a.rcount, 1u);
            a.rkey[pos] = pack_key(B[w], cand);
            a.rq[pos] = lo;
        }
    } else {
        a.res[item] = rootp<P>(B[w]);
    }
}

template <int WB, int P, bool EXACT, bool WALK, bool YG>
int launch_dtw4_t(const DtwArgs &a, cudaStream_t st) {
    DTWLB_CUDA(cudaMemsetAsync(a.queue, 0, sizeof(unsigned), st));
    const int64_t chunks = ceil_div(a.total, kChunk4);
    int64_t warps = std::min<int64_t>(chunks, (int64_t)148 * 48);  // persistent-ish: <= 48 warps per SM
    const int64_t grid = ceil_div(warps * 32, NT);
    const size_t smem = Dtw4Cfg<WB, YG>::smem + (YG ? (size_t)(NT / 32) * a.LP * sizeof(float) : 0);
    auto k = dtw4_kernel<WB, P, EXACT, WALK, YG>;
    DTWLB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<(unsigned)grid, NT, smem, st>>>(a);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

template <int WB, int P, bool EXACT, bool WALK>
int launch_dtw_t(const DtwArgs &a, cudaStream_t st) {
    // w <= 32: y window in registers (or, DTWLB_DTW_YG=1, read through L1); 32 < w <= 64:
    // the y window read through L1 (the band alone needs 2w+2 registers)
    static const bool env_yg = [] { const char *e = getenv("DTWLB_DTW_YG"); return e && atoi(e); }();
    if (!a.queue) {
        set_error(DTWLB_EINVAL, "internal: the DTW kernel needs its work-queue counter");
        return DTWLB_EINVAL;
    }
    if constexpr (WB <= 32) {
        if (env_yg) return launch_dtw4_t<WB, P, EXACT, WALK, true>(a, st);
        return launch_dtw4_t<WB, P, EXACT, WALK, false>(a, st);
    } else {
        return launch_dtw4_t<WB, P, EXACT, WALK, true>(a, st);
    }
}

template <int P, bool WALK>
int launch_dtw_p(const DtwArgs &a, cudaStream_t st) {
    const int w = a.w;
#define DTWLB_EX(W_) if (w == W_) return launch_dtw_t<W_, P, true, WALK>(a, st)
    DTWLB_EX(0); DTWLB_EX(12); DTWLB_EX(25); DTWLB_EX(50); DTWLB_EX(51);
#undef DTWLB_EX
    if (w <= 4) return launch_dtw_t<4, P, false, WALK>(a, st);
    if (w <= 8) return launch_dtw_t<8, P, false, WALK>(a, st);
    if (w <= 16) return launch_dtw_t<16, P, false, WALK>(a, st);
    if (w <= 32) return launch_dtw_t<32, P, false, WALK>(a, st);
    if (w <= 64) return launch_dtw_t<64, P, false, WALK>(a, st);
    set_error(DTWLB_EINVAL, "internal: register-band DTW needs w <= 64");
    return DTWLB_EINVAL;
}

__global__ void build_ysh_kernel(const float *__restrict__ y, int64_t rows, int n, float *__restrict__ ysh,
                                 int LP) {
    const int64_t total = rows * (int64_t)LP;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / LP;
        const int u = (int)(t - r * LP);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int j = u + s - kYPadL;  // ysh[s][r][u] = ypad[r][u + s]
            ysh[(int64_t)s * rows * LP + t] = (j >= 0 && j < n) ? y[r * n + j] : kInf;
        }
    }
}

}  // namespace

int launch_build_ysh(const float *y, int64_t rows, int n, float *ysh, int LP, cudaStream_t st) {
    if (rows == 0) return DTWLB_OK;
    const int64_t total = rows * (int64_t)LP;
    const int grid = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 16);
    build_ysh_kernel<<<grid, 256, 0, st>>>(y, rows, n, ysh, LP);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

// Generic path needs raw query rows and a scratch band; the caller passes them via
// the globals below (set by launch_dtw_generic).
int launch_topk_merge(const DtwArgs &a, cudaStream_t st) {
    topk_merge_kernel<<<148, 256, 0, st>>>(a);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

int launch_dtw(const DtwArgs &a, int p, bool walk, cudaStream_t st) {
    if (a.total == 0) return DTWLB_OK;
    if (p == 0) {  // DTW_inf: pairs mode only (dtw_band)
        if (walk) {
            set_error(DTWLB_EUNSUPPORTED, "nn_search: p = infinity unsupported");
            return DTWLB_EUNSUPPORTED;
        }
        return launch_dtw_p<0, false>(a, st);
    }
    if (p == 4) {  // DTW_4: pairs mode only (dtw_band)
        if (walk) {
            set_error(DTWLB_EUNSUPPORTED, "nn_search: p = 4 unsupported");
            return DTWLB_EUNSUPPORTED;
        }
        return launch_dtw_p<4, false>(a, st);
    }
    if (p == 1) return walk ? launch_dtw_p<1, true>(a, st) : launch_dtw_p<1, false>(a, st);
    return walk ? launch_dtw_p<2, true>(a, st) : launch_dtw_p<2, false>(a, st);
}

bool dtw_generic_needs_scratch(int w) { return (size_t)128 * ((2 * w + 2) | 1) * sizeof(float) > 200 * 1024; }

int launch_dtw_generic(const DtwArgs &a, const float *yraw, float *scratch, int p, bool walk,
                       cudaStream_t st) {
    if (a.total == 0) return DTWLB_OK;
    const int64_t grid = ceil_div(a.total, 128);
    // the band (2w+2 floats per pair) in shared memory when 128 of them fit (odd pitch: the
    // threads' same-index cells fall in different banks), else in the global scratch
    int pitch = (2 * a.w + 2) | 1;
    size_t smem = (size_t)128 * pitch * sizeof(float);
    if (dtw_generic_needs_scratch(a.w)) { pitch = 0; smem = 0; }
    if (smem > 48 * 1024) {
        DTWLB_CUDA(cudaFuncSetAttribute(dtw_generic_kernel<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        DTWLB_CUDA(cudaFuncSetAttribute(dtw_generic_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        DTWLB_CUDA(cudaFuncSetAttribute(dtw_generic_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        DTWLB_CUDA(cudaFuncSetAttribute(dtw_generic_kernel<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        DTWLB_CUDA(cudaFuncSetAttribute(dtw_generic_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        DTWLB_CUDA(cudaFuncSetAttribute(dtw_generic_kernel<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    if (p == 4) {
        if (walk) {
            set_error(DTWLB_EUNSUPPORTED, "nn_search: p = 4 unsupported");
            return DTWLB_EUNSUPPORTED;
        }
        dtw_generic_kernel<4, false><<<(unsigned)grid, 128, smem, st>>>(a, yraw, scratch, pitch);
    } else if (p == 0) {
        if (walk) {
            set_error(DTWLB_EUNSUPPORTED, "nn_search: p = infinity unsupported");
            return DTWLB_EUNSUPPORTED;
        }
        dtw_generic_kernel<0, false><<<(unsigned)grid, 128, smem, st>>>(a, yraw, scratch, pitch);
    } else if (p == 1) {
        if (walk) dtw_generic_kernel<1, true><<<(unsigned)grid, 128, smem, st>>>(a, yraw, scratch, pitch);
        else dtw_generic_kernel<1, false><<<(unsigned)grid, 128, smem, st>>>(a, yraw, scratch, pitch);
    } else {
        if (walk) dtw_generic_kernel<2, true><<<(unsigned)grid, 128, smem, st>>>(a, yraw, scratch, pitch);
        else dtw_generic_kernel<2, false><<<(unsigned)grid, 128, smem, st>>>(a, yraw, scratch, pitch);
    }
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

}  // namespace dtwlb
