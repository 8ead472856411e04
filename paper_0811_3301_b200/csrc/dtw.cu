// dtw.cu -- banded DTW_p (a5): the recursion of P:199-210 (section "Dynamic Time
// Warping") evaluated in its forward (prefix) form, which equals the suffix form
// by reversing both series:
//
//   D(i,j) = |x_i - y_j|^p + min(D(i-1,j), D(i,j-1), D(i-1,j-1)),  |i-j| <= w,
//   D(-1,-1) = 0, everything else outside the band = +inf;  DTW_p^p = D(n-1,n-1).
//
// B200 design: thread-per-pair with the 2w+1-wide band held in REGISTERS
// (template WB >= w, exact instantiations for the configs' w), so each cell is
// the minimal 3-op SASS sequence FADD (x-y), FMNMX3, FADD|abs| / FFMA.  Two rows
// are advanced per pass in an interleaved order (row i cell d, then row i+1 cell
// d-1), giving two independent dependency chains per thread and letting both
// cells share one y value.  The query row is read as 128-bit vectors from four
// pre-shifted, +inf-padded copies (out-of-range columns cost +inf, so no column
// tests), i.e. one 16-byte L1-resident load per 8 cells.
// Early abandoning (not in the paper, reading c15): every path crosses
// every row and costs are >= 0, so once a row's minimum exceeds the threshold
// tau^p(1+eps) the pair cannot enter the top-k and is scored +inf.  Lanes are
// desynchronised: a lane whose pair finishes or is abandoned immediately takes
// the next pair of its warp's queue (ballot-based refill), so one long pair
// does not idle the other 31 lanes.
#include "kernels.cuh"

namespace dtwlb {

int dtw_padded_len(int n) { return ((n + kYPadL + 2 * 64 + 8) + 3) & ~3; }

namespace {

constexpr int NT = 128;

template <int P>
__device__ __forceinline__ float cell(float m, float t) {
    if constexpr (P == 1) return m + fabsf(t);
    else return fmaf(t, t, m);
}

// y window loads: shared memory (WALK: the warp's query is staged) or read-only global
template <bool SMEM>
__device__ __forceinline__ float4 ld4(const float *p) {
    if constexpr (SMEM) return *reinterpret_cast<const float4 *>(p);
    else return __ldg(reinterpret_cast<const float4 *>(p));
}

__device__ __forceinline__ float f4get(const float4 &v, int k) {
    return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
}

// B holds row i-1; computes rows i (x = xa) and i+1 (x = xb); B <- row i+1.
// ys: aligned pointer with ys[d] = y[i + d - w] (padded), d = 0..2WB+1.
template <int WB, int P, bool EXACT, bool SMEM>
__device__ __forceinline__ void two_rows(float (&B)[2 * WB + 2], float xa, float xb,
                                         const float *__restrict__ ys, int w2) {
    constexpr int NB = 2 * WB + 1;
    float a_prev = kInf, rb_prev = kInf;
    float4 yv4;
#pragma unroll
    for (int d = 0; d < NB; ++d) {
        if ((d & 3) == 0) yv4 = ld4<SMEM>(ys + d);
        const float yv = f4get(yv4, d & 3);
        float a = cell<P>(min3f(B[d], B[d + 1], a_prev), xa - yv);
        if (!EXACT && d > w2) a = kInf;
        if (d >= 1) {
            float b = cell<P>(min3f(a_prev, a, rb_prev), xb - yv);
            if (!EXACT && d - 1 > w2) b = kInf;
            B[d - 1] = b;
            rb_prev = b;
        }
        a_prev = a;
    }
    {
        constexpr int d = NB;  // row i+1, cell 2WB uses y[i+1+2WB-w]
        if ((d & 3) == 0) yv4 = ld4<SMEM>(ys + d);
        const float yv = f4get(yv4, d & 3);
        float b = cell<P>(fminf(a_prev, rb_prev), xb - yv);
        if (!EXACT && d - 1 > w2) b = kInf;
        B[NB - 1] = b;
    }
}

template <int WB, int P, bool EXACT, bool SMEM>
__device__ __forceinline__ void one_row(float (&B)[2 * WB + 2], float xa, const float *__restrict__ ys,
                                        int w2) {
    constexpr int NB = 2 * WB + 1;
    float a_prev = kInf;
    float4 yv4;
#pragma unroll
    for (int d = 0; d < NB; ++d) {
        if ((d & 3) == 0) yv4 = ld4<SMEM>(ys + d);
        float a = cell<P>(min3f(B[d], B[d + 1], a_prev), xa - f4get(yv4, d & 3));
        if (!EXACT && d > w2) a = kInf;
        B[d] = a;
        a_prev = a;
    }
}

// x[i0 .. i0+7] of a candidate row (0 beyond n); vector loads when the row allows it
__device__ __forceinline__ void load_x8(float (&xv)[8], const float *__restrict__ xr, int i0, int n) {
    if (((n & 3) == 0) && i0 + 8 <= n) {
        const float4 a = __ldg(reinterpret_cast<const float4 *>(xr + i0));
        const float4 b = __ldg(reinterpret_cast<const float4 *>(xr + i0 + 4));
        xv[0] = a.x; xv[1] = a.y; xv[2] = a.z; xv[3] = a.w;
        xv[4] = b.x; xv[5] = b.y; xv[6] = b.z; xv[7] = b.w;
    } else {
#pragma unroll
        for (int t = 0; t < 8; ++t) xv[t] = i0 + t < n ? __ldg(xr + i0 + t) : 0.f;
    }
}

// LB_Keogh term of row i: d(x_i, [L(y)_i, U(y)_i])^p.  Every banded path visits row i
// in some column j with |i-j| <= w, at cost |x_i - y_j|^p >= this term, so the sum of
// the terms of the rows not yet computed bounds what the path still has to pay
// (cascading abandon, reading c19).
template <int P>
__device__ __forceinline__ float row_lb(float x, float u, float l) {
    const float d = max3f(x - u, l - x, 0.f);
    return P == 1 ? d : d * d;
}

template <int WB>
__device__ __forceinline__ float band_min(const float (&B)[2 * WB + 2]) {
    float m = B[0];
#pragma unroll
    for (int d = 1; d + 1 < 2 * WB + 1; d += 2) m = min3f(m, B[d], B[d + 1]);
    if ((2 * WB + 1) % 2 == 0) m = fminf(m, B[2 * WB]);
    return m;
}

template <int WB, int P, bool EXACT, bool WALK>
__global__ void __launch_bounds__(NT)
dtw_kernel(DtwArgs a, int ipw) {
    constexpr int NB = 2 * WB + 1;
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * NT + threadIdx.x) >> 5;
    const int n = a.n, w = EXACT ? WB : a.w, w2 = 2 * w;
    int64_t a0, a1;
    // WALK: the warp's chunk belongs to one query q (found once per warp)
    int q = 0;
    int64_t item_base = 0, lpos = 0;
    const float *yq = nullptr;
    float thr_q = kInf;
    if constexpr (WALK) {
        if (gw >= a.nchunks) return;
        int lo = 0, hi = a.Qb;  // chunk_off[lo] <= gw < chunk_off[hi]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (a.chunk_off[mid] <= gw) lo = mid; else hi = mid;
        }
        q = lo;
        item_base = a.item_off[q];
        const int64_t cnt = a.item_off[q + 1] - item_base;
        const int64_t k0 = (gw - a.chunk_off[q]) * (int64_t)ipw;
        a0 = item_base + k0;
        a1 = item_base + (cnt < k0 + ipw ? cnt : k0 + ipw);
        lpos = a.pos[q];
        // stage the query's four shifted copies in this warp's shared-memory slice:
        // desynchronised lanes then read 16-byte chunks from shared memory (~4-8
        // wavefronts per warp load) instead of scattered L1 lines (~32)
        extern __shared__ __align__(16) float ysm[];
        float *mine = ysm + (size_t)(threadIdx.x >> 5) * 4 * a.LP;
        const float *src = a.ysh + (int64_t)q * a.LP;
        for (int s = 0; s < 4; ++s)
            for (int t = lane * 4; t < a.LP; t += 128)
                *reinterpret_cast<float4 *>(mine + s * a.LP + t) =
                    __ldg(reinterpret_cast<const float4 *>(src + (int64_t)s * a.ysh_stride_s + t));
        __syncwarp();
        yq = mine;
        thr_q = a.thr[q];
        DCHECK(k0 < cnt, "dtw chunk gw=%lld q=%d k0=%lld cnt=%lld", (long long)gw, q, (long long)k0, (long long)cnt);
    } else {
        a0 = gw * ipw;
        if (a0 >= a.total) return;
        a1 = (a.total < a0 + ipw) ? a.total : a0 + ipw;
    }

    int64_t cursor = a0;
    bool has = false;
    int64_t item = 0;
    const float *xr = nullptr, *yb = nullptr;
    const int64_t ystride = WALK ? a.LP : a.ysh_stride_s;  // elements between shifted copies
    float thr = kInf;
    int i = 0;
    float B[NB + 1];
    float xv[8];  // x of the current 8-row block
    // cascading abandon: rest = LB_Keogh^p terms of the rows not yet computed
    const bool casc = WALK && a.b1 != nullptr;
    float rest = 0.f;
    const float *ur = nullptr, *lr = nullptr;
    unsigned long long rows_done = 0, n_abandon = 0, n_started = 0;

    while (true) {
        // ---- refill lanes without a pair ----
        const unsigned need = __ballot_sync(0xffffffffu, !has);
        if (need) {
            const int64_t mine = cursor + __popc(need & ((1u << lane) - 1));
            cursor += __popc(need);
            if (!has && mine < a1) {
                item = mine;
                float beta = 0.f;
                if constexpr (WALK) {
                    const int64_t j = lpos + (item - item_base);
                    DCHECK(j >= 0 && j < a.cap, "dtw item %lld q=%d j=%lld", (long long)item, q, (long long)j);
                    const unsigned long long key = a.list[(int64_t)q * a.cap + j];
                    const uint32_t c = (uint32_t)(key & 0xffffffffu);
                    DCHECK((int64_t)c < a.Ndb, "dtw key c=%u N=%lld q=%d j=%lld key=%llx", c, (long long)a.Ndb, q,
                           (long long)j, key);
                    beta = __uint_as_float((uint32_t)(key >> 32));
                    thr = thr_q;
                    xr = a.db + (int64_t)c * n;
                    yb = yq;
                    if (casc) {
                        rest = fabsf(__ldg(a.b1 + (int64_t)q * a.ldb + c));  // beta1 = sum of all row terms
                        ur = a.Uq + (int64_t)q * n;
                        lr = a.Lq + (int64_t)q * n;
                    }
                } else {
                    thr = kInf;
                    xr = a.db + item * n;
                    yb = a.ysh + item * a.LP;
                }
                DCHECK(item < a.total, "dtw item %lld total %lld", (long long)item, (long long)a.total);
                if (beta > thr) {
                    a.res[item] = kInf;  // pruned by the bound under the current threshold
                } else {
                    has = true;
                    ++n_started;
                    i = 0;
                    load_x8(xv, xr, 0, n);
#pragma unroll
                    for (int d = 0; d <= NB; ++d) B[d] = kInf;
#pragma unroll
                    for (int d = 0; d < NB; ++d)
                        if (d == w) B[d] = 0.f;  // virtual D(-1,-1) = 0 sits on the diagonal
                }
            }
        }
        if (!__any_sync(0xffffffffu, has) && cursor >= a1) break;

        if (has) {
            // ---- advance this lane's pair by up to 8 rows ----
            // x of this block was loaded with the previous block (or at setup); issue the
            // loads of the next block now so their latency hides behind this block's cells
            const int i0 = i, iend = min(n, i + 8);
            float xn[8];
            load_x8(xn, xr, iend, n);
            if (casc) {
#pragma unroll
                for (int t = 0; t < 8; ++t)
                    if (i0 + t < iend) rest -= row_lb<P>(xv[t], __ldg(ur + i0 + t), __ldg(lr + i0 + t));
            }
            while (i + 1 < iend) {
                const int s0 = i - w + kYPadL;
                const float *ys = yb + (int64_t)(s0 & 3) * ystride + (s0 & ~3);
                two_rows<WB, P, EXACT, WALK>(B, xv[0], xv[1], ys, w2);
#pragma unroll
                for (int t = 0; t < 6; ++t) xv[t] = xv[t + 2];
                i += 2;
            }
            if (i < iend) {
                const int s0 = i - w + kYPadL;
                const float *ys = yb + (int64_t)(s0 & 3) * ystride + (s0 & ~3);
                one_row<WB, P, EXACT, WALK>(B, xv[0], ys, w2);
                i += 1;
            }
#pragma unroll
            for (int t = 0; t < 8; ++t) xv[t] = xn[t];
            rows_done += (unsigned long long)(i - i0);
            if (i >= n) {
                float r = B[WB];
                if constexpr (!EXACT) {
#pragma unroll
                    for (int d = 0; d < NB; ++d)
                        if (d == w) r = B[d];
                }
                a.res[item] = WALK ? r : rootp<P>(r);
                has = false;
            } else if (band_min<WB>(B) + rest > thr) {
                a.res[item] = kInf;  // early abandon (readings c15, c19)
                ++n_abandon;
                has = false;
            }
        }
    }
    if (a.cells) {
        unsigned long long cells = rows_done * (unsigned long long)(2 * w + 1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cells += __shfl_xor_sync(0xffffffffu, cells, o);
        if (lane == 0) atomicAdd(a.cells, cells);
    }
    if (a.started) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) n_started += __shfl_xor_sync(0xffffffffu, n_started, o);
        if (lane == 0 && n_started) atomicAdd(a.started, n_started);
    }
    if (a.abandoned) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) n_abandon += __shfl_xor_sync(0xffffffffu, n_abandon, o);
        if (lane == 0 && n_abandon) atomicAdd(a.abandoned, n_abandon);
    }
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
__device__ __forceinline__ void four_rows(float (&B)[2 * WB + 2], const float (&Y)[(2 * WB + 4 + 3) / 4 * 4],
                                          const float (&x)[4], int w2) {
    constexpr int NB = 2 * WB + 1;
    float p0 = kInf, p1 = kInf, p2 = kInf, p3 = kInf;   // left neighbours (same row)
    float a0 = kInf, a1 = kInf, a2 = kInf;              // row r cell (d-r-1): diag of row r+1
#pragma unroll
    for (int d = 0; d < NB + 3; ++d) {
        const float yv = Y[d];
        float c0 = kInf, c1 = kInf, c2 = kInf;
        if (d < NB) {  // row 0, cell d: up = B[d+1], diag = B[d]
            c0 = cell<P>(min3f(B[d], B[d + 1], p0), x[0] - yv);
            if (!EXACT && d > w2) c0 = kInf;
            p0 = c0;
        }
        if (d >= 1 && d - 1 < NB) {  // row 1, cell d-1: up = row0 cell d, diag = row0 cell d-1
            const float up = d < NB ? c0 : kInf;
            c1 = cell<P>(min3f(a0, up, p1), x[1] - yv);
            if (!EXACT && d - 1 > w2) c1 = kInf;
            p1 = c1;
        }
        if (d >= 2 && d - 2 < NB) {  // row 2, cell d-2
            const float up = (d - 1 < NB) ? c1 : kInf;
            c2 = cell<P>(min3f(a1, up, p2), x[2] - yv);
            if (!EXACT && d - 2 > w2) c2 = kInf;
            p2 = c2;
        }
        if (d >= 3) {  // row 3, cell d-3 (stored: B becomes row i+3)
            const float up = (d - 2 < NB) ? c2 : kInf;
            float c3 = cell<P>(min3f(a2, up, p3), x[3] - yv);
            if (!EXACT && d - 3 > w2) c3 = kInf;
            p3 = c3;
            B[d - 3] = c3;
        }
        a0 = c0;
        a1 = c1;
        a2 = c2;
    }
}

template <int WB, int P, bool EXACT, bool WALK>
__global__ void __launch_bounds__(NT)
dtw4_kernel(DtwArgs a) {
    constexpr int NB = 2 * WB + 1;
    constexpr int NY = (2 * WB + 4 + 3) / 4 * 4;  // window length, a multiple of 4 (aligned refills)
    const int lane = threadIdx.x & 31;
    const int n = a.n, w = EXACT ? WB : a.w, w2 = 2 * w;
    const int sh = (kYPadL - w) & 3;  // alignment class of (i - w) for i % 4 == 0
    const int64_t total = a.total;
    const int64_t nchunks = (total + kChunk4 - 1) / kChunk4;

    int64_t cbeg = 0, cend = 0, cursor = 0;
    bool has = false;
    int64_t item = 0;
    int q = 0;  // WALK: query of the lane's last item (items are in query order)
    const float *xr = nullptr, *yr = nullptr;
    float thr = kInf;
    int i = 0;
    float B[NB + 1], Y[NY];
    // cascading abandon: rest = LB_Keogh^p terms of the rows not yet computed
    const bool casc = WALK && a.b1 != nullptr;
    float rest = 0.f;
    const float *ur = nullptr, *lr = nullptr;
    unsigned long long rows_done = 0, n_abandon = 0, n_started = 0;

    while (true) {
        unsigned need = __ballot_sync(0xffffffffu, !has);
        if (need && cursor >= cend) {  // the warp's chunk is exhausted: grab the next one
            int64_t c = 0;
            if (lane == 0) c = atomicAdd(a.queue, 1u);
            c = __shfl_sync(0xffffffffu, c, 0);
            if (c < nchunks) {
                cbeg = c * kChunk4;
                cend = cbeg + kChunk4 < total ? cbeg + kChunk4 : total;
                cursor = cbeg;
                if constexpr (WALK) {
                    int lo = 0, hi = a.Qb;  // item_off[lo] <= cbeg < item_off[hi]
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if (a.item_off[mid] <= cbeg) lo = mid; else hi = mid;
                    }
                    q = lo;  // only read when a lane starts its next item (from this chunk on)
                }
            }
        }
        if (need && cursor < cend) {
            const int64_t mine = cursor + __popc(need & ((1u << lane) - 1));
            cursor += __popc(need);
            if (!has && mine < cend) {
                item = mine;
                float beta = 0.f;
                if constexpr (WALK) {
                    while (item >= a.item_off[q + 1]) ++q;
                    const int64_t j = a.pos[q] + (item - a.item_off[q]);
                    DCHECK(j >= 0 && j < a.cap, "dtw4 item %lld q=%d j=%lld", (long long)item, q, (long long)j);
                    const unsigned long long key = a.list[(int64_t)q * a.cap + j];
                    const uint32_t c = (uint32_t)(key & 0xffffffffu);
                    DCHECK((int64_t)c < a.Ndb, "dtw4 key c=%u q=%d", c, q);
                    beta = __uint_as_float((uint32_t)(key >> 32));
                    thr = a.thr[q];
                    xr = a.db + (int64_t)c * n;
                    if (casc) {
                        rest = fabsf(__ldg(a.b1 + (int64_t)q * a.ldb + c));  // beta1 = sum of all row terms
                        ur = a.Uq + (int64_t)q * n;
                        lr = a.Lq + (int64_t)q * n;
                    }
                    yr = a.ysh + (int64_t)sh * a.ysh_stride_s + (int64_t)q * a.LP;
                } else {
                    thr = kInf;
                    xr = a.db + item * n;
                    yr = a.ysh + (int64_t)sh * a.ysh_stride_s + item * a.LP;
                }
                if (beta > thr) {
                    a.res[item] = kInf;
                } else {
                    has = true;
                    ++n_started;
                    i = 0;
#pragma unroll
                    for (int d = 0; d <= NB; ++d) B[d] = kInf;
#pragma unroll
                    for (int d = 0; d < NB; ++d)
                        if (d == w) B[d] = 0.f;
                    // Y[d] = ypad[-w + kYPadL + d]; the copy `sh` makes base (kYPadL - w - sh) aligned
                    const float *ys = yr + (kYPadL - w - sh);
#pragma unroll
                    for (int d = 0; d < NY; d += 4) {
                        const float4 v = __ldg(reinterpret_cast<const float4 *>(ys + d));
                        Y[d] = v.x;
                        Y[d + 1] = v.y;
                        Y[d + 2] = v.z;
                        Y[d + 3] = v.w;
                    }
                }
            }
        }
        if (!__any_sync(0xffffffffu, has)) {
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
        if (has) {
            const int i0 = i;
            // up to two blocks of four rows, then the abandon test
#pragma unroll 1
            for (int blk = 0; blk < 2 && i + 4 <= n; ++blk) {
                float xv[4];
                if ((n & 3) == 0) {
                    const float4 v = __ldg(reinterpret_cast<const float4 *>(xr + i));
                    xv[0] = v.x; xv[1] = v.y; xv[2] = v.z; xv[3] = v.w;
                } else {
#pragma unroll
                    for (int t = 0; t < 4; ++t) xv[t] = __ldg(xr + i + t);
                }
                if (casc) {
                    if ((n & 3) == 0) {
                        const float4 u4 = __ldg(reinterpret_cast<const float4 *>(ur + i));
                        const float4 l4 = __ldg(reinterpret_cast<const float4 *>(lr + i));
                        rest -= row_lb<P>(xv[0], u4.x, l4.x) + row_lb<P>(xv[1], u4.y, l4.y) +
                                row_lb<P>(xv[2], u4.z, l4.z) + row_lb<P>(xv[3], u4.w, l4.w);
                    } else {
#pragma unroll
                        for (int t = 0; t < 4; ++t) rest -= row_lb<P>(xv[t], __ldg(ur + i + t), __ldg(lr + i + t));
                    }
                }
                four_rows<WB, P, EXACT>(B, Y, xv, w2);
                i += 4;
                // shift the y window by four and append y[i + w + 1 .. i + w + 4] (next block)
#pragma unroll
                for (int d = 0; d + 4 < NY; ++d) Y[d] = Y[d + 4];
                {
                    const float4 v = __ldg(reinterpret_cast<const float4 *>(yr + (kYPadL - w - sh) + i + NY - 4));
                    Y[NY - 4] = v.x; Y[NY - 3] = v.y; Y[NY - 2] = v.z; Y[NY - 1] = v.w;
                }
            }
            if (i + 4 > n && i < n) {  // tail rows (n % 4 != 0): one row at a time
                while (i < n) {
                    if (casc) rest -= row_lb<P>(__ldg(xr + i), __ldg(ur + i), __ldg(lr + i));
                    float prev = kInf;
#pragma unroll
                    for (int d = 0; d < NB; ++d) {
                        float c = cell<P>(min3f(B[d], B[d + 1], prev), __ldg(xr + i) - Y[d]);
                        if (!EXACT && d > w2) c = kInf;
                        B[d] = c;
                        prev = c;
                    }
                    ++i;
#pragma unroll
                    for (int d = 0; d + 1 < NY; ++d) Y[d] = Y[d + 1];
                    Y[NY - 1] = __ldg(yr + (kYPadL - w - sh) + i + NY - 1);
                }
            }
            rows_done += (unsigned long long)(i - i0);
            if (i >= n) {
                float r = B[WB];
                if constexpr (!EXACT) {
#pragma unroll
                    for (int d = 0; d < NB; ++d)
                        if (d == w) r = B[d];
                }
                a.res[item] = WALK ? r : rootp<P>(r);
                has = false;
            } else if (band_min<WB>(B) + rest > thr) {
                a.res[item] = kInf;  // early abandon (readings c15, c19)
                ++n_abandon;
                has = false;
            }
        }
    }
    if (a.cells) {
        unsigned long long cells = rows_done * (unsigned long long)(2 * w + 1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cells += __shfl_xor_sync(0xffffffffu, cells, o);
        if (lane == 0) atomicAdd(a.cells, cells);
    }
    if (a.started) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) n_started += __shfl_xor_sync(0xffffffffu, n_started, o);
        if (lane == 0 && n_started) atomicAdd(a.started, n_started);
    }
    if (a.abandoned) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) n_abandon += __shfl_xor_sync(0xffffffffu, n_abandon, o);
        if (lane == 0 && n_abandon) atomicAdd(a.abandoned, n_abandon);
    }
}

// Generic fallback for w > 64: one thread per pair, band kept in global scratch.
template <int P, bool WALK>
__global__ void dtw_generic_kernel(DtwArgs a, const float *__restrict__ yraw, float *__restrict__ scratch) {
    const int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (item >= a.total) return;
    const int n = a.n, w = a.w, nb = 2 * w + 1;
    const float *xr, *yr;
    float thr = kInf;
    if constexpr (WALK) {
        int lo = 0, hi = a.Qb;
        while (hi - lo > 1) { int mid = (lo + hi) >> 1; if (a.item_off[mid] <= item) lo = mid; else hi = mid; }
        const int64_t j = a.pos[lo] + (item - a.item_off[lo]);
        const unsigned long long key = a.list[(int64_t)lo * a.cap + j];
        const float beta = __uint_as_float((uint32_t)(key >> 32));
        thr = a.thr[lo];
        if (beta > thr) { a.res[item] = kInf; return; }
        xr = a.db + (int64_t)(key & 0xffffffffu) * n;
        yr = yraw + (int64_t)lo * n;
    } else {
        xr = a.db + item * n;
        yr = yraw + item * n;
    }
    float *B = scratch + item * (int64_t)(nb + 1);
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
        if (rmin > thr) { a.res[item] = kInf; return; }
    }
    a.res[item] = WALK ? B[w] : rootp<P>(B[w]);
}

template <int WB, int P, bool EXACT, bool WALK>
int launch_dtw4_t(const DtwArgs &a, cudaStream_t st) {
    DTWLB_CUDA(cudaMemsetAsync(a.queue, 0, sizeof(unsigned), st));
    const int64_t chunks = ceil_div(a.total, kChunk4);
    int64_t warps = std::min<int64_t>(chunks, (int64_t)148 * 48);  // persistent-ish: <= 48 warps per SM
    const int64_t grid = ceil_div(warps * 32, NT);
    dtw4_kernel<WB, P, EXACT, WALK><<<(unsigned)grid, NT, 0, st>>>(a);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

template <int WB, int P, bool EXACT, bool WALK>
int launch_dtw_t(const DtwArgs &a, cudaStream_t st) {
    if constexpr (WB <= 32) {
        if (a.queue) return launch_dtw4_t<WB, P, EXACT, WALK>(a, st);
    }
    const int ipw = kDtwIpw;
    const int64_t warps = WALK ? a.nchunks : ceil_div(a.total, ipw);
    const int64_t grid = ceil_div(warps * 32, NT);
    const size_t smem = WALK ? (size_t)(NT / 32) * 4 * a.LP * sizeof(float) : 0;
    if (smem > 48 * 1024)
        DTWLB_CUDA(cudaFuncSetAttribute(dtw_kernel<WB, P, EXACT, WALK>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dtw_kernel<WB, P, EXACT, WALK><<<(unsigned)grid, NT, smem, st>>>(a, ipw);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
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
int launch_dtw(const DtwArgs &a, int p, bool walk, cudaStream_t st) {
    if (a.total == 0) return DTWLB_OK;
    if (p == 1) return walk ? launch_dtw_p<1, true>(a, st) : launch_dtw_p<1, false>(a, st);
    return walk ? launch_dtw_p<2, true>(a, st) : launch_dtw_p<2, false>(a, st);
}

int launch_dtw_generic(const DtwArgs &a, const float *yraw, float *scratch, int p, bool walk,
                       cudaStream_t st) {
    if (a.total == 0) return DTWLB_OK;
    const int64_t grid = ceil_div(a.total, 128);
    if (p == 1) {
        if (walk) dtw_generic_kernel<1, true><<<(unsigned)grid, 128, 0, st>>>(a, yraw, scratch);
        else dtw_generic_kernel<1, false><<<(unsigned)grid, 128, 0, st>>>(a, yraw, scratch);
    } else {
        if (walk) dtw_generic_kernel<2, true><<<(unsigned)grid, 128, 0, st>>>(a, yraw, scratch);
        else dtw_generic_kernel<2, false><<<(unsigned)grid, 128, 0, st>>>(a, yraw, scratch);
    }
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

}  // namespace dtwlb
