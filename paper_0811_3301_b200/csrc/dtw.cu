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

__device__ __forceinline__ float f4get(const float4 &v, int k) {
    return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
}

// B holds row i-1; computes rows i (x = xa) and i+1 (x = xb); B <- row i+1.
// ys: aligned pointer with ys[d] = y[i + d - w] (padded), d = 0..2WB+1.
template <int WB, int P, bool EXACT>
__device__ __forceinline__ void two_rows(float (&B)[2 * WB + 2], float xa, float xb,
                                         const float *__restrict__ ys, int w2) {
    constexpr int NB = 2 * WB + 1;
    float a_prev = kInf, rb_prev = kInf;
    float4 yv4;
#pragma unroll
    for (int d = 0; d < NB; ++d) {
        if ((d & 3) == 0) yv4 = __ldg(reinterpret_cast<const float4 *>(ys + d));
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
        if ((d & 3) == 0) yv4 = __ldg(reinterpret_cast<const float4 *>(ys + d));
        const float yv = f4get(yv4, d & 3);
        float b = cell<P>(fminf(a_prev, rb_prev), xb - yv);
        if (!EXACT && d - 1 > w2) b = kInf;
        B[NB - 1] = b;
    }
}

template <int WB, int P, bool EXACT>
__device__ __forceinline__ void one_row(float (&B)[2 * WB + 2], float xa, const float *__restrict__ ys,
                                        int w2) {
    constexpr int NB = 2 * WB + 1;
    float a_prev = kInf;
    float4 yv4;
#pragma unroll
    for (int d = 0; d < NB; ++d) {
        if ((d & 3) == 0) yv4 = __ldg(reinterpret_cast<const float4 *>(ys + d));
        float a = cell<P>(min3f(B[d], B[d + 1], a_prev), xa - f4get(yv4, d & 3));
        if (!EXACT && d > w2) a = kInf;
        B[d] = a;
        a_prev = a;
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

template <int WB, int P, bool EXACT, bool WALK>
__global__ void __launch_bounds__(NT)
dtw_kernel(DtwArgs a, int ipw) {
    constexpr int NB = 2 * WB + 1;
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * NT + threadIdx.x) >> 5;
    const int64_t a0 = gw * ipw;
    if (a0 >= a.total) return;
    const int64_t a1 = (a.total < a0 + ipw) ? a.total : a0 + ipw;
    const int n = a.n, w = EXACT ? WB : a.w, w2 = 2 * w;

    int64_t cursor = a0;
    bool has = false;
    int64_t item = 0;
    const float *xr = nullptr, *yb = nullptr;
    float thr = kInf;
    int i = 0;
    float B[NB + 1];
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
                    // query of this item: last q with item_off[q] <= item
                    int lo = 0, hi = a.Qb;  // item_off[lo] <= item < item_off[hi]
                    while (hi - lo > 1) {
                        int mid = (lo + hi) >> 1;
                        if (a.item_off[mid] <= item) lo = mid; else hi = mid;
                    }
                    const int q = lo;
                    const int64_t j = a.pos[q] + (item - a.item_off[q]);
                    DCHECK(q >= 0 && q < a.Qb && item >= a.item_off[q] && item < a.item_off[q + 1] && j >= 0 && j < a.cap,
                           "dtw item %lld q=%d j=%lld pos=%d off=%d,%d", (long long)item, q, (long long)j, a.pos[q],
                           a.item_off[q], a.item_off[q + 1]);
                    const unsigned long long key = a.list[(int64_t)q * a.cap + j];
                    const uint32_t c = (uint32_t)(key & 0xffffffffu);
                    DCHECK((int64_t)c < a.Ndb, "dtw key c=%u N=%lld q=%d j=%lld key=%llx", c, (long long)a.Ndb, q, (long long)j, key);
                    beta = __uint_as_float((uint32_t)(key >> 32));
                    thr = a.thr[q];
                    xr = a.db + (int64_t)c * n;
                    yb = a.ysh + (int64_t)q * a.LP;
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
            const int i0 = i, iend = min(n, i + 8);
            while (i + 1 < iend) {
                const int s0 = i - w + kYPadL;
                const float *ys = yb + (int64_t)(s0 & 3) * a.ysh_stride_s + (s0 & ~3);
                two_rows<WB, P, EXACT>(B, __ldg(xr + i), __ldg(xr + i + 1), ys, w2);
                i += 2;
            }
            if (i < iend) {
                const int s0 = i - w + kYPadL;
                const float *ys = yb + (int64_t)(s0 & 3) * a.ysh_stride_s + (s0 & ~3);
                one_row<WB, P, EXACT>(B, __ldg(xr + i), ys, w2);
                i += 1;
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
            } else if (band_min<WB>(B) > thr) {
                a.res[item] = kInf;  // early abandon (reading c15)
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
int launch_dtw_t(const DtwArgs &a, cudaStream_t st) {
    const int ipw = 64;
    const int64_t warps = ceil_div(a.total, ipw);
    const int64_t grid = ceil_div(warps * 32, NT);
    dtw_kernel<WB, P, EXACT, WALK><<<(unsigned)grid, NT, 0, st>>>(a, ipw);
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
