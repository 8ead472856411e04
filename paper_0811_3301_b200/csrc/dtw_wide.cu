// dtw_wide.cu -- banded DTW_p for WIDE bands (w > 64: the band no longer fits one thread's
// registers), the a5 step of the cascade.  Recursion of P:199-210 (section "Dynamic Time
// Warping") in its forward (prefix) form, as dtw.cu:
//
//   D(i,j) = |x_i - y_j|^p + min(D(i-1,j), D(i,j-1), D(i-1,j-1)),  |i-j| <= w,
//   D(-1,-1) = 0, everything else outside the band = +inf;  DTW_p^p = D(n-1,n-1).
//
// B200 design: ONE PAIR PER FOUR LANES.  The 2w+1-cell band of a row is split into four
// segments of S cells held in the registers of four consecutive lanes (S = 51 for w = 100).
// Lane t processes row r = s - t at step s (a skewed pipeline): the left neighbour of its
// first cell is lane t-1's last cell of the same row, computed one step earlier, and the
// up neighbour of its last cell is lane t+1's first cell of the previous row, computed
// first in the same step -- two warp shuffles per row, every other cell dependency is in
// registers, so a cell is the same 3-op FADD, FMNMX3, FFMA|FADD sequence as dtw4_kernel.
// The query values of a lane's cells sit in a register window that shifts by four columns
// every four rows (4 new values loaded one block ahead, like the row's x values).
// UNCONSTRAINED DTW (w >= n-1, the Appendix B workload P:1079-1092) uses COLUMN coordinates
// instead: lane t owns columns [tS, tS+S) of every row, its query values are constant, and
// the only exchange is the last column to lane t+1 (one shuffle per row); columns beyond n
// never feed a valid cell (dependencies point left and up only).
// Eight pairs per warp advance in lockstep phases of 8 rows: pairs start at step multiples of
// 8, the exact early abandon (reading c15: a row whose minimum exceeds tau^p(1+eps) ends the
// pair; the four lanes record their segment minima of the checkpoint row and combine them
// with two shuffles) and the refills of finished groups happen at the same phase for every
// group, so the control flow stays warp-uniform.  Work items come from a global counter in
// chunks of 32.
#include "kernels.cuh"

namespace dtwlb {

namespace {

constexpr int KW4 = 4;     // lanes per pair (default; KW = 8 for narrower segments, see dtw_wide_plan)
constexpr int NTW = 128;   // threads per CTA
constexpr int kWChunk = 32;

template <int P>
__device__ __forceinline__ float wcell(float m, float t) {
    if constexpr (P == 1) return m + fabsf(t);
    else if constexpr (P == 0) return fmaxf(m, fabsf(t));  // DTW_inf
    else if constexpr (P == 4) { const float t2 = t * t; return fmaf(t2, t2, m); }  // DTW_4
    else return fmaf(t, t, m);
}

// in-band cells of rows 0 .. r-1 (see dtw.cu band_cells)
__device__ __forceinline__ unsigned long long wband_cells(int r, int n, int w) {
    const long long m = r < w ? r : w;
    const long long a0 = n - w;
    const long long tt = r > a0 ? r - a0 : 0;
    return (unsigned long long)((long long)r * (2 * w + 1) - (m * w - m * (m - 1) / 2) - tt * (tt + 1) / 2);
}

// COL = false: band coordinates (cell e of lane t = band position d = tS + e, column r - w + d);
//      true : column coordinates (cell e of lane t = column tS + e), w >= n - 1 only.
// yp: padded query rows [rows][LPW], yp[u] = y[u - padL] (+inf outside [0, n)).
template <int S>
constexpr int wide_min_blocks() { return S <= 25 ? 5 : (S <= 32 ? 4 : 2); }  // (S = 25: 128 registers, 16 warps per SM)
// lanes t == 0 of every group of KW lanes
template <int KW>
__host__ __device__ constexpr unsigned group_leads() { return KW == 8 ? 0x01010101u : 0x11111111u; }

template <int KW, int S, int P, bool WALK, bool COL>
__global__ void __launch_bounds__(NTW, wide_min_blocks<S>())
dtw_wide_kernel(DtwArgs a, const float *__restrict__ yp, int LPW, int padL) {
    static_assert(KW == 4 || KW == 8, "lanes per pair");
    constexpr int NY = COL ? S : S + 3;
    const int lane = threadIdx.x & 31, t = lane & (KW - 1);
    const unsigned FULL = 0xffffffffu;
    const int n = a.n, w = a.w, NB = 2 * w + 1;
    const int64_t total = (WALK && a.dev_total) ? (int64_t)*a.dev_total : a.total;
    // band mode: lane KW-1 holds M = KW*S - NB invalid cells at its top positions (0 <= M < KW);
    // they are reset to +inf after every row so they never feed a valid cell
    const int M = COL ? 0 : KW * S - NB;
    const int mfirst = (!COL && t == KW - 1) ? S - M : S;  // first invalid cell of this lane
    // cell holding D(n-1, n-1): band position w, or column n-1
    const int dfin = COL ? n - 1 : w;
    const int tfin = dfin / S, efin = dfin - tfin * S;

    bool busy = false;
    int s0 = 0;
    uint32_t cand = 0;
    int qy = 0;
    int64_t item = 0;
    float thr = kInf;
    const float *xr = nullptr, *yr = nullptr;
    float B[S], Y[NY], xc[4], xn[4], yn[4];
    // column coordinates: the rows alternate between B and B2 (cell e reads the previous row's
    // e-1 and e after its left neighbour overwrote e-1: in place, every cell would cost a move)
    float B2[COL ? S : 1];
    float res_hold = kInf;  // COL: the result cell D(n-1, n-1), captured when its row is computed
    // cascading abandon (readings c15, c19; as dtw4_kernel): rest = LB_Keogh^p terms of the rows
    // not yet computed = beta1 (from the gate slot) minus the terms of the rows lane 0 of the
    // group has computed; rest_snap = its value after the checkpoint row (r & 7 == 7)
    const bool casc = WALK && (a.b1 != nullptr || a.b1h != nullptr);
    float rest = 0.f, rest_snap = 0.f, u_nx = 0.f, l_nx = 0.f;  // (U, L of lane 0's next row)
    const float *ur = nullptr, *lr = nullptr;
    float left_in = kInf, diag_in = kInf, segmin = kInf;
    unsigned long long n_cells = 0;
    unsigned n_started = 0, n_abandon = 0;
    int64_t wcur = 0, wend = 0;
    bool more_items = true;

    for (int s = 0;; s += 4) {
        // ---------------- refill (phase 0 of 8): free groups start new pairs at s0 = s
        if ((s & 7) == 0) {
            while (true) {
                const unsigned needm = __ballot_sync(FULL, t == 0 && !busy) & group_leads<KW>();
                if (!needm || !more_items) break;
                if (wcur >= wend) {
                    int64_t base = 0;
                    if (lane == 0) base = (int64_t)atomicAdd(a.queue, (unsigned)kWChunk);
                    base = __shfl_sync(FULL, base, 0);
                    if (base >= total) { more_items = false; break; }
                    wcur = base;
                    wend = base + kWChunk < total ? base + kWChunk : total;
                }
                const int rank = __popc(needm & ((1u << (lane & ~(KW - 1))) - 1u));
                const int take = __popc(needm);
                const int64_t mine = wcur + rank;
                const bool got = !busy && mine < wend;
                wcur = wcur + take < wend ? wcur + take : wend;
                if (got) {
                    item = mine;
                    float beta = 0.f;
                    if constexpr (WALK) {
                        int lo = 0, hi = a.Qb;  // item_off[lo] <= item < item_off[hi]
                        while (hi - lo > 1) {
                            const int mid = (lo + hi) >> 1;
                            if (a.item_off[mid] <= item) lo = mid; else hi = mid;
                        }
                        qy = lo;
                        const int64_t j = a.pos[qy] + (item - a.item_off[qy]);
                        const unsigned long long key = a.list[list_base(a.loff, a.cap, qy) + j];
                        cand = (uint32_t)(key & 0xffffffffu);
                        beta = key_bound(key);
                        thr = *reinterpret_cast<volatile float *>(a.thr + qy);
                        xr = a.db + (int64_t)cand * n;
                        yr = yp + (int64_t)qy * LPW;
                        if (casc) {
                            const int64_t gi = (int64_t)qy * a.ldb + cand;
                            rest = fabsf(a.b1 ? __ldg(a.b1 + gi) : __half2float(a.b1h[gi]));
                            rest_snap = rest;
                            ur = a.Uq + (int64_t)qy * n;
                            lr = a.Lq + (int64_t)qy * n;
                            u_nx = __ldg(ur);  // row 0 (lane 0 starts there)
                            l_nx = __ldg(lr);
                        }
                    } else {
                        cand = (uint32_t)item;
                        thr = kInf;
                        xr = a.db + item * n;
                        yr = yp + item * LPW;
                    }
                    if (!(beta > thr)) {  // (WALK: else pruned by its bound before any cell)
                        busy = true;
                        s0 = s;
                        ++n_started;
                        // row -1: D(-1, -1) = 0 (band position w), everything else +inf
#pragma unroll
                        for (int e = 0; e < S; ++e) B[e] = (!COL && t * S + e == w) ? 0.f : kInf;
                        left_in = kInf;
                        diag_in = (COL && t == 0) ? 0.f : kInf;
                        segmin = kInf;
                        const int rb = -t;  // first block's first row of this lane
                        if constexpr (COL) {
#pragma unroll
                            for (int e = 0; e < S; ++e) Y[e] = yr[padL + t * S + e];
                        } else {
                            // window of the block BEFORE the first (the block start shifts it)
#pragma unroll
                            for (int k = 4; k < NY; ++k) Y[k] = yr[padL + rb - 4 - w + t * S + k];
#pragma unroll
                            for (int k = 0; k < 4; ++k) yn[k] = yr[padL + rb - w + t * S + S - 1 + k];
                        }
#pragma unroll
                        for (int k = 0; k < 4; ++k) xn[k] = (rb + k >= 0 && rb + k < n) ? __ldg(xr + rb + k) : 0.f;
                    } else if constexpr (!WALK) {
                        a.res[item] = kInf;
                    }
                }
            }
            if (!__any_sync(FULL, busy)) {
                if (!more_items) break;
                continue;
            }
        }
        // ---------------- block start: rows rb .. rb+3 of this lane
        const int rb = s - s0 - t;
        if (busy) {
            if constexpr (!COL) {
#pragma unroll
                for (int k = 0; k < S - 1; ++k) Y[k] = Y[k + 4];
#pragma unroll
                for (int k = 0; k < 4; ++k) Y[S - 1 + k] = yn[k];
#pragma unroll
                for (int k = 0; k < 4; ++k) yn[k] = yr[padL + rb + 4 - w + t * S + S - 1 + k];
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) xc[k] = xn[k];
#pragma unroll
            for (int k = 0; k < 4; ++k) xn[k] = (rb + 4 + k >= 0 && rb + 4 + k < n) ? __ldg(xr + rb + 4 + k) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int r = rb + u;
            const bool active = busy && r >= 0 && r < n;
            if constexpr (COL) {
                auto col_row = [&](float (&Bi)[COL ? S : 1], float (&Bo)[COL ? S : 1]) {
                    // computed unconditionally (no divergent merge, hence no moves): a lane's rows
                    // before row 0 see +inf everywhere and stay +inf (the start state), rows after
                    // n-1 are garbage -- the result cell is captured at row n-1 -- and idle lanes
                    // are re-initialised at their refill
                    float dg = diag_in, lf = left_in;
#pragma unroll
                    for (int e = 0; e < S; ++e) {
                        const float up = Bi[e];
                        const float v = wcell<P>(min3f(dg, up, lf), xc[u] - Y[e]);
                        dg = up;
                        lf = v;
                        Bo[e] = v;
                    }
                    if (WALK && active && (r & 7) == 7) {
                        float m = Bo[0];
#pragma unroll
                        for (int e = 1; e + 1 < S; e += 2) m = min3f(m, Bo[e], Bo[e + 1]);
                        if ((S & 1) == 0) m = fminf(m, Bo[S - 1]);
                        segmin = m;
                    }
                    if (busy && r == n - 1 && t == tfin) {
#pragma unroll
                        for (int e = 0; e < S; ++e)
                            if (e == efin) res_hold = Bo[e];
                    }
                    float recv = __shfl_up_sync(FULL, Bo[S - 1], 1, KW);
                    if (t == 0) recv = kInf;
                    diag_in = left_in;
                    left_in = recv;
                };
                if (u & 1) col_row(B2, B);  // (u is a constant of the unrolled loop)
                else col_row(B, B2);
            } else {
                float v0 = B[0];
                if (active) {
                    v0 = wcell<P>(min3f(B[0], B[1], left_in), xc[u] - Y[u]);
                    B[0] = v0;
                }
                float upl = __shfl_down_sync(FULL, v0, 1, KW);
                if (t == KW - 1) upl = kInf;
                if (active) {
                    float prev = v0;
#pragma unroll
                    for (int e = 1; e < S - 1; ++e) {
                        const float v = wcell<P>(min3f(B[e], B[e + 1], prev), xc[u] - Y[e + u]);
                        B[e] = v;
                        prev = v;
                    }
                    B[S - 1] = wcell<P>(min3f(B[S - 1], upl, prev), xc[u] - Y[S - 1 + u]);
#pragma unroll
                    for (int e = (S > KW - 1 ? S - (KW - 1) : 0); e < S; ++e)
                        if (e >= mfirst) B[e] = kInf;
                    if (WALK && (r & 7) == 7) {
                        float m = B[0];
#pragma unroll
                        for (int e = 1; e + 1 < S; e += 2) m = min3f(m, B[e], B[e + 1]);
                        if ((S & 1) == 0) m = fminf(m, B[S - 1]);
                        segmin = m;
                    }
                }
                float recv = __shfl_up_sync(FULL, B[S - 1], 1, KW);
                if (t == 0) recv = kInf;
                left_in = recv;
            }
            if (casc && t == 0 && active) {
                const float uu = u_nx, ll = l_nx;
                if (r + 1 < n) {  // the next row's envelope, loaded a row (a 51-cell chain) ahead
                    u_nx = __ldg(ur + r + 1);
                    l_nx = __ldg(lr + r + 1);
                }
                const float d = max3f(xc[u] - uu, ll - xc[u], 0.f);
                rest -= P == 1 ? d : (P == 4 ? (d * d) * (d * d) : d * d);
                if ((r & 7) == 7) rest_snap = rest;
            }
            const int ph = s + u - s0;  // group phase (uniform in the group)
            // ---- completion: the last lane finished row n-1 (the shuffles run warp-uniformly:
            //      every lane enters when any group completes)
            const bool done = busy && ph == n - 1 + KW - 1;
            if (__any_sync(FULL, done)) {
                float res = kInf;
#pragma unroll
                for (int e = 0; e < S; ++e)
                    if (t == tfin && e == efin) res = COL ? res_hold : B[e];
#pragma unroll
                for (int o = 1; o < KW; o <<= 1) res = fminf(res, __shfl_xor_sync(FULL, res, o, KW));
                if (done && t == 0) {
                    n_cells += wband_cells(n, n, w);
                    if constexpr (WALK) {
                        if (res <= thr) {
                            const unsigned pos = atomicAdd(a.rcount, 1u);
                            DCHECK(pos < a.rcap, "wide result buffer overflow pos=%u", pos);
                            a.rkey[pos] = pack_key(res, cand);
                            a.rq[pos] = qy;
                        }
                    } else {
                        a.res[item] = rootp<P>(res);
                    }
                }
                if (done) busy = false;
            }
            // ---- exact early abandon (reading c15): checkpoint row 8m+7 complete in all lanes
            if constexpr (WALK) {
                if (((s + u) & 7) == ((KW + 6) & 7)) {  // (uniform: every group's s0 is a multiple of 8)
                    float m = segmin;
#pragma unroll
                    for (int o = 1; o < KW; o <<= 1) m = fminf(m, __shfl_xor_sync(FULL, m, o, KW));
                    // + the LB_Keogh terms of the rows after the checkpoint row (lane 0's snapshot)
                    if (casc) m += fmaxf(__shfl_sync(FULL, rest_snap, lane & ~(KW - 1)), 0.f);
                    if (busy && ph >= KW + 6) {
                        thr = fminf(thr, *reinterpret_cast<volatile float *>(a.thr + qy));
                        if (!a.no_abandon && m > thr) {
                            if (t == 0) {
                                ++n_abandon;
                                n_cells += wband_cells(ph - KW + 2, n, w);  // rows 0 .. ph-KW+1 done
                            }
                            busy = false;
                        }
                    }
                }
            }
        }
    }
    if (a.cells) {
        unsigned long long c = n_cells;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
        if (lane == 0 && c) atomicAdd(a.cells, c);
    }
    if (a.started) {
        unsigned c = t == 0 ? n_started : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
        if (lane == 0 && c) atomicAdd(a.started, (unsigned long long)c);
    }
    if (a.abandoned) {
        unsigned c = n_abandon;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
        if (lane == 0 && c) atomicAdd(a.abandoned, (unsigned long long)c);
    }
}

__global__ void build_ywide_kernel(const float *__restrict__ y, int64_t rows, int n, float *__restrict__ yp,
                                   int LPW, int padL) {
    const int64_t total = rows * (int64_t)LPW;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / LPW;
        const int j = (int)(t - r * LPW) - padL;
        yp[t] = (j >= 0 && j < n) ? y[r * n + j] : kInf;
    }
}

template <int KW, int S, int P, bool WALK, bool COL>
int launch_wide_t(const DtwArgs &a, const float *yp, int LPW, int padL, cudaStream_t st) {
    DTWLB_CUDA(cudaMemsetAsync(a.queue, 0, sizeof(unsigned), st));
    int dev = 0, nsm = 148;
    DTWLB_CUDA(cudaGetDevice(&dev));
    DTWLB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    // enough warps to hold every pair of the round (32 / KW per warp), at most the CTAs that are
    // resident at once (register-limited: 4 per SM at S = 25, more than the launch bound's minimum)
    auto kern = dtw_wide_kernel<KW, S, P, WALK, COL>;
    static int resident = 0;
    if (resident == 0) {
        int nb = 0;
        DTWLB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, NTW, 0));
        resident = std::max(nb, 1);
    }
    const int64_t warps = std::min<int64_t>(ceil_div(std::max<int64_t>(a.total, 1), 32 / KW),
                                            (int64_t)nsm * (NTW / 32) * resident);
    const int64_t grid = ceil_div(warps * 32, NTW);
    kern<<<(unsigned)grid, NTW, 0, st>>>(a, yp, LPW, padL);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

template <int P, bool WALK>
int launch_wide_p(const DtwArgs &a, const float *yp, int LPW, int padL, int mode, int S, int KW, cudaStream_t st) {
    if (mode == 1) {  // column coordinates (w >= n - 1)
        if (KW == 8) {
            switch (S) {
                case 13: return launch_wide_t<8, 13, P, WALK, true>(a, yp, LPW, padL, st);
                case 16: return launch_wide_t<8, 16, P, WALK, true>(a, yp, LPW, padL, st);
                case 32: return launch_wide_t<8, 32, P, WALK, true>(a, yp, LPW, padL, st);
            }
        } else {
            switch (S) {
                case 16: return launch_wide_t<4, 16, P, WALK, true>(a, yp, LPW, padL, st);
                case 25: return launch_wide_t<4, 25, P, WALK, true>(a, yp, LPW, padL, st);
                case 32: return launch_wide_t<4, 32, P, WALK, true>(a, yp, LPW, padL, st);
                case 48: return launch_wide_t<4, 48, P, WALK, true>(a, yp, LPW, padL, st);
                case 64: return launch_wide_t<4, 64, P, WALK, true>(a, yp, LPW, padL, st);
            }
        }
    } else {
        if (KW == 8 && S == 26) return launch_wide_t<8, 26, P, WALK, false>(a, yp, LPW, padL, st);
        if (KW == 4 && S == 51) return launch_wide_t<4, 51, P, WALK, false>(a, yp, LPW, padL, st);
    }
    set_error(DTWLB_EINVAL, "internal: no wide DTW kernel for KW = %d, S = %d", KW, S);
    return DTWLB_EINVAL;
}

// Lanes per pair KW and segment length S for (n, w): mode 1 = column coordinates (w >= n-1,
// n <= 256), mode 2 = band coordinates (w = 100, 101); 0 = none (generic kernel).  KW = 4 lanes
// per pair; DTWLB_WIDE_KW=8 halves each lane's serial cell chain and its registers (more warps
// resident) but measured slower: C3 w = 100 DTW 56.0 vs 44.8 ms, Appendix B 2.64 vs 2.89 10^12
// cells/s (profiles/r02o_wide_kw.txt) -- twice the shuffles per cell and a 7-row pipeline skew.
int wide_plan(int n, int w, int *S_out, int *KW_out) {
    static const int env_kw = [] { const char *e = getenv("DTWLB_WIDE_KW"); return e ? atoi(e) : 0; }();
    const int KW = env_kw == 8 ? 8 : 4;
    *KW_out = KW;
    if (w >= n - 1 && n <= 256) {
        const int need = (n + KW - 1) / KW;
        const int o8[] = {13, 16, 32}, o4[] = {16, 25, 32, 48, 64};
        const int *opts = KW == 8 ? o8 : o4;
        const int nopt = KW == 8 ? 3 : 5;
        for (int i = 0; i < nopt; ++i)
            if (opts[i] >= need) { *S_out = opts[i]; return 1; }
    }
    const int S = (2 * w + 1 + KW - 1) / KW;
    if ((KW == 8 && S == 26) || (KW == 4 && S == 51)) { *S_out = S; return 2; }
    return 0;
}

}  // namespace

int dtw_wide_plan(int n, int w, int *S_out) {
    int KW = 0;
    return wide_plan(n, w, S_out, &KW);
}

int dtw_wide_padded(int n, int w, int S, int *padL) {
    int S2 = 0, KW = 4;
    wide_plan(n, w, &S2, &KW);
    *padL = (w + 8 + 3) / 4 * 4;
    return (*padL + n + KW * S + 16 + 3) / 4 * 4;
}

int launch_build_ywide(const float *y, int64_t rows, int n, float *yp, int LPW, int padL, cudaStream_t st) {
    if (rows == 0) return DTWLB_OK;
    const int64_t total = rows * (int64_t)LPW;
    const int grid = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 16);
    build_ywide_kernel<<<grid, 256, 0, st>>>(y, rows, n, yp, LPW, padL);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

int launch_dtw_wide(const DtwArgs &a, const float *yp, int LPW, int padL, int p, bool walk, cudaStream_t st) {
    int S = 0, KW = 4;
    const int mode = wide_plan(a.n, a.w, &S, &KW);
    if (mode == 0) {
        set_error(DTWLB_EINVAL, "internal: no wide DTW kernel for n = %d, w = %d", a.n, a.w);
        return DTWLB_EINVAL;
    }
    if (!a.queue) {
        set_error(DTWLB_EINVAL, "internal: the wide DTW kernel needs its work-queue counter");
        return DTWLB_EINVAL;
    }
    if (walk && !a.dev_total && a.total == 0) return DTWLB_OK;
    if (p == 0) {
        if (walk) {
            set_error(DTWLB_EUNSUPPORTED, "nn_search: p = infinity unsupported");
            return DTWLB_EUNSUPPORTED;
        }
        return launch_wide_p<0, false>(a, yp, LPW, padL, mode, S, KW, st);
    }
    if (p == 4) {
        if (walk) {
            set_error(DTWLB_EUNSUPPORTED, "nn_search: p = 4 unsupported");
            return DTWLB_EUNSUPPORTED;
        }
        return launch_wide_p<4, false>(a, yp, LPW, padL, mode, S, KW, st);
    }
    if (p == 1) return walk ? launch_wide_p<1, true>(a, yp, LPW, padL, mode, S, KW, st)
                            : launch_wide_p<1, false>(a, yp, LPW, padL, mode, S, KW, st);
    return walk ? launch_wide_p<2, true>(a, yp, LPW, padL, mode, S, KW, st)
                : launch_wide_p<2, false>(a, yp, LPW, padL, mode, S, KW, st);
}

}  // namespace dtwlb
