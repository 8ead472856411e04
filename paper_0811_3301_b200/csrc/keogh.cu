// keogh.cu -- the LB_Keogh pass (a2): Alg. 2/3 lines P:507-514 / P:589-597.
//
//   beta1(q, c) = sum_i d(x_c,i, [L_q,i, U_q,i])^p,  d(v,[a,b]) = max(v - b, a - v, 0)
//
// Design (B200): every (query, candidate) pair of a query-block x database-tile
// is evaluated; the pass is structurally an outer product reduced over i with
// a non-bilinear inner op (no tensor-core contraction), so it is register-tiled
// SIMT: a 256-thread CTA owns 64 queries x 128 candidates, each thread a 4x8
// pair tile.  Chunks of 32 samples of the envelopes U, L and of the candidate
// rows are staged in shared memory with cp.async (double-buffered), read back
// as 128-bit vectors, and each loaded value is reused 8x (envelope) or 4x
// (candidate) from registers.  Per pair-element: FADD, FADD, FMNMX3, FADD|FFMA
// (d = max(x - U, L - x, 0); 3 FMA-pipe ops + 1 half-rate ALU op, issue-bound).
// Per-chunk partial sums are folded into the total at each chunk end (two-level
// summation keeps the fp32 error at ~(32 + n/32) ulp instead of n ulp).
// CTAs are ordered query-tile-fastest so each database tile is fetched from
// HBM once and served from L2 to every query tile; the envelopes of the whole
// query block stay L2-resident.  The i-tail beyond n is zero-filled on both
// sides, which contributes max(0-0, 0-0, 0) = 0.
//
// The same tile kernel evaluates the piecewise-sum pre-filter over
// segment sums (PAA = true): D = n/8 "samples" per row, directed rounding (the forward
// term alone: the C-ABI lb_piecewise).  nn_search's symmetric gate -- the max of this
// forward term and the REVERSE term, the query's segment sums against the candidate's
// envelope sums, sum_j d(P(y)_j, [P(L(x))_j, P(U(x))_j])^p, a lower bound of
// LB_Keogh_p(y, x) <= DTW_p(y, x) = DTW_p(x, y) (symmetry; DESIGN.md reading
// c20) -- is gate_sym_kernel below.
#include <cfloat>
#include <cstdlib>

#include <cuda_fp16.h>

#include "kernels.cuh"

namespace dtwlb {

namespace {

constexpr int TQ = 64, TC = 128, KC = 32, KP = KC + 4;  // KP: padded pitch (floats)
constexpr int NT = 256;

template <bool PAA>
struct Stage {  // chunk of the operands, written by cp.async (double-buffered)
    float X[TC][KP];           // candidate rows (LB_Keogh) or their lower sums (PAA)
    float X2[PAA ? TC : 1][KP];  // PAA: upper sums of the candidate segments
    float U[TQ][KP];
    float L[TQ][KP];
};
// Stage chunk [k0, k0+KC) of rows r0.. of a [rows][n] matrix into S[R][KP].
template <int R, bool VEC>
__device__ __forceinline__ void stage_rows(float (*S)[KP], const float *__restrict__ g, int64_t r0,
                                           int64_t rows, int n, int k0) {
    if constexpr (VEC) {
        // R rows x 8 vectors of 16 B
        for (int t = threadIdx.x; t < R * (KC / 4); t += NT) {
            int r = t >> 3, v = t & 7;
            int64_t row = r0 + r;
            int k = k0 + v * 4;
            bool ok = row < rows && k < n;  // n % 4 == 0 here, so a vector is all-in or all-out
            const float *src = ok ? g + row * (int64_t)n + k : g;
            cp_async16(&S[r][v * 4], src, ok ? 16 : 0);
        }
    } else {
        for (int t = threadIdx.x; t < R * KC; t += NT) {
            int r = t / KC, v = t - r * KC;
            int64_t row = r0 + r;
            int k = k0 + v;
            bool ok = row < rows && k < n;
            const float *src = ok ? g + row * (int64_t)n + k : g;
            cp_async4(&S[r][v], src, ok ? 4 : 0);
        }
    }
}

// PAA = false: LB_Keogh^p, d = max(x - U, L - x, 0), FADD, FADD, FMNMX3, FADD|FFMA.
// PAA = true:  piecewise-sum bound over segment sums with directed rounding:
//   d = max(Xlo - Uhi, Llo - Xhi, 0) (rounded down), acc += d^p (rounded down), so the
//   result never exceeds the exact sum_j d(X_j, [L_j, U_j])^p; same 4 ops per element.
// Two elements at once: the four subtractions are two packed FADD2 (sm_100 f32x2, per
// component the same IEEE operation as FADD / FADD.RM), then FMNMX3 and the accumulation
// per element: 3 issue slots per element instead of 4.
template <int P, bool PAA>
__device__ __forceinline__ float lb_elem2(float acc, float2 xl, float2 xh, float2 u, float2 l) {
    float2 a, b;
    if constexpr (PAA) {
        a = __fadd2_rd(xl, make_float2(-u.x, -u.y));
        b = __fadd2_rd(l, make_float2(-xh.x, -xh.y));
    } else {
        a = __fadd2_rn(xl, make_float2(-u.x, -u.y));
        b = __fadd2_rn(l, make_float2(-xh.x, -xh.y));
    }
    const float d0 = max3f(a.x, b.x, 0.f), d1 = max3f(a.y, b.y, 0.f);
    if constexpr (PAA) {
        if constexpr (P == 1) return __fadd_rd(__fadd_rd(acc, d0), d1);
        else return __fmaf_rd(d1, d1, __fmaf_rd(d0, d0, acc));
    } else {
        return accp<P>(accp<P>(acc, d0), d1);
    }
}

template <int P, bool PAA>
__device__ __forceinline__ float lb_elem(float acc, float xl, float xh, float u, float l) {
    if constexpr (PAA) {
        const float d = max3f(__fsub_rd(xl, u), __fsub_rd(l, xh), 0.f);
        if constexpr (P == 1) return __fadd_rd(acc, d);
        else return __fmaf_rd(d, d, acc);
    } else {
        return accp<P>(acc, max3f(xl - u, l - xl, 0.f));
    }
}

template <int P, bool VEC, bool ROOTED, bool PAA>
__global__ void __launch_bounds__(NT, 2)
keogh_tile_kernel(const float *__restrict__ U, const float *__restrict__ L, const float *__restrict__ db,
                  const float *__restrict__ db2, int64_t Q, int64_t N, int n, void *__restrict__ out,
                  int64_t ldo, int nqt) {
    extern __shared__ __align__(16) unsigned char smraw[];
    Stage<PAA> *st = reinterpret_cast<Stage<PAA> *>(smraw);

    const int64_t tile = blockIdx.x;
    const int64_t q0 = (tile % nqt) * TQ;
    const int64_t c0 = (tile / nqt) * TC;
    const int tid = threadIdx.x;
    const int cg = tid & 15;  // candidates c0 + cg + 16 j, j < 8
    const int qg = tid >> 4;  // queries   q0 + 4 qg + r, r < 4

    float acc[4][8];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[r][j] = 0.f;

    const int nchunks = (n + KC - 1) / KC;
    stage_rows<TC, VEC>(st[0].X, db, c0, N, n, 0);
    if constexpr (PAA) stage_rows<TC, VEC>(st[0].X2, db2, c0, N, n, 0);
    stage_rows<TQ, VEC>(st[0].U, U, q0, Q, n, 0);
    stage_rows<TQ, VEC>(st[0].L, L, q0, Q, n, 0);
    cp_commit();

    for (int ch = 0; ch < nchunks; ++ch) {
        if (ch + 1 < nchunks) {
            Stage<PAA> &nx = st[(ch + 1) & 1];
            stage_rows<TC, VEC>(nx.X, db, c0, N, n, (ch + 1) * KC);
            if constexpr (PAA) stage_rows<TC, VEC>(nx.X2, db2, c0, N, n, (ch + 1) * KC);
            stage_rows<TQ, VEC>(nx.U, U, q0, Q, n, (ch + 1) * KC);
            stage_rows<TQ, VEC>(nx.L, L, q0, Q, n, (ch + 1) * KC);
        }
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        const Stage<PAA> &s = st[ch & 1];
        // LB_Keogh: per-chunk partial sums (two-level summation); PAA: accumulate directly
        // (rounded down, so any order stays a lower bound; frees 32 registers for the
        // packed subtractions)
        float part[PAA ? 1 : 4][PAA ? 1 : 8];
        if constexpr (!PAA) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int j = 0; j < 8; ++j) part[r][j] = 0.f;
        }

#pragma unroll 2
        for (int k = 0; k < KC; k += 4) {
            float4 uv[4], lv[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                uv[r] = *reinterpret_cast<const float4 *>(&s.U[4 * qg + r][k]);
                lv[r] = *reinterpret_cast<const float4 *>(&s.L[4 * qg + r][k]);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float4 xv = *reinterpret_cast<const float4 *>(&s.X[cg + 16 * j][k]);
                float4 xw = xv;
                if constexpr (PAA) xw = *reinterpret_cast<const float4 *>(&s.X2[cg + 16 * j][k]);
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if constexpr (PAA) {
                        float t = acc[r][j];
                        t = lb_elem2<P, PAA>(t, make_float2(xv.x, xv.y), make_float2(xw.x, xw.y),
                                             make_float2(uv[r].x, uv[r].y), make_float2(lv[r].x, lv[r].y));
                        t = lb_elem2<P, PAA>(t, make_float2(xv.z, xv.w), make_float2(xw.z, xw.w),
                                             make_float2(uv[r].z, uv[r].w), make_float2(lv[r].z, lv[r].w));
                        acc[r][j] = t;
                    } else {
                        float t = part[r][j];
                        t = lb_elem<P, PAA>(t, xv.x, xw.x, uv[r].x, lv[r].x);
                        t = lb_elem<P, PAA>(t, xv.y, xw.y, uv[r].y, lv[r].y);
                        t = lb_elem<P, PAA>(t, xv.z, xw.z, uv[r].z, lv[r].z);
                        t = lb_elem<P, PAA>(t, xv.w, xw.w, uv[r].w, lv[r].w);
                        part[r][j] = t;
                    }
                }
            }
        }
        if constexpr (!PAA) {
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[r][j] += part[r][j];
        }
        __syncthreads();
    }

#pragma unroll
    for (int r = 0; r < 4; ++r) {
        int64_t q = q0 + 4 * qg + r;
        if (q >= Q) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            int64_t c = c0 + cg + 16 * j;
            if (c >= N) continue;
            float v = acc[r][j];
            if constexpr (PAA) {
                // Cauchy-Schwarz per segment: sum_{i in C_j} d_i^2 >= (sum d_i)^2 / |C_j| >= D_j^2 / s
                if constexpr (P == 2) v = __fmul_rd(v, 1.0f / kSeg);
                if constexpr (ROOTED) v = P == 1 ? v : __fsqrt_rd(v);
            } else if constexpr (ROOTED) {
                v = rootp<P>(v);
            }
            if constexpr (PAA && !ROOTED) {  // nn_search's gate block: fp16, rounded down (still a lower bound)
                __half *o = reinterpret_cast<__half *>(out) + q * ldo + c;
                const __half h = __float2half_rd(v);
                *o = h;
            } else {
                float *o = reinterpret_cast<float *>(out) + q * ldo + c;
                *o = v;
            }
        }
    }
}

template <int P, bool VEC, bool ROOTED, bool PAA>
int launch_tile_t(const float *U, const float *L, const float *db, const float *db2, int64_t Q, int64_t N,
                  int n, void *out, int64_t ldo, cudaStream_t st) {
    const size_t smem = 2 * sizeof(Stage<PAA>);
    auto k = keogh_tile_kernel<P, VEC, ROOTED, PAA>;
    DTWLB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t nqt = ceil_div(Q, TQ), nct = ceil_div(N, TC);
    const int64_t tiles = nqt * nct;
    if (tiles > 0x7fffffffLL) {
        set_error(DTWLB_EINVAL, "bound pass: problem too large (%lld tiles)", (long long)tiles);
        return DTWLB_EINVAL;
    }
    k<<<(unsigned)tiles, NT, smem, st>>>(U, L, db, db2, Q, N, n, out, ldo, (int)nqt);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

template <bool PAA>
int launch_tile(const float *U, const float *L, const float *db, const float *db2, int64_t Q, int64_t N, int n,
                int p, bool rooted, void *out, int64_t ldo, cudaStream_t st) {
    if (Q == 0 || N == 0) return DTWLB_OK;
    const bool vec = (n % 4 == 0) && ((reinterpret_cast<uintptr_t>(U) | reinterpret_cast<uintptr_t>(L) |
                                       reinterpret_cast<uintptr_t>(db) | reinterpret_cast<uintptr_t>(db2)) %
                                      16 == 0);
#define DTWLB_K(P_, V_, R_) return launch_tile_t<P_, V_, R_, PAA>(U, L, db, db2, Q, N, n, out, ldo, st)
    if (p == 1) {
        if (vec) { if (rooted) DTWLB_K(1, true, true); else DTWLB_K(1, true, false); }
        else { if (rooted) DTWLB_K(1, false, true); else DTWLB_K(1, false, false); }
    } else {
        if (vec) { if (rooted) DTWLB_K(2, true, true); else DTWLB_K(2, true, false); }
        else { if (rooted) DTWLB_K(2, false, true); else DTWLB_K(2, false, false); }
    }
#undef DTWLB_K
}

// ---------------------------------------------------------------- fused symmetric gate
// Both terms of the symmetric piecewise-sum gate (readings c18, c20) in ONE tile pass: per
// (query, candidate) pair the forward term (candidate sums against the query's envelope sums)
// and the reverse term (query sums against the candidate's envelope sums) accumulate in two
// register tiles and the maximum is written once -- instead of a forward launch writing the
// fp16 gate block and a reverse launch reading it back (a read-modify-write of the whole block
// whose load stalled the reverse epilogue).  With Dp <= 32 (n <= 256) the single chunk is staged
// once (one 110 KB stage: 2 CTAs per SM).
//
// Midpoint form (4 full-rate FADD/FFMA per element instead of FADD2 + FMNMX3 + FFMA, which
// issue at half rate: 4.4 vs 5.3 cycles per element, profiles/r02h_isa_probe.txt).  Every
// operand is an interval in midpoint-radius form, outward-rounded by paa_mid_kernel: a point
// sum X_j lies in [m - r, m + r] (r ~ 1 ulp) and a box [P(L)_j, P(U)_j] inside [m - r, m + r].
// The distance of a point of the first to the second is >= |m_x - m_b| - (r_x + r_b), so
//   d_j >= max(|m_x - m_b| - R, 0),  R = r_b + max over the CTA's point intervals of r_x
// (the point radii are ~1 ulp: the tile maximum, taken per segment in shared memory, loosens
// the bound by ~1e-6 and leaves one radius per element).  Per element, rounded so the fp32
// value never exceeds the exact one: t1 = m_x - m_b toward zero (|t1| <= |exact|), t2 = |t1| - R
// rounded down, t3 = t2 + |t2| = 2 max(t2, 0) (exact), acc += t3^p rounded down; the total is
// scaled by 2^-p (exact) -- the same bound as max(Xlo - Uhi, Llo - Xhi, 0), whose two terms are
// (t1 sign-split) |m_x - m_b| - R.  The three subtractions of two elements issue as three packed
// FADD2 (mid_elem2).
struct SymStage {
    float X[TC][KP], X2[TC][KP];    // candidate segment sums: midpoint, radius            (forward)
    float XR[TC][KP], XR2[TC][KP];  // candidate envelope boxes [P(L(x)), P(U(x))]: m, r   (reverse)
    float U[TQ][KP], L[TQ][KP];     // query envelope boxes [P(L(y)), P(U(y))]: m, r       (forward)
    float UR[TQ][KP], LR[TQ][KP];   // query segment sums: midpoint, radius                (reverse)
};

// Two elements per step: the three subtractions as packed FADD2 (per component the same IEEE
// operation, rounding mode and |.| / negation operand modifiers as FADD): 3 FADD2 + 2 FFMA = 5
// issue slots per two elements instead of 8 (the FP32 pipe still does 4 ops per element).
template <int P>
__device__ __forceinline__ float mid_elem2(float acc, float2 mx, float2 mb, float2 R) {
    const float2 t1 = __fadd2_rz(mx, make_float2(-mb.x, -mb.y));                      // |t1| <= |mx - mb|
    const float2 t2 = __fadd2_rd(make_float2(fabsf(t1.x), fabsf(t1.y)), make_float2(-R.x, -R.y));  // <= |mx - mb| - R
    const float2 t3 = __fadd2_rn(t2, make_float2(fabsf(t2.x), fabsf(t2.y)));           // 2 max(t2, 0), exact
    if constexpr (P == 1) return __fadd_rd(__fadd_rd(acc, t3.x), t3.y);
    else return __fmaf_rd(t3.y, t3.y, __fmaf_rd(t3.x, t3.x, acc));
}

template <int P, bool VEC, bool ROOTED>
__global__ void __launch_bounds__(NT, 2)
gate_sym_kernel(const float *__restrict__ Qm, const float *__restrict__ Qr, const float *__restrict__ Ym,
                const float *__restrict__ Yr, const float *__restrict__ Xm, const float *__restrict__ Xr,
                const float *__restrict__ Bm, const float *__restrict__ Br, int64_t Q, int64_t N, int n,
                void *__restrict__ out, int64_t ldo, int nqt) {
    extern __shared__ __align__(16) unsigned char smraw[];
    SymStage *st = reinterpret_cast<SymStage *>(smraw);
    __shared__ float red[2][8][KC];  // partial tile maxima of the point radii
    const int64_t tile = blockIdx.x;
    const int64_t q0 = (tile % nqt) * TQ;
    const int64_t c0 = (tile / nqt) * TC;
    const int tid = threadIdx.x;
    const int cg = tid & 15, qg = tid >> 4;
    float acc[4][8], accr[4][8];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int j = 0; j < 8; ++j) { acc[r][j] = 0.f; accr[r][j] = 0.f; }
    const int nchunks = (n + KC - 1) / KC;
    const int nbuf = nchunks > 1 ? 2 : 1;
    auto stage = [&](SymStage &S, int k0) {
        stage_rows<TC, VEC>(S.X, Xm, c0, N, n, k0);
        stage_rows<TC, VEC>(S.X2, Xr, c0, N, n, k0);
        stage_rows<TC, VEC>(S.XR, Bm, c0, N, n, k0);
        stage_rows<TC, VEC>(S.XR2, Br, c0, N, n, k0);
        stage_rows<TQ, VEC>(S.U, Qm, q0, Q, n, k0);
        stage_rows<TQ, VEC>(S.L, Qr, q0, Q, n, k0);
        stage_rows<TQ, VEC>(S.UR, Ym, q0, Q, n, k0);
        stage_rows<TQ, VEC>(S.LR, Yr, q0, Q, n, k0);
    };
    stage(st[0], 0);
    cp_commit();
    for (int ch = 0; ch < nchunks; ++ch) {
        if (ch + 1 < nchunks) stage(st[(ch + 1) % nbuf], (ch + 1) * KC);
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        SymStage &S = st[ch % nbuf];
        {   // per segment: the tile maxima of the point radii (128 candidates, 64 queries), added
            // to the other side's box radii (rounded up; FLT_MAX stays the "whole line" padding)
            const int k = tid & (KC - 1), part = tid >> 5;  // 8 parts
            float mc = 0.f, mq = 0.f;
#pragma unroll 4
            for (int c = part * (TC / 8); c < (part + 1) * (TC / 8); ++c) mc = fmaxf(mc, S.X2[c][k]);
#pragma unroll 4
            for (int q = part * (TQ / 8); q < (part + 1) * (TQ / 8); ++q) mq = fmaxf(mq, S.LR[q][k]);
            red[0][part][k] = mc;
            red[1][part][k] = mq;
            __syncthreads();
            mc = red[0][0][k];
            mq = red[1][0][k];
#pragma unroll
            for (int t = 1; t < 8; ++t) { mc = fmaxf(mc, red[0][t][k]); mq = fmaxf(mq, red[1][t][k]); }
            for (int q = part; q < TQ; q += 8) S.L[q][k] = fminf(__fadd_ru(S.L[q][k], mc), FLT_MAX);
            for (int c = part; c < TC; c += 8) S.XR2[c][k] = fminf(__fadd_ru(S.XR2[c][k], mq), FLT_MAX);
            __syncthreads();
        }
#pragma unroll 2
        for (int k = 0; k < KC; k += 4) {
            {   // forward: candidate sums against the query's envelope box
                float4 mv[4], rv[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    mv[r] = *reinterpret_cast<const float4 *>(&S.U[4 * qg + r][k]);
                    rv[r] = *reinterpret_cast<const float4 *>(&S.L[4 * qg + r][k]);
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float4 xv = *reinterpret_cast<const float4 *>(&S.X[cg + 16 * j][k]);
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        float t = acc[r][j];
                        t = mid_elem2<P>(t, make_float2(xv.x, xv.y), make_float2(mv[r].x, mv[r].y),
                                         make_float2(rv[r].x, rv[r].y));
                        t = mid_elem2<P>(t, make_float2(xv.z, xv.w), make_float2(mv[r].z, mv[r].w),
                                         make_float2(rv[r].z, rv[r].w));
                        acc[r][j] = t;
                    }
                }
            }
            {   // reverse: query sums against the candidate's envelope box
                float4 yv[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) yv[r] = *reinterpret_cast<const float4 *>(&S.UR[4 * qg + r][k]);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float4 bm = *reinterpret_cast<const float4 *>(&S.XR[cg + 16 * j][k]);
                    const float4 br = *reinterpret_cast<const float4 *>(&S.XR2[cg + 16 * j][k]);
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        float t = accr[r][j];
                        t = mid_elem2<P>(t, make_float2(yv[r].x, yv[r].y), make_float2(bm.x, bm.y),
                                         make_float2(br.x, br.y));
                        t = mid_elem2<P>(t, make_float2(yv[r].z, yv[r].w), make_float2(bm.z, bm.w),
                                         make_float2(br.z, br.w));
                        accr[r][j] = t;
                    }
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int64_t q = q0 + 4 * qg + r;
        if (q >= Q) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t c = c0 + cg + 16 * j;
            if (c >= N) continue;
            // max of two lower bounds (exact); the accumulators hold sums of (2 d)^p: scale by
            // 2^-p (exact), and by 1/s for p = 2 (reading c18)
            float v = fmaxf(acc[r][j], accr[r][j]);
            if constexpr (P == 2) v = __fmul_rd(v, 0.25f / kSeg);
            else v = v * 0.5f;
            if constexpr (ROOTED) {
                if constexpr (P == 2) v = __fsqrt_rd(v);
                reinterpret_cast<float *>(out)[q * ldo + c] = v;
            } else {
                reinterpret_cast<__half *>(out)[q * ldo + c] = __float2half_rd(v);
            }
        }
    }
}

template <int P, bool VEC, bool ROOTED>
int launch_sym_t(const float *Qm, const float *Qr, const float *Ym, const float *Yr, const float *Xm,
                 const float *Xr, const float *Bm, const float *Br, int64_t Q, int64_t N, int Dp, void *out,
                 int64_t ldo, cudaStream_t st) {
    const int nchunks = (Dp + KC - 1) / KC;
    const size_t smem = (nchunks > 1 ? 2 : 1) * sizeof(SymStage);
    auto k = gate_sym_kernel<P, VEC, ROOTED>;
    DTWLB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t nqt = ceil_div(Q, TQ), nct = ceil_div(N, TC);
    const int64_t tiles = nqt * nct;
    if (tiles > 0x7fffffffLL) {
        set_error(DTWLB_EINVAL, "bound pass: problem too large (%lld tiles)", (long long)tiles);
        return DTWLB_EINVAL;
    }
    k<<<(unsigned)tiles, NT, smem, st>>>(Qm, Qr, Ym, Yr, Xm, Xr, Bm, Br, Q, N, Dp, out, ldo, (int)nqt);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

// ---------------------------------------------------------------- piecewise sums
// One thread per (row, segment): directed fp64 sums of the s samples, then a directed
// conversion to fp32 (the interval [lo, hi] contains the exact sum).
__global__ void paa_sums_kernel(const float *__restrict__ x, int64_t count, int n, float *__restrict__ lo,
                                float *__restrict__ hi, float pad_lo, float pad_hi, bool lo_only_down) {
    const int D = paa_dims(n), Dp = paa_pitch(n);
    const int64_t total = count * Dp;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / Dp;
        const int j = (int)(t - r * Dp);
        if (j >= D) {
            if (lo) lo[t] = pad_lo;
            if (hi) hi[t] = pad_hi;
            continue;
        }
        const float *xr = x + r * n;
        const int i1 = min(n, (j + 1) * kSeg);
        double sd = 0.0, su = 0.0;
        for (int i = j * kSeg; i < i1; ++i) {
            const double v = (double)__ldg(xr + i);
            sd = __dadd_rd(sd, v);
            su = __dadd_ru(su, v);
        }
        if (lo) lo[t] = __double2float_rd(sd);
        if (hi) hi[t] = __double2float_ru(su);
    }
    (void)lo_only_down;
}

// Midpoint-radius form of the segment sums (the fused gate's operands): one thread per (row,
// segment); directed fp64 sums s_lo = sum(lo_src) rounded down, s_hi = sum(hi_src) rounded up
// (lo_src = hi_src = x: the point sum X_j in [s_lo, s_hi]; lo_src = L, hi_src = U: the box
// [P(L)_j, P(U)_j] inside [s_lo, s_hi]); m = fp32(nearest) of (s_lo + s_hi) / 2 and r = fp32
// (rounded up) of max(s_hi - m, m - s_lo), so [s_lo, s_hi] lies in [m - r, m + r].  Padding
// segments: m = 0, r = pad_r (0 for points, FLT_MAX for boxes: "the whole line", d = 0).
__global__ void paa_mid_kernel(const float *__restrict__ lo_src, const float *__restrict__ hi_src, int64_t count,
                               int n, float *__restrict__ m_out, float *__restrict__ r_out, float pad_r) {
    const int D = paa_dims(n), Dp = paa_pitch(n);
    const int64_t total = count * Dp;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / Dp;
        const int j = (int)(t - r * Dp);
        if (j >= D) {
            m_out[t] = 0.f;
            r_out[t] = pad_r;
            continue;
        }
        const float *lr = lo_src + r * n, *hr = hi_src + r * n;
        const int i1 = min(n, (j + 1) * kSeg);
        double sd = 0.0, su = 0.0;
        for (int i = j * kSeg; i < i1; ++i) {
            sd = __dadd_rd(sd, (double)__ldg(lr + i));
            su = __dadd_ru(su, (double)__ldg(hr + i));
        }
        const float m = __double2float_rn(0.5 * sd + 0.5 * su);  // (halving is exact)
        const double md = (double)m;
        const double rad = fmax(__dsub_ru(su, md), __dsub_ru(md, sd));
        m_out[t] = m;
        r_out[t] = fminf(__double2float_ru(rad), FLT_MAX);
    }
}

}  // namespace

int launch_paa_mid(const float *lo_src, const float *hi_src, int64_t count, int n, float *m, float *r, bool box,
                   cudaStream_t st) {
    if (count == 0) return DTWLB_OK;
    const int64_t total = count * paa_pitch(n);
    const int grid = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 16);
    paa_mid_kernel<<<grid, 256, 0, st>>>(lo_src, hi_src, count, n, m, r, box ? FLT_MAX : 0.f);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

int launch_paa_sums(const float *x, int64_t count, int n, float *lo, float *hi, cudaStream_t st) {
    if (count == 0) return DTWLB_OK;
    const int64_t total = count * paa_pitch(n);
    const int grid = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 16);
    paa_sums_kernel<<<grid, 256, 0, st>>>(x, count, n, lo, hi, 0.f, 0.f, false);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

int launch_paa_env_sums(const float *U, const float *L, int64_t count, int n, float *Uhi, float *Llo,
                        cudaStream_t st) {
    if (count == 0) return DTWLB_OK;
    const int64_t total = count * paa_pitch(n);
    const int grid = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 16);
    paa_sums_kernel<<<grid, 256, 0, st>>>(U, count, n, nullptr, Uhi, 0.f, kInf, false);
    DTWLB_LAUNCH_CHECK();
    paa_sums_kernel<<<grid, 256, 0, st>>>(L, count, n, Llo, nullptr, -kInf, 0.f, false);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

int launch_paa_bound(const float *Uhi, const float *Llo, const float *Xlo, const float *Xhi, int64_t Q,
                     int64_t N, int n, int p, bool rooted, void *out, int64_t ldo, cudaStream_t st) {
    return launch_tile<true>(Uhi, Llo, Xlo, Xhi, Q, N, paa_pitch(n), p, rooted, out, ldo, st);
}

int launch_paa_bound_sym(const float *Qm, const float *Qr, const float *Ym, const float *Yr, const float *Xm,
                         const float *Xr, const float *Bm, const float *Br, int64_t Q, int64_t N, int n, int p,
                         bool rooted, void *out, int64_t ldo, cudaStream_t st) {
    if (Q == 0 || N == 0) return DTWLB_OK;
    const int Dp = paa_pitch(n);  // a multiple of 4: 16-byte rows
#define DTWLB_S(P_, R_) return launch_sym_t<P_, true, R_>(Qm, Qr, Ym, Yr, Xm, Xr, Bm, Br, Q, N, Dp, out, ldo, st)
    if (p == 1) { if (rooted) DTWLB_S(1, true); else DTWLB_S(1, false); }
    else { if (rooted) DTWLB_S(2, true); else DTWLB_S(2, false); }
#undef DTWLB_S
}

int launch_keogh(const float *U, const float *L, const float *db, int64_t Q, int64_t N, int n, int p,
                 bool rooted, float *out, int64_t ldo, cudaStream_t st) {
    return launch_tile<false>(U, L, db, db, Q, N, n, p, rooted, out, ldo, st);
}

}  // namespace dtwlb
