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
// (candidate) from registers.  Per pair-element: FMNMX, FMNMX (the clamp of x
// into [L, U], ALU pipe), FADD, FFMA|FADD (FMA pipe): 4 ops split 2/2 over the
// two pipes, which measured faster than the 3-FMA-pipe-op form
// max(x-U, L-x, 0) ("LB_Keogh instruction mix").  Per-chunk partial
// sums are folded into the total at each chunk end (two-level summation keeps
// the fp32 error at ~(32 + n/32) ulp instead of n ulp).
// CTAs are ordered query-tile-fastest so each database tile is fetched from
// HBM once and served from L2 to every query tile; the envelopes of the whole
// query block stay L2-resident.  The i-tail beyond n is zero-filled on both
// sides, which contributes max(0-0, 0-0, 0) = 0.
#include <cstdlib>

#include "kernels.cuh"

namespace dtwlb {

namespace {

constexpr int TQ = 64, TC = 128, KC = 32, KP = KC + 4;  // KP: padded pitch (floats)
constexpr int NT = 256;

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int src_bytes) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem, int src_bytes) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

struct Stage {  // chunk of the operands, written by cp.async (double-buffered)
    float X[TC][KP];
    float U[TQ][KP];
    float L[TQ][KP];
};
// acc + |d|^p for a signed deviation d (p=1: FADD with |.| operand; p=2: FFMA)
template <int P>
__device__ __forceinline__ float acc_dev(float acc, float d) {
    if constexpr (P == 1) return acc + fabsf(d);
    else return fmaf(d, d, acc);
}

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

template <int P, bool VEC, bool ROOTED, int VAR, int MINB>
__global__ void __launch_bounds__(NT, MINB)
keogh_tile_kernel(const float *__restrict__ U, const float *__restrict__ L, const float *__restrict__ db,
                  int64_t Q, int64_t N, int n, float *__restrict__ out, int64_t ldo, int nqt) {
    extern __shared__ __align__(16) unsigned char smraw[];
    Stage *st = reinterpret_cast<Stage *>(smraw);

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
    stage_rows<TQ, VEC>(st[0].U, U, q0, Q, n, 0);
    stage_rows<TQ, VEC>(st[0].L, L, q0, Q, n, 0);
    cp_commit();

    for (int ch = 0; ch < nchunks; ++ch) {
        if (ch + 1 < nchunks) {
            Stage &nx = st[(ch + 1) & 1];
            stage_rows<TC, VEC>(nx.X, db, c0, N, n, (ch + 1) * KC);
            stage_rows<TQ, VEC>(nx.U, U, q0, Q, n, (ch + 1) * KC);
            stage_rows<TQ, VEC>(nx.L, L, q0, Q, n, (ch + 1) * KC);
        }
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        const Stage &s = st[ch & 1];
        float part[4][8];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int j = 0; j < 8; ++j) part[r][j] = 0.f;

#pragma unroll 2
        for (int k = 0; k < KC; k += 4) {
            float4 xv[8], uv[4], lv[4];
#pragma unroll
            for (int j = 0; j < 8; ++j) xv[j] = *reinterpret_cast<const float4 *>(&s.X[cg + 16 * j][k]);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                uv[r] = *reinterpret_cast<const float4 *>(&s.U[4 * qg + r][k]);
                lv[r] = *reinterpret_cast<const float4 *>(&s.L[4 * qg + r][k]);
            }
            if constexpr (VAR == 1) {
                // d = x - clamp(x, L, U) (= x - H(x,y)_i of Eq. (1)); acc += |d|^p:
                // FMNMX, FMNMX (ALU pipe), FADD, FFMA|FADD (FMA pipe)
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        part[r][j] = acc_dev<P>(part[r][j], xv[j].x - fminf(fmaxf(xv[j].x, lv[r].x), uv[r].x));
                        part[r][j] = acc_dev<P>(part[r][j], xv[j].y - fminf(fmaxf(xv[j].y, lv[r].y), uv[r].y));
                        part[r][j] = acc_dev<P>(part[r][j], xv[j].z - fminf(fmaxf(xv[j].z, lv[r].z), uv[r].z));
                        part[r][j] = acc_dev<P>(part[r][j], xv[j].w - fminf(fmaxf(xv[j].w, lv[r].w), uv[r].w));
                    }
            } else {
                // d = max(x - U, L - x, 0); acc += d^p: FADD, FADD, FMNMX3(.., 0), FFMA|FADD
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        float d;
                        d = max3f(xv[j].x - uv[r].x, lv[r].x - xv[j].x, 0.f); part[r][j] = accp<P>(part[r][j], d);
                        d = max3f(xv[j].y - uv[r].y, lv[r].y - xv[j].y, 0.f); part[r][j] = accp<P>(part[r][j], d);
                        d = max3f(xv[j].z - uv[r].z, lv[r].z - xv[j].z, 0.f); part[r][j] = accp<P>(part[r][j], d);
                        d = max3f(xv[j].w - uv[r].w, lv[r].w - xv[j].w, 0.f); part[r][j] = accp<P>(part[r][j], d);
                    }
            }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[r][j] += part[r][j];
        __syncthreads();
    }

#pragma unroll
    for (int r = 0; r < 4; ++r) {
        int64_t q = q0 + 4 * qg + r;
        if (q >= Q) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            int64_t c = c0 + cg + 16 * j;
            if (c < N) out[q * ldo + c] = ROOTED ? rootp<P>(acc[r][j]) : acc[r][j];
        }
    }
}

// DTWLB_KEOGH_VAR (experiments): 0 = max3 form, 1 CTA/SM; 1 = clamp form, 1 CTA/SM;
// 2 = max3 form, 2 CTAs/SM; 3 = clamp form, 2 CTAs/SM.
int keogh_variant() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("DTWLB_KEOGH_VAR");
        v = e ? atoi(e) : 2;  // default: max3 form, 2 CTAs per SM (measured best)
        if (v < 0 || v > 3) v = 2;
    }
    return v;
}

template <int P, bool VEC, bool ROOTED, int VAR, int MINB>
int launch_keogh_v(const float *U, const float *L, const float *db, int64_t Q, int64_t N, int n,
                   float *out, int64_t ldo, cudaStream_t st) {
    const size_t smem = 2 * sizeof(Stage);
    auto k = keogh_tile_kernel<P, VEC, ROOTED, VAR, MINB>;
    DTWLB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t nqt = ceil_div(Q, TQ), nct = ceil_div(N, TC);
    const int64_t tiles = nqt * nct;
    if (tiles > 0x7fffffffLL) {
        set_error(DTWLB_EINVAL, "lb_keogh: problem too large (%lld tiles)", (long long)tiles);
        return DTWLB_EINVAL;
    }
    k<<<(unsigned)tiles, NT, smem, st>>>(U, L, db, Q, N, n, out, ldo, (int)nqt);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

template <int P, bool VEC, bool ROOTED>
int launch_keogh_t(const float *U, const float *L, const float *db, int64_t Q, int64_t N, int n,
                   float *out, int64_t ldo, cudaStream_t st) {
    switch (keogh_variant()) {
        case 1: return launch_keogh_v<P, VEC, ROOTED, 1, 1>(U, L, db, Q, N, n, out, ldo, st);
        case 2: return launch_keogh_v<P, VEC, ROOTED, 0, 2>(U, L, db, Q, N, n, out, ldo, st);
        case 3: return launch_keogh_v<P, VEC, ROOTED, 1, 2>(U, L, db, Q, N, n, out, ldo, st);
        default: return launch_keogh_v<P, VEC, ROOTED, 0, 1>(U, L, db, Q, N, n, out, ldo, st);
    }
}

}  // namespace

int launch_keogh(const float *U, const float *L, const float *db, int64_t Q, int64_t N, int n, int p,
                 bool rooted, float *out, int64_t ldo, cudaStream_t st) {
    if (Q == 0 || N == 0) return DTWLB_OK;
    const bool vec = (n % 4 == 0) && ((reinterpret_cast<uintptr_t>(U) | reinterpret_cast<uintptr_t>(L) |
                                       reinterpret_cast<uintptr_t>(db)) % 16 == 0);
#define DTWLB_K(P_, V_, R_) return launch_keogh_t<P_, V_, R_>(U, L, db, Q, N, n, out, ldo, st)
    if (p == 1) {
        if (vec) { if (rooted) DTWLB_K(1, true, true); else DTWLB_K(1, true, false); }
        else { if (rooted) DTWLB_K(1, false, true); else DTWLB_K(1, false, false); }
    } else {
        if (vec) { if (rooted) DTWLB_K(2, true, true); else DTWLB_K(2, true, false); }
        else { if (rooted) DTWLB_K(2, false, true); else DTWLB_K(2, false, false); }
    }
#undef DTWLB_K
}

}  // namespace dtwlb
