// improved.cu -- the LB_Improved pass (a4): Alg. 3 lines P:599-606.
//
//   LB_Improved^p = beta1 + beta2,  beta2 = sum_i d(y_i, [L(H)_i, U(H)_i])^p,
//   H = H(x, y) the projection of x on the envelope of y (Eq. (1)).
//
// B200 design -- a closed form for the envelope of H (DESIGN.md "LB_Improved
// without a per-candidate sliding window").  For every i, U(y)_k >= y_i for all
// k in the window of i, so with v_k = max(x_k, L(y)_k) and H_k = min(v_k, U(y)_k):
//   y_i > U(H)_i  <=>  max_k v_k < y_i, and then U(H)_i = max_k v_k exactly;
//   max_k v_k = max(U(x)_i, U(L(y))_i).
// Symmetrically for the lower side.  Hence, exactly (min/max do not round):
//   d(y_i, [L(H)_i, U(H)_i]) = max(y_i - max(U(x)_i, LU_i), min(L(x)_i, UL_i) - y_i, 0)
// with U(x), L(x) the candidate's own envelope (query independent: computed once
// per database) and LU = U(L(y)), UL = L(U(y)) computed once per query.  The
// per-candidate sliding max/min of Alg. 3 disappears: 6 ops per element.
//
// Kernel: one CTA per database tile of Ct candidates whose envelopes U(x), L(x)
// are staged in shared memory; each warp walks queries, ballots which of the
// tile's candidates survived LB_Keogh (lo < beta1 <= min(hi, thr)), loads the
// query's y, LU, UL into registers (EPL values per lane each) and evaluates the
// survivors one by one (lanes over i, butterfly reduction).  LIST mode appends
// (beta_lb, c) keys of pairs with beta_lb <= thr to the query's list; DENSE mode
// (the lb_improved C-ABI call) writes the rooted bound for every pair.
#include "kernels.cuh"

namespace dtwlb {

int improved_epl(int n) {
    if (n <= 128) return 4;
    if (n <= 256) return 8;
    if (n <= 512) return 16;
    if (n <= 1024) return 32;
    return 0;
}

namespace {

// 16 warps per CTA when the query registers allow it (EPL <= 16), else 8.
template <int EPL>
struct ImpCfg { static constexpr int NT = EPL <= 16 ? 512 : 256; };

template <int P, int EPL, bool KEOGH_ONLY, bool DENSE>
__global__ void __launch_bounds__(ImpCfg<EPL>::NT)
improved_kernel(ImprovedArgs a, int Ct) {
    constexpr int NT = ImpCfg<EPL>::NT;
    constexpr int NW = NT / 32;
    extern __shared__ __align__(16) float sm[];
    constexpr int NV = EPL / 4;         // float4 vectors per lane per array
    constexpr int NPAD = 32 * EPL;      // padded row length
    float *sU = sm;                     // [Ct][NPAD]
    float *sL = sm + (size_t)Ct * NPAD;  // [Ct][NPAD]

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t c0 = (int64_t)blockIdx.x * Ct;
    const int ct = (int)((a.N - c0) < Ct ? (a.N - c0) : Ct);
    const int n = a.n;

    // stage U(x), L(x) of the tile; padding U=+inf, L=-inf contributes d = 0
    for (int t = threadIdx.x; t < Ct * NPAD; t += NT) {
        int r = t / NPAD, i = t - r * NPAD;
        bool ok = r < ct && i < n;
        sU[t] = ok ? __ldg(a.Ux + (c0 + r) * (int64_t)n + i) : kInf;
        sL[t] = ok ? __ldg(a.Lx + (c0 + r) * (int64_t)n + i) : -kInf;
    }
    __syncthreads();

    unsigned long long evals = 0;
    for (int64_t q = warp; q < a.Qb; q += NW) {
        const float thr = a.thr ? a.thr[q] : kInf;
        const float lo = a.lo ? a.lo[q] : -kInf;
        const float hi = fminf(a.hi ? a.hi[q] : kInf, thr);
        const float *b1row = a.beta1 + q * a.ldb + c0;
        // survivor masks over the tile (Ct <= 64)
        float b1v0 = lane < ct ? b1row[lane] : kInf;
        float b1v1 = lane + 32 < ct ? b1row[lane + 32] : kInf;
        // (the padding value +inf must not pass a range whose hi is +inf: test lane < ct)
        unsigned m0 = __ballot_sync(0xffffffffu, lane < ct && (DENSE || (b1v0 > lo && b1v0 <= hi)));
        unsigned m1 = __ballot_sync(0xffffffffu, lane + 32 < ct && (DENSE || (b1v1 > lo && b1v1 <= hi)));
        if ((m0 | m1) == 0) continue;
        evals += __popc(m0) + __popc(m1);

        float4 y[NV], lu[NV], ul[NV];
        if constexpr (!KEOGH_ONLY) {
            const float *yr = a.yq + q * NPAD, *lur = a.LUq + q * NPAD, *ulr = a.ULq + q * NPAD;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                int e = 4 * (lane + 32 * v);
                y[v] = __ldg(reinterpret_cast<const float4 *>(yr + e));
                lu[v] = __ldg(reinterpret_cast<const float4 *>(lur + e));
                ul[v] = __ldg(reinterpret_cast<const float4 *>(ulr + e));
            }
        }
        // accepted results of this (query, tile) group, one per lane slot
        unsigned long long mykey = 0;
        int nacc = 0;
        for (int half = 0; half < 2; ++half) {
            unsigned m = half ? m1 : m0;
            while (m) {
                const int bit = __ffs(m) - 1;
                m &= m - 1;
                const int tc = bit + 32 * half;
                const float b1 = __shfl_sync(0xffffffffu, half ? b1v1 : b1v0, bit);
                float beta2 = 0.f;
                if constexpr (!KEOGH_ONLY) {
                    const float *ur = sU + (size_t)tc * NPAD, *lr = sL + (size_t)tc * NPAD;
                    float s = 0.f;
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        int e = 4 * (lane + 32 * v);
                        float4 ux = *reinterpret_cast<const float4 *>(ur + e);
                        float4 lx = *reinterpret_cast<const float4 *>(lr + e);
                        // d = max(y - max(Ux, LU), min(Lx, UL) - y, 0)
                        s = accp<P>(s, max3f(y[v].x - fmaxf(ux.x, lu[v].x), fminf(lx.x, ul[v].x) - y[v].x, 0.f));
                        s = accp<P>(s, max3f(y[v].y - fmaxf(ux.y, lu[v].y), fminf(lx.y, ul[v].y) - y[v].y, 0.f));
                        s = accp<P>(s, max3f(y[v].z - fmaxf(ux.z, lu[v].z), fminf(lx.z, ul[v].z) - y[v].z, 0.f));
                        s = accp<P>(s, max3f(y[v].w - fmaxf(ux.w, lu[v].w), fminf(lx.w, ul[v].w) - y[v].w, 0.f));
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                    beta2 = s;
                }
                const float beta = b1 + beta2;
                if constexpr (DENSE) {
                    if (lane == 0) a.dense[q * a.ldd + c0 + tc] = rootp<P>(beta);
                } else if (beta <= thr) {
                    if (lane == (nacc & 31)) mykey = pack_key(beta, (uint32_t)(c0 + tc));
                    ++nacc;
                    if ((nacc & 31) == 0) {  // flush 32 keys
                        int base = 0;
                        if (lane == 0) base = atomicAdd(a.list_len + q, 32);
                        base = __shfl_sync(0xffffffffu, base, 0);
                        DCHECK(base + 32 <= a.cap, "list flush q=%lld base=%d cap=%lld", (long long)q, base, (long long)a.cap);
                        a.list[q * a.cap + base + lane] = mykey;
                    }
                }
            }
        }
        if constexpr (!DENSE) {
            const int rem = nacc & 31;
            if (rem) {
                int base = 0;
                if (lane == 0) base = atomicAdd(a.list_len + q, rem);
                base = __shfl_sync(0xffffffffu, base, 0);
                DCHECK(base + rem <= a.cap, "list tail q=%lld base=%d rem=%d cap=%lld", (long long)q, base, rem, (long long)a.cap);
                if (lane < rem) a.list[q * a.cap + base + lane] = mykey;
            }
        }
    }
    if (a.n_eval && lane == 0 && evals) atomicAdd(a.n_eval, evals);
}

template <int P, int EPL, bool KO, bool DENSE>
int launch_imp_t(const ImprovedArgs &a, cudaStream_t st) {
    constexpr int NPAD = 32 * EPL;
    const int Ct = std::min(64, 16384 / NPAD);  // 128 KB of staged envelopes at most
    const size_t smem = (size_t)2 * Ct * NPAD * sizeof(float);
    auto k = improved_kernel<P, EPL, KO, DENSE>;
    DTWLB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t grid = ceil_div(a.N, Ct);
    k<<<(unsigned)grid, ImpCfg<EPL>::NT, smem, st>>>(a, Ct);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

template <int P, bool KO, bool DENSE>
int launch_imp_e(const ImprovedArgs &a, int epl, cudaStream_t st) {
    switch (epl) {
        case 4: return launch_imp_t<P, 4, KO, DENSE>(a, st);
        case 8: return launch_imp_t<P, 8, KO, DENSE>(a, st);
        case 16: return launch_imp_t<P, 16, KO, DENSE>(a, st);
        case 32: return launch_imp_t<P, 32, KO, DENSE>(a, st);
    }
    set_error(DTWLB_EUNSUPPORTED, "LB_Improved pass: n = %d exceeds 1024", a.n);
    return DTWLB_EUNSUPPORTED;
}

}  // namespace

int launch_improved(const ImprovedArgs &a, int p, bool keogh_only, bool dense, cudaStream_t st) {
    if (a.Qb == 0 || a.N == 0) return DTWLB_OK;
    const int epl = a.npadE / 32;
    if (p == 1) {
        if (keogh_only) return dense ? launch_imp_e<1, true, true>(a, epl, st) : launch_imp_e<1, true, false>(a, epl, st);
        return dense ? launch_imp_e<1, false, true>(a, epl, st) : launch_imp_e<1, false, false>(a, epl, st);
    }
    if (keogh_only) return dense ? launch_imp_e<2, true, true>(a, epl, st) : launch_imp_e<2, true, false>(a, epl, st);
    return dense ? launch_imp_e<2, false, true>(a, epl, st) : launch_imp_e<2, false, false>(a, epl, st);
}

}  // namespace dtwlb
