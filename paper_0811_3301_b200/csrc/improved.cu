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
// Two kernels:
//  * select_mask_kernel -- bandwidth-bound stream over the dense beta1 block that
//    computes, per (64-candidate tile, query), the 64-bit mask of LB_Keogh survivors
//    of the current range (lo < beta1 <= min(hi, thr)) and appends the non-empty
//    ones to the tile's (query, mask) list, so sparse ranges cost nothing per empty
//    (tile, query) pair in the next kernel.
//  * improved_kernel -- one CTA per tile of Ct candidates whose U(x), L(x) are
//    staged in shared memory; each warp walks entries of the tile's list with a
//    one-deep software pipeline (the next entry's
//    y, LU, UL, beta1 and threshold are loaded while the current query's survivors
//    are evaluated: lanes over i, butterfly reduction).  LIST mode appends
//    (beta_lb, c) keys of pairs with beta_lb <= thr to the query's list; DENSE mode
//    (the lb_improved C-ABI call) writes the rooted bound of every pair.
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

// ---------------------------------------------------------------- masks
// One warp per (query, group of 8 consecutive 64-candidate tiles).
constexpr int kTilesPerWarp = 8;
__global__ void __launch_bounds__(256)
select_mask_kernel(const float *__restrict__ beta1, int64_t ldb, int64_t Qb, int64_t N,
                   const float *__restrict__ lo, const float *__restrict__ hi, const float *__restrict__ thr,
                   bool all, unsigned long long *__restrict__ tile_m, int *__restrict__ tile_q,
                   int *__restrict__ tile_cnt, int64_t ntiles) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t groups = (ntiles + kTilesPerWarp - 1) / kTilesPerWarp;
    const int64_t q = gw / groups;
    if (q >= Qb) return;
    const int64_t t0 = (gw - q * groups) * kTilesPerWarp;
    const float l = all ? -kInf : (lo ? lo[q] : -kInf);
    float h = all ? kInf : (hi ? hi[q] : kInf);
    if (!all && thr) h = fminf(h, thr[q]);
    const float *row = beta1 + q * ldb;
    float v[2 * kTilesPerWarp];
#pragma unroll
    for (int t = 0; t < kTilesPerWarp; ++t) {
        const int64_t c = (t0 + t) * 64 + lane;
        v[2 * t] = c < N ? __ldg(row + c) : kInf;
        v[2 * t + 1] = c + 32 < N ? __ldg(row + c + 32) : kInf;
    }
#pragma unroll
    for (int t = 0; t < kTilesPerWarp; ++t) {
        const int64_t c = (t0 + t) * 64 + lane;
        // (test c < N explicitly: the +inf padding must not pass a range whose hi is +inf)
        const unsigned m0 = __ballot_sync(0xffffffffu, c < N && v[2 * t] > l && v[2 * t] <= h);
        const unsigned m1 = __ballot_sync(0xffffffffu, c + 32 < N && v[2 * t + 1] > l && v[2 * t + 1] <= h);
        const unsigned long long m = ((unsigned long long)m1 << 32) | m0;
        if (lane == t && t0 + t < ntiles && m) {  // append (q, mask) to the tile's list
            const int64_t tt = t0 + t;
            const int pos = atomicAdd(tile_cnt + tt, 1);
            tile_q[tt * Qb + pos] = (int)q;
            tile_m[tt * Qb + pos] = m;
        }
    }
}

// ---------------------------------------------------------------- LB_Improved
template <int EPL>
struct ImpCfg {
    static constexpr int NT = EPL <= 8 ? 512 : 256;  // register budget of the double-buffered query
    static constexpr bool PREFETCH = EPL <= 16;      // n <= 512: prefetch the next query's registers
};

template <int NV>
struct QRegs {
    float4 y[NV], lu[NV], ul[NV];
    float b1a, b1b, thr;
};

template <int EPL, bool KEOGH_ONLY>
__device__ __forceinline__ void load_query(QRegs<EPL / 4> &r, const ImprovedArgs &a, int64_t q, int64_t c0t,
                                           int lane) {
    constexpr int NV = EPL / 4, NPAD = 32 * EPL;
    if constexpr (!KEOGH_ONLY) {
        const float *yr = a.yq + q * NPAD, *lur = a.LUq + q * NPAD, *ulr = a.ULq + q * NPAD;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const int e = 4 * (lane + 32 * v);
            r.y[v] = __ldg(reinterpret_cast<const float4 *>(yr + e));
            r.lu[v] = __ldg(reinterpret_cast<const float4 *>(lur + e));
            r.ul[v] = __ldg(reinterpret_cast<const float4 *>(ulr + e));
        }
    }
    // beta1 of the 64-tile: lane holds slots lane and lane + 32
    const float *b = a.beta1 + q * a.ldb + c0t;
    const int64_t rem = a.N - c0t;
    r.b1a = lane < rem ? __ldg(b + lane) : kInf;
    r.b1b = lane + 32 < rem ? __ldg(b + lane + 32) : kInf;
    r.thr = a.thr ? __ldg(a.thr + q) : kInf;
}

template <int P, int EPL, bool KEOGH_ONLY, bool DENSE>
__global__ void __launch_bounds__(ImpCfg<EPL>::NT)
improved_kernel(ImprovedArgs a, int Ct) {
    constexpr int NT = ImpCfg<EPL>::NT;
    constexpr int NW = NT / 32;
    constexpr int NV = EPL / 4;
    constexpr int NPAD = 32 * EPL;
    extern __shared__ __align__(16) float sm[];
    float *sU = sm;                      // [Ct][NPAD]
    float *sL = sm + (size_t)Ct * NPAD;  // [Ct][NPAD]

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int subs = 64 / Ct;
    const int64_t tile = blockIdx.x / subs;
    const int sub = (int)(blockIdx.x - tile * subs);
    const int64_t c0t = tile * 64;               // first candidate of the 64-tile
    const int64_t c0 = c0t + (int64_t)sub * Ct;  // first candidate staged by this CTA
    if (c0 >= a.N) return;
    const int ct = (int)((a.N - c0) < Ct ? (a.N - c0) : Ct);
    const int n = a.n;
    const unsigned long long submask = (Ct == 64 ? ~0ull : ((1ull << Ct) - 1)) << (sub * Ct);

    // stage U(x), L(x) of the CTA's candidates; padding U=+inf, L=-inf contributes d = 0
    for (int t = threadIdx.x; t < Ct * NPAD; t += NT) {
        int r = t / NPAD, i = t - r * NPAD;
        bool ok = r < ct && i < n;
        sU[t] = ok ? __ldg(a.Ux + (c0 + r) * (int64_t)n + i) : kInf;
        sL[t] = ok ? __ldg(a.Lx + (c0 + r) * (int64_t)n + i) : -kInf;
    }
    __syncthreads();

    unsigned long long evals = 0;
    // this tile's (query, survivor mask) entries; warp w takes entries w, w+NW, ...
    const int cnt = a.tile_cnt[tile];
    const int *eq = a.tile_q + tile * a.Qb;
    const unsigned long long *em = a.tile_m + tile * a.Qb;
    int e = warp;
    if (e < cnt) {
        QRegs<NV> cur, nxt;
        int64_t qe = eq[e];
        unsigned long long m = em[e] & submask;
        load_query<EPL, KEOGH_ONLY>(cur, a, qe, c0t, lane);
        while (true) {
            const int en = e + NW;
            const bool more = en < cnt;
            int64_t qn = 0;
            unsigned long long mn = 0;
            if (more) {  // prefetch the next entry's query registers
                qn = eq[en];
                mn = em[en] & submask;
                if constexpr (ImpCfg<EPL>::PREFETCH) load_query<EPL, KEOGH_ONLY>(nxt, a, qn, c0t, lane);
            }
            const int64_t q = qe;
            evals += __popcll(m);
            unsigned long long mykey = 0;
            int nacc = 0;
            while (m) {
                // up to 4 survivors at once: 4 independent accumulation chains (ILP).
                // Everything below is warp-uniform control flow (m, nb are uniform).
                int bits[4];
                int nb = 0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int bt = m ? __ffsll(m) - 1 : -1;
                    bits[u] = bt;
                    if (bt >= 0) { m &= m - 1; ++nb; }
                }
#pragma unroll
                for (int u = 1; u < 4; ++u) bits[u] = bits[u] >= 0 ? bits[u] : bits[0];
                float s4[4] = {0.f, 0.f, 0.f, 0.f};
                if constexpr (!KEOGH_ONLY) {
                    int off[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) off[u] = (bits[u] - sub * Ct) * NPAD + 4 * lane;
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        const float4 y = cur.y[v], lu = cur.lu[v], ul = cur.ul[v];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const float4 ux = *reinterpret_cast<const float4 *>(sU + off[u] + 128 * v);
                            const float4 lx = *reinterpret_cast<const float4 *>(sL + off[u] + 128 * v);
                            // d = max(y - max(Ux, LU), min(Lx, UL) - y, 0)
                            float t = s4[u];
                            t = accp<P>(t, max3f(y.x - fmaxf(ux.x, lu.x), fminf(lx.x, ul.x) - y.x, 0.f));
                            t = accp<P>(t, max3f(y.y - fmaxf(ux.y, lu.y), fminf(lx.y, ul.y) - y.y, 0.f));
                            t = accp<P>(t, max3f(y.z - fmaxf(ux.z, lu.z), fminf(lx.z, ul.z) - y.z, 0.f));
                            t = accp<P>(t, max3f(y.w - fmaxf(ux.w, lu.w), fminf(lx.w, ul.w) - y.w, 0.f));
                            s4[u] = t;
                        }
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                        for (int u = 0; u < 4; ++u) s4[u] += __shfl_xor_sync(0xffffffffu, s4[u], o);
                }
                float b1v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    b1v[u] = __shfl_sync(0xffffffffu, bits[u] < 32 ? cur.b1a : cur.b1b, bits[u] & 31);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float beta = b1v[u] + s4[u];
                    const int64_t c = c0t + bits[u];
                    if constexpr (DENSE) {
                        if (u < nb && lane == 0) a.dense[q * a.ldd + c] = rootp<P>(beta);
                    } else if (u < nb && beta <= cur.thr) {
                        if (lane == (nacc & 31)) mykey = pack_key(beta, (uint32_t)c);
                        ++nacc;
                        if ((nacc & 31) == 0) {  // flush 32 keys
                            int base = 0;
                            if (lane == 0) base = atomicAdd(a.list_len + q, 32);
                            base = __shfl_sync(0xffffffffu, base, 0);
                            DCHECK(base + 32 <= a.cap, "list flush q=%lld base=%d", (long long)q, base);
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
                    DCHECK(base + rem <= a.cap, "list tail q=%lld base=%d rem=%d", (long long)q, base, rem);
                    if (lane < rem) a.list[q * a.cap + base + lane] = mykey;
                }
            }
            if (!more) break;
            if constexpr (ImpCfg<EPL>::PREFETCH) cur = nxt;
            else load_query<EPL, KEOGH_ONLY>(cur, a, qn, c0t, lane);
            e = en;
            qe = qn;
            m = mn;
        }
    }
    if (a.n_eval && lane == 0 && evals) atomicAdd(a.n_eval, evals);
}

template <int P, int EPL, bool KO, bool DENSE>
int launch_imp_t(const ImprovedArgs &a, int64_t ntiles, cudaStream_t st) {
    constexpr int NPAD = 32 * EPL;
    const int Ct = std::min(64, 16384 / NPAD);  // 128 KB of staged envelopes at most
    const size_t smem = (size_t)2 * Ct * NPAD * sizeof(float);
    auto k = improved_kernel<P, EPL, KO, DENSE>;
    DTWLB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t grid = ntiles * (64 / Ct);
    k<<<(unsigned)grid, ImpCfg<EPL>::NT, smem, st>>>(a, Ct);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

template <int P, bool KO, bool DENSE>
int launch_imp_e(const ImprovedArgs &a, int epl, int64_t ntiles, cudaStream_t st) {
    switch (epl) {
        case 4: return launch_imp_t<P, 4, KO, DENSE>(a, ntiles, st);
        case 8: return launch_imp_t<P, 8, KO, DENSE>(a, ntiles, st);
        case 16: return launch_imp_t<P, 16, KO, DENSE>(a, ntiles, st);
        case 32: return launch_imp_t<P, 32, KO, DENSE>(a, ntiles, st);
    }
    set_error(DTWLB_EUNSUPPORTED, "LB_Improved pass: n = %d exceeds 1024", a.n);
    return DTWLB_EUNSUPPORTED;
}

}  // namespace

// scratch bytes of the per-tile lists: masks (8 B) + queries (4 B) per (tile, query), + counts
size_t improved_scratch_bytes(int64_t Qb, int64_t N) {
    const int64_t nt = ceil_div(N, 64);
    return (size_t)nt * Qb * 12 + (size_t)nt * 4 + 256;
}
void improved_scratch_bind(ImprovedArgs &a, void *p) {
    const int64_t nt = ceil_div(a.N, 64);
    char *c = static_cast<char *>(p);
    a.tile_m = reinterpret_cast<unsigned long long *>(c);
    a.tile_q = reinterpret_cast<int *>(c + (size_t)nt * a.Qb * 8);
    a.tile_cnt = reinterpret_cast<int *>(c + (size_t)nt * a.Qb * 12);
}

int launch_improved(const ImprovedArgs &a, int p, bool keogh_only, bool dense, cudaStream_t st) {
    if (a.Qb == 0 || a.N == 0) return DTWLB_OK;
    const int64_t ntiles = ceil_div(a.N, 64);
    {   // per-tile (query, survivor mask) lists into the caller-provided scratch
        DTWLB_CUDA(cudaMemsetAsync(a.tile_cnt, 0, sizeof(int) * ntiles, st));
        const int64_t warps = ceil_div(ntiles, kTilesPerWarp) * a.Qb;
        select_mask_kernel<<<(unsigned)ceil_div(warps * 32, 256), 256, 0, st>>>(
            a.beta1, a.ldb, a.Qb, a.N, a.lo, a.hi, a.thr, dense, a.tile_m, a.tile_q, a.tile_cnt, ntiles);
        DTWLB_LAUNCH_CHECK();
    }
    const int epl = a.npadE / 32;
    if (p == 1) {
        if (keogh_only) return dense ? launch_imp_e<1, true, true>(a, epl, ntiles, st)
                                     : launch_imp_e<1, true, false>(a, epl, ntiles, st);
        return dense ? launch_imp_e<1, false, true>(a, epl, ntiles, st)
                     : launch_imp_e<1, false, false>(a, epl, ntiles, st);
    }
    if (keogh_only) return dense ? launch_imp_e<2, true, true>(a, epl, ntiles, st)
                                 : launch_imp_e<2, true, false>(a, epl, ntiles, st);
    return dense ? launch_imp_e<2, false, true>(a, epl, ntiles, st)
                 : launch_imp_e<2, false, false>(a, epl, ntiles, st);
}

}  // namespace dtwlb
