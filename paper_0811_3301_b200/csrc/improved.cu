// improved.cu -- the survivor passes of the cascade on sparse (query, candidate) pairs:
// LB_Keogh (a2) when a piecewise-sum pre-filter gated the pairs, and
// LB_Improved (a4, Alg. 3 lines P:599-606):
//
//   beta1 = sum_i d(x_i, [L(y)_i, U(y)_i])^p                        (LB_Keogh^p)
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
//  * select_mask_kernel -- bandwidth-bound stream over the dense gate-bound block
//    (the piecewise-sum bound beta0, or beta1 itself without the pre-filter) that
//    computes, per (64-candidate tile, query), the 64-bit mask of gate survivors of
//    the current range (lo < gate <= min(hi, thr)) and appends the non-empty ones
//    to the tile's (query, mask) list, so sparse ranges cost nothing per empty
//    (tile, query) pair in the next kernel.
//  * improved_kernel -- one CTA per tile of Ct candidates whose x (when beta1 is
//    computed here), U(x) and L(x) are staged in shared memory; each warp walks
//    entries of the tile's list (query registers of the next entry prefetched
//    while the current one is evaluated).  Lanes run over i; four survivors are
//    evaluated at once (four independent accumulation chains) and reduced with a
//    transposed butterfly (6 shuffles for 4 sums; lane l ends with survivor l/8).
//    Phase 1 (B1X): beta1 of the gate survivors from x in shared memory; its
//    survivors (beta1 <= thr) form the phase-2 mask.  Phase 2: beta2 and the key
//    (beta1 + beta2, c) of each pair with LB_Improved^p <= thr, appended to the
//    query's list with one warp-aggregated atomic per group.  DENSE mode (the
//    lb_improved C-ABI call) writes the rooted bound of every pair instead.
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
select_mask_kernel(const float *__restrict__ gate, int64_t ldb, int64_t Qb, int64_t N,
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
    const float *row = gate + q * ldb;
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

// ---------------------------------------------------------------- survivor passes
template <int EPL, bool B1X>
struct ImpCfg {
    static constexpr int NT = EPL <= 8 ? 512 : 256;
    // prefetch the next entry's query registers while the current one is evaluated
    // (n <= 256; beyond that the doubled query registers would spill)
    static constexpr bool PREFETCH = EPL <= 8;
};

// query-side registers of one entry: lane holds elements 4*lane + 128*v .. +3
template <int NV, bool B1X, bool KO>
struct QRegs {
    float4 u[B1X ? NV : 1], l[B1X ? NV : 1];             // U(y), L(y)       (phase 1)
    float4 y[KO ? 1 : NV], lu[KO ? 1 : NV], ul[KO ? 1 : NV];  // y, U(L), L(U)  (phase 2)
    float b1a, b1b;                                      // beta1 of slots lane, lane+32 (!B1X)
    float thr;
};

template <int EPL, bool B1X, bool KO>
__device__ __forceinline__ void load_p1(QRegs<EPL / 4, B1X, KO> &r, const ImprovedArgs &a, int64_t q,
                                        int64_t c0t, int lane) {
    constexpr int NV = EPL / 4, NPAD = 32 * EPL;
    if constexpr (B1X) {
        const float *ur = a.Uq + q * NPAD, *lr = a.Lq + q * NPAD;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const int e = 4 * (lane + 32 * v);
            r.u[v] = __ldg(reinterpret_cast<const float4 *>(ur + e));
            r.l[v] = __ldg(reinterpret_cast<const float4 *>(lr + e));
        }
    } else {
        const float *b = a.gate + q * a.ldb + c0t;
        const int64_t rem = a.N - c0t;
        r.b1a = lane < rem ? __ldg(b + lane) : kInf;
        r.b1b = lane + 32 < rem ? __ldg(b + lane + 32) : kInf;
    }
    r.thr = a.thr ? __ldg(a.thr + q) : kInf;
}

template <int EPL, bool B1X, bool KO>
__device__ __forceinline__ void load_p2(QRegs<EPL / 4, B1X, KO> &r, const ImprovedArgs &a, int64_t q,
                                        int lane) {
    constexpr int NV = EPL / 4, NPAD = 32 * EPL;
    if constexpr (!KO) {
        const float *yr = a.yq + q * NPAD, *lur = a.LUq + q * NPAD, *ulr = a.ULq + q * NPAD;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const int e = 4 * (lane + 32 * v);
            r.y[v] = __ldg(reinterpret_cast<const float4 *>(yr + e));
            r.lu[v] = __ldg(reinterpret_cast<const float4 *>(lur + e));
            r.ul[v] = __ldg(reinterpret_cast<const float4 *>(ulr + e));
        }
    }
}

// Up to four set bits of m (lowest first), removed from m; missing slots repeat
// the first bit (evaluated redundantly, results discarded).  Returns the count.
__device__ __forceinline__ int take4(unsigned long long &m, int (&bits)[4]) {
    int nb = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int bt = __ffsll(m) - 1;  // -1 if m == 0
        bits[u] = bt;
        if (bt >= 0) { m &= m - 1; ++nb; }
    }
#pragma unroll
    for (int u = 1; u < 4; ++u) bits[u] = bits[u] >= 0 ? bits[u] : bits[0];
    return nb;
}

// Transposed butterfly: four per-lane partial sums -> lane l holds the warp
// total of sum number l >> 3.  6 shuffles instead of 4 x 5.
__device__ __forceinline__ float reduce4(float s0, float s1, float s2, float s3, int lane) {
    const bool hi16 = lane & 16;
    float k0 = hi16 ? s2 : s0, k1 = hi16 ? s3 : s1;
    const float o0 = hi16 ? s0 : s2, o1 = hi16 ? s1 : s3;
    k0 += __shfl_xor_sync(0xffffffffu, o0, 16);
    k1 += __shfl_xor_sync(0xffffffffu, o1, 16);
    const bool hi8 = lane & 8;
    float v = hi8 ? k1 : k0;
    v += __shfl_xor_sync(0xffffffffu, hi8 ? k0 : k1, 8);
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    return v;
}

__device__ __forceinline__ int pick4(const int (&b)[4], int u) {
    return u == 0 ? b[0] : (u == 1 ? b[1] : (u == 2 ? b[2] : b[3]));
}

// Append the keys of the lanes with `pass` (one lane per survivor) to query q's list.
__device__ __forceinline__ void append_keys(const ImprovedArgs &a, int64_t q, bool pass, float beta, int64_t c,
                                            int lane) {
    const unsigned bal = __ballot_sync(0xffffffffu, pass);
    if (!bal) return;
    int base = 0;
    if (lane == 0) base = atomicAdd(a.list_len + q, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (pass) {
        const int pos = base + __popc(bal & ((1u << lane) - 1));
        DCHECK(pos < a.cap, "list append q=%lld pos=%d", (long long)q, pos);
        a.list[q * a.cap + pos] = pack_key(beta, (uint32_t)c);
    }
}

template <int P, int EPL, bool B1X, bool KO, bool DENSE>
__global__ void __launch_bounds__(ImpCfg<EPL, B1X>::NT)
improved_kernel(ImprovedArgs a, int Ct) {
    constexpr int NT = ImpCfg<EPL, B1X>::NT;
    constexpr bool PREFETCH = ImpCfg<EPL, B1X>::PREFETCH;
    constexpr int NW = NT / 32;
    constexpr int NV = EPL / 4;
    constexpr int NPAD = 32 * EPL;
    extern __shared__ __align__(16) float sm[];
    // [Ct][NPAD] blocks: x (B1X), U(x), L(x) (!KO); then per-warp beta1 slots [NW][64]
    float *sX = sm;
    float *sU = sm + (B1X ? (size_t)Ct * NPAD : 0);
    float *sL = sU + (KO ? 0 : (size_t)Ct * NPAD);
    float *sB1 = sL + (KO ? 0 : (size_t)Ct * NPAD);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int subs = 64 / Ct;
    const int64_t tile = blockIdx.x / subs;
    const int sub = (int)(blockIdx.x - tile * subs);
    const int64_t c0t = tile * 64;               // first candidate of the 64-tile
    const int64_t c0 = c0t + (int64_t)sub * Ct;  // first candidate staged by this CTA
    if (c0 >= a.N) return;
    const int cnt = a.tile_cnt[tile];
    if (cnt == 0) return;
    const int ct = (int)((a.N - c0) < Ct ? (a.N - c0) : Ct);
    const int n = a.n;
    const unsigned long long submask = (Ct == 64 ? ~0ull : ((1ull << Ct) - 1)) << (sub * Ct);

    // stage the tile: x padded with 0 (the query's padded U = +inf, L = -inf give d = 0);
    // U(x) = +inf, L(x) = -inf padding gives d = 0 in phase 2
    for (int t = threadIdx.x; t < Ct * NPAD; t += NT) {
        const int r = t / NPAD, i = t - r * NPAD;
        const bool ok = r < ct && i < n;
        const int64_t g = (c0 + r) * (int64_t)n + i;
        if constexpr (B1X) sX[t] = ok ? __ldg(a.xdb + g) : 0.f;
        if constexpr (!KO) {
            sU[t] = ok ? __ldg(a.Ux + g) : kInf;
            sL[t] = ok ? __ldg(a.Lx + g) : -kInf;
        }
    }
    __syncthreads();

    float *myB1 = sB1 + warp * 64;
    unsigned long long evals1 = 0, evals2 = 0;
    const int *eq = a.tile_q + tile * a.Qb;
    const unsigned long long *em = a.tile_m + tile * a.Qb;
    const int u_me = lane >> 3;  // survivor slot this lane ends up holding after reduce4
    int e = warp;
    if (e >= cnt) return;
    QRegs<NV, B1X, KO> cur, nxt;
    int64_t qe = eq[e];
    unsigned long long mcur = em[e] & submask;
    load_p1<EPL, B1X, KO>(cur, a, qe, c0t, lane);
    if (PREFETCH) load_p2<EPL, B1X, KO>(cur, a, qe, lane);
    while (true) {
        const int en = e + NW;
        const bool more = en < cnt;
        int64_t qn = 0;
        unsigned long long mn = 0;
        if (more) {
            qn = eq[en];
            mn = em[en] & submask;
            if constexpr (PREFETCH) {
                load_p1<EPL, B1X, KO>(nxt, a, qn, c0t, lane);
                load_p2<EPL, B1X, KO>(nxt, a, qn, lane);
            }
        }
        const int64_t q = qe;
        unsigned long long m = mcur;
        // ---------------- phase 1: beta1 (B1X) -> phase-2 mask
        unsigned long long m2 = 0;
        if constexpr (B1X) {
            while (m) {
                int bits[4];
                const int nb = take4(m, bits);
                evals1 += nb;
                float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const float4 uu = cur.u[v], ll = cur.l[v];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float4 x = *reinterpret_cast<const float4 *>(
                            sX + (bits[u] - sub * Ct) * NPAD + 4 * lane + 128 * v);
                        float t = s[u];
                        t = accp<P>(t, max3f(x.x - uu.x, ll.x - x.x, 0.f));
                        t = accp<P>(t, max3f(x.y - uu.y, ll.y - x.y, 0.f));
                        t = accp<P>(t, max3f(x.z - uu.z, ll.z - x.z, 0.f));
                        t = accp<P>(t, max3f(x.w - uu.w, ll.w - x.w, 0.f));
                        s[u] = t;
                    }
                }
                const float b1 = reduce4(s[0], s[1], s[2], s[3], lane);
                const int myb = pick4(bits, u_me);
                const bool lead = (lane & 7) == 0 && u_me < nb;
                if constexpr (!DENSE) {
                    // keep beta1 for the DTW walk's cascading abandon: the gate slot (beta0,
                    // already consumed by this range's mask) takes -beta1 (<= 0, so no later
                    // range re-selects it; the walk reads |.|)
                    if (lead && b1 <= cur.thr) a.gate_w[q * a.ldb + c0t + myb] = -b1;
                }
                if constexpr (KO) {
                    if constexpr (DENSE) {
                        if (lead) a.dense[q * a.ldd + c0t + myb] = rootp<P>(b1);
                    } else {
                        append_keys(a, q, lead && b1 <= cur.thr, b1, c0t + myb, lane);
                    }
                } else {
                    const bool pass = lead && (DENSE || b1 <= cur.thr);
                    if (pass) myB1[myb] = b1;
                    const unsigned bal = __ballot_sync(0xffffffffu, pass);
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if ((bal >> (8 * u)) & 1u) m2 |= 1ull << bits[u];
                }
            }
            __syncwarp();
        } else {
            m2 = m;
        }
        // ---------------- phase 2: beta2, LB_Improved^p = beta1 + beta2
        if constexpr (!KO) {
            if (!PREFETCH && m2) load_p2<EPL, B1X, KO>(cur, a, q, lane);
            while (m2) {
                int bits[4];
                const int nb = take4(m2, bits);
                evals2 += nb;
                float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const float4 y = cur.y[v], lu = cur.lu[v], ul = cur.ul[v];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int off = (bits[u] - sub * Ct) * NPAD + 4 * lane + 128 * v;
                        const float4 ux = *reinterpret_cast<const float4 *>(sU + off);
                        const float4 lx = *reinterpret_cast<const float4 *>(sL + off);
                        // d = max(y - max(Ux, LU), min(Lx, UL) - y, 0)
                        float t = s[u];
                        t = accp<P>(t, max3f(y.x - fmaxf(ux.x, lu.x), fminf(lx.x, ul.x) - y.x, 0.f));
                        t = accp<P>(t, max3f(y.y - fmaxf(ux.y, lu.y), fminf(lx.y, ul.y) - y.y, 0.f));
                        t = accp<P>(t, max3f(y.z - fmaxf(ux.z, lu.z), fminf(lx.z, ul.z) - y.z, 0.f));
                        t = accp<P>(t, max3f(y.w - fmaxf(ux.w, lu.w), fminf(lx.w, ul.w) - y.w, 0.f));
                        s[u] = t;
                    }
                }
                const float b2 = reduce4(s[0], s[1], s[2], s[3], lane);
                const int myb = pick4(bits, u_me);
                float b1;
                if constexpr (B1X) {
                    b1 = myB1[myb];
                } else {
                    const float va = __shfl_sync(0xffffffffu, cur.b1a, myb & 31);
                    const float vb = __shfl_sync(0xffffffffu, cur.b1b, myb & 31);
                    b1 = myb < 32 ? va : vb;
                }
                const float beta = b1 + b2;
                const bool lead = (lane & 7) == 0 && u_me < nb;
                if constexpr (DENSE) {
                    if (lead) a.dense[q * a.ldd + c0t + myb] = rootp<P>(beta);
                } else {
                    append_keys(a, q, lead && beta <= cur.thr, beta, c0t + myb, lane);
                }
            }
            if constexpr (B1X) __syncwarp();
        } else if constexpr (!B1X) {
            // Alg. 2 (keogh-only) over the dense beta1 block: the gate survivors are the keys
            while (m2) {
                int bits[4];
                const int nb = take4(m2, bits);
                const int myb = pick4(bits, u_me);
                const float va = __shfl_sync(0xffffffffu, cur.b1a, myb & 31);
                const float vb = __shfl_sync(0xffffffffu, cur.b1b, myb & 31);
                const float b1 = myb < 32 ? va : vb;
                const bool lead = (lane & 7) == 0 && u_me < nb;
                if constexpr (DENSE) {
                    if (lead) a.dense[q * a.ldd + c0t + myb] = rootp<P>(b1);
                } else {
                    append_keys(a, q, lead && b1 <= cur.thr, b1, c0t + myb, lane);
                }
            }
        }
        if (!more) break;
        if constexpr (PREFETCH) {
            cur = nxt;
        } else {
            load_p1<EPL, B1X, KO>(cur, a, qn, c0t, lane);
        }
        e = en;
        qe = qn;
        mcur = mn;
    }
    if (lane == 0) {
        if (a.n_eval && evals2) atomicAdd(a.n_eval, evals2);
        if (a.n_eval_keogh && evals1) atomicAdd(a.n_eval_keogh, evals1);
    }
}

template <int P, int EPL, bool B1X, bool KO, bool DENSE>
int launch_imp_t(const ImprovedArgs &a, int64_t ntiles, cudaStream_t st) {
    constexpr int NPAD = 32 * EPL;
    constexpr int NT = ImpCfg<EPL, B1X>::NT;
    const int arrays = (B1X ? 1 : 0) + (KO ? 0 : 2);
    // staged rows: at most 64 candidates and 192 KB (3 arrays) / 128 KB (2 arrays)
    const int Ct = std::min(64, 16384 / NPAD);
    const size_t smem = (size_t)arrays * Ct * NPAD * sizeof(float) + (size_t)(NT / 32) * 64 * sizeof(float);
    auto k = improved_kernel<P, EPL, B1X, KO, DENSE>;
    DTWLB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t grid = ntiles * (64 / Ct);
    k<<<(unsigned)grid, NT, smem, st>>>(a, Ct);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

template <int P, bool B1X, bool KO, bool DENSE>
int launch_imp_e(const ImprovedArgs &a, int epl, int64_t ntiles, cudaStream_t st) {
    switch (epl) {
        case 4: return launch_imp_t<P, 4, B1X, KO, DENSE>(a, ntiles, st);
        case 8: return launch_imp_t<P, 8, B1X, KO, DENSE>(a, ntiles, st);
        case 16: return launch_imp_t<P, 16, B1X, KO, DENSE>(a, ntiles, st);
        case 32: return launch_imp_t<P, 32, B1X, KO, DENSE>(a, ntiles, st);
    }
    set_error(DTWLB_EUNSUPPORTED, "LB_Improved pass: n = %d exceeds 1024", a.n);
    return DTWLB_EUNSUPPORTED;
}

template <int P>
int launch_imp_p(const ImprovedArgs &a, int epl, bool keogh_only, bool dense, int64_t ntiles, cudaStream_t st) {
    if (a.xdb) {  // beta1 computed here (pre-filtered cascade)
        if (keogh_only) return launch_imp_e<P, true, true, false>(a, epl, ntiles, st);
        return dense ? launch_imp_e<P, true, false, true>(a, epl, ntiles, st)
                     : launch_imp_e<P, true, false, false>(a, epl, ntiles, st);
    }
    if (keogh_only) return launch_imp_e<P, false, true, false>(a, epl, ntiles, st);
    return dense ? launch_imp_e<P, false, false, true>(a, epl, ntiles, st)
                 : launch_imp_e<P, false, false, false>(a, epl, ntiles, st);
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
            a.gate, a.ldb, a.Qb, a.N, a.lo, a.hi, a.thr, dense, a.tile_m, a.tile_q, a.tile_cnt, ntiles);
        DTWLB_LAUNCH_CHECK();
    }
    const int epl = a.npadE / 32;
    return p == 1 ? launch_imp_p<1>(a, epl, keogh_only, dense, ntiles, st)
                  : launch_imp_p<2>(a, epl, keogh_only, dense, ntiles, st);
}

}  // namespace dtwlb
