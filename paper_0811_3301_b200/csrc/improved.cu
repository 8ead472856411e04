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
#include <type_traits>

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
// One warp per (64-candidate tile, block of 32 queries): lane l reads candidates 2l and
// 2l + 1 of the tile (one 8-byte / 4-byte vector per lane: the tile's row of a query in
// one 256 / 128-byte access) for each query in turn; two ballots (even / odd candidates)
// are bit-interleaved into the query's 64-bit survivor mask, lane j keeps query j's
// mask, and the non-empty ones are appended to the tile's list with ONE atomic per warp.
__device__ __forceinline__ float2 gate_pair(const float *g, int64_t i) {
    return __ldg(reinterpret_cast<const float2 *>(g + i));
}
__device__ __forceinline__ float2 gate_pair(const __half *g, int64_t i) {
    return __half22float2(*reinterpret_cast<const __half2 *>(g + i));
}
// bit k of x -> bit 2k of the result
__device__ __forceinline__ unsigned long long spread_bits(unsigned x) {
    unsigned long long v = x;
    v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
    v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
    v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
    v = (v | (v << 2)) & 0x3333333333333333ull;
    v = (v | (v << 1)) & 0x5555555555555555ull;
    return v;
}

template <typename T>
__global__ void __launch_bounds__(256)
select_mask_kernel(const T *__restrict__ gate, int64_t ldb, int64_t Qb, int64_t N,
                   const float *__restrict__ lo, const float *__restrict__ hi, const float *__restrict__ thr,
                   bool all, unsigned long long *__restrict__ tile_m, int *__restrict__ tile_q,
                   int *__restrict__ tile_cnt, int64_t ntiles, int *__restrict__ q_count) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t tt = gw % ntiles;   // tile
    const int64_t qb = gw / ntiles;   // block of 32 queries
    const int64_t q0 = qb * 32;
    if (q0 >= Qb) return;
    const int nq = Qb - q0 < 32 ? (int)(Qb - q0) : 32;
    // this lane's query bounds (query q0 + lane), broadcast per iteration
    float my_l = -kInf, my_h = kInf;
    if (!all && lane < nq) {
        if (lo) my_l = lo[q0 + lane];
        if (hi) my_h = hi[q0 + lane];
        if (thr) my_h = fminf(my_h, thr[q0 + lane]);
    }
    const int64_t c0 = tt * 64 + 2 * lane;  // candidates c0, c0 + 1 (ldb is a multiple of 4)
    const bool ok0 = c0 < N, ok1 = c0 + 1 < N;
    unsigned my_e = 0, my_o = 0;  // even / odd candidate ballots of query q0 + lane
#pragma unroll 8
    for (int j = 0; j < nq; ++j) {
        const T *row = gate + (q0 + j) * ldb;
        float2 v = make_float2(kInf, kInf);
        if (ok0) v = gate_pair(row, c0);  // c0 + 1 <= ldb - 1: in the padded row
        const float l = __shfl_sync(0xffffffffu, my_l, j), h = __shfl_sync(0xffffffffu, my_h, j);
        // (test c < N explicitly: the +inf / padding must not pass a range whose hi is +inf)
        const unsigned me = __ballot_sync(0xffffffffu, ok0 && v.x > l && v.x <= h);
        const unsigned mo = __ballot_sync(0xffffffffu, ok1 && v.y > l && v.y <= h);
        if (lane == j) { my_e = me; my_o = mo; }
    }
    const unsigned long long my_m = spread_bits(my_e) | (spread_bits(my_o) << 1);
    if (q_count && my_m) atomicAdd(q_count + q0 + lane, __popcll(my_m));
    const unsigned has = __ballot_sync(0xffffffffu, my_m != 0);
    if (!has) return;
    int base = 0;
    if (lane == 0) base = atomicAdd(tile_cnt + tt, __popc(has));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (my_m) {
        const int pos = base + __popc(has & ((1u << lane) - 1u));
        tile_q[tt * Qb + pos] = (int)(q0 + lane);
        tile_m[tt * Qb + pos] = my_m;
    }
}

// fp16 gate block (the pre-filtered cascade): one warp per (256-candidate super-tile, block
// of 32 queries); lane l reads candidates 8l .. 8l+7 of the super-tile (one 16-byte vector
// per query row: 512 bytes per row per warp, eight rows in flight), eight ballots per row;
// lane j keeps query j's ballots and turns them into the four 64-bit tile masks (candidate
// 64t + 8m + k = bit 8m + k of tile t: byte t of ballot k, spread to bits 8m).
__device__ __forceinline__ unsigned long long spread8(unsigned x) {  // bit m -> bit 8m
    unsigned long long v = x & 0xffu;
    v = (v | (v << 28)) & 0x0000000F0000000Full;
    v = (v | (v << 14)) & 0x0003000300030003ull;
    v = (v | (v << 7)) & 0x0101010101010101ull;
    return v;
}

__global__ void __launch_bounds__(256)
select_mask8_kernel(const __half *__restrict__ gate, int64_t ldb, int64_t Qb, int64_t N,
                    const float *__restrict__ lo, const float *__restrict__ hi, const float *__restrict__ thr,
                    bool all, unsigned long long *__restrict__ tile_m, int *__restrict__ tile_q,
                    int *__restrict__ tile_cnt, int64_t ntiles, int *__restrict__ q_count) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nst = (ntiles + 3) / 4;
    const int64_t sti = gw % nst;  // super-tile
    const int64_t qb = gw / nst;   // block of 32 queries
    const int64_t q0 = qb * 32;
    if (q0 >= Qb) return;
    const int nq = Qb - q0 < 32 ? (int)(Qb - q0) : 32;
    float my_l = -kInf, my_h = kInf;
    if (!all && lane < nq) {
        if (lo) my_l = lo[q0 + lane];
        if (hi) my_h = hi[q0 + lane];
        if (thr) my_h = fminf(my_h, thr[q0 + lane]);
    }
    const int64_t c0 = sti * 256 + 8 * lane;  // this lane's 8 candidates (ldb % 8 == 0)
    const bool inrow = c0 < ldb;
    const int nvalid = c0 >= N ? 0 : (N - c0 >= 8 ? 8 : (int)(N - c0));
    unsigned bk[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // query q0 + lane: ballot k (candidate 8l + k of lane l)
    // eight rows' loads issued before their ballots (the compiler kept one in flight per warp
    // when each load fed its ballots directly: the pass ran at ~half of the HBM bandwidth)
    for (int j0 = 0; j0 < nq; j0 += 8) {
        uint4 raws[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            raws[u] = make_uint4(0x7c007c00u, 0x7c007c00u, 0x7c007c00u, 0x7c007c00u);  // +inf
            if (inrow && j0 + u < nq) raws[u] = __ldg(reinterpret_cast<const uint4 *>(gate + (q0 + j0 + u) * ldb + c0));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = j0 + u;
            if (j >= nq) break;
            const float l = __shfl_sync(0xffffffffu, my_l, j), h = __shfl_sync(0xffffffffu, my_h, j);
            const unsigned wv[4] = {raws[u].x, raws[u].y, raws[u].z, raws[u].w};
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float v = __half2float(__ushort_as_half((unsigned short)((k & 1) ? wv[k >> 1] >> 16 : wv[k >> 1] & 0xffffu)));
                // (test c < N explicitly: the +inf / padding must not pass a range whose hi is +inf)
                const unsigned b = __ballot_sync(0xffffffffu, k < nvalid && v > l && v <= h);
                if (lane == j) bk[k] = b;
            }
        }
    }
    unsigned long long m[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        m[t] = 0ull;
#pragma unroll
        for (int k = 0; k < 8; ++k) m[t] |= spread8(bk[k] >> (8 * t)) << k;
    }
#pragma unroll
    if (q_count && lane < nq) {  // the range's gate survivors of query q0 + lane in this super-tile
        const int c = __popcll(m[0]) + __popcll(m[1]) + __popcll(m[2]) + __popcll(m[3]);
        if (c) atomicAdd(q_count + q0 + lane, c);
    }
    for (int t = 0; t < 4; ++t) {
        const int64_t tt = sti * 4 + t;
        const unsigned has = __ballot_sync(0xffffffffu, m[t] != 0ull);
        if (!has || tt >= ntiles) continue;
        int base = 0;
        if (lane == 0) base = atomicAdd(tile_cnt + tt, __popc(has));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (m[t]) {
            const int pos = base + __popc(has & ((1u << lane) - 1u));
            tile_q[tt * Qb + pos] = (int)(q0 + lane);
            tile_m[tt * Qb + pos] = m[t];
        }
    }
}

// ---------------------------------------------------------------- survivor passes
template <int EPL, bool B1X>
struct ImpCfg {
    static constexpr int NT = EPL <= 8 ? 512 : (EPL == 16 ? 384 : 256);
    // prefetch the next entry's phase-1 query registers (U, L) while the current one is
    // evaluated, and issue the current entry's phase-2 loads (y, LU, UL) before its phase 1
    // (n <= 256; beyond that the extra query registers would spill)
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
        const float *b = static_cast<const float *>(a.gate) + q * a.ldb + c0t;  // float when !B1X
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

// Compact the set bits of the warp-uniform 64-bit mask m into lst[0..cnt) (ascending),
// padded with zeros to a multiple of 8 (padding slots are evaluated redundantly on
// local row 0 and discarded).  Returns cnt.  Caller syncs the warp before reading.
__device__ __forceinline__ int compact_mask(unsigned long long m, int *lst, int lane) {
    const unsigned lo = (unsigned)m, hi = (unsigned)(m >> 32);
    const unsigned lt = (1u << lane) - 1u;
    const int nlo = __popc(lo);
    if ((lo >> lane) & 1u) lst[__popc(lo & lt)] = lane;
    if ((hi >> lane) & 1u) lst[nlo + __popc(hi & lt)] = lane + 32;
    const int cnt = nlo + __popc(hi);
    if (lane < ((8 - (cnt & 7)) & 7)) lst[cnt + lane] = 0;
    return cnt;
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

__device__ __forceinline__ int pick4(const int4 &b, int u) {
    return u == 0 ? b.x : (u == 1 ? b.y : (u == 2 ? b.z : b.w));
}

// W-wide butterfly (W in {1, 2, 4, 8}): lane l ends with the warp total of slot l >> (5 - log2 W).
template <int W>
__device__ __forceinline__ float reduceW(const float (&s)[8], int lane) {
    if constexpr (W == 8) {
        // transposed: keep the half of the slots this lane's half-warp owns at each level
        const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
        float k[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            k[j] = h16 ? s[4 + j] : s[j];
            k[j] += __shfl_xor_sync(0xffffffffu, h16 ? s[j] : s[4 + j], 16);
        }
        float m0 = h8 ? k[2] : k[0], m1 = h8 ? k[3] : k[1];
        m0 += __shfl_xor_sync(0xffffffffu, h8 ? k[0] : k[2], 8);
        m1 += __shfl_xor_sync(0xffffffffu, h8 ? k[1] : k[3], 8);
        float v = h4 ? m1 : m0;
        v += __shfl_xor_sync(0xffffffffu, h4 ? m0 : m1, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        return v;
    } else if constexpr (W == 4) {
        return reduce4(s[0], s[1], s[2], s[3], lane);
    } else if constexpr (W == 2) {
        const bool hi16 = lane & 16;
        float v = hi16 ? s[1] : s[0];
        v += __shfl_xor_sync(0xffffffffu, hi16 ? s[0] : s[1], 16);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        return v;
    } else {
        float v = s[0];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    }
}

// Phase-1 partial sums of W survivors (local rows li[0..W)): lane covers samples
// 4*lane + 128*v .. +3 of beta1 = sum_i d(x_i, [L_i, U_i])^p.
template <int W, int P, int NV, int NPAD>
__device__ __forceinline__ float p1_group(const float *sX, const int (&li)[8], const float4 (&uq)[NV],
                                          const float4 (&lq)[NV], int lane) {
    float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const float4 uu = uq[v], ll = lq[v];
#pragma unroll
        for (int u = 0; u < W; ++u) {
            const float4 x = *reinterpret_cast<const float4 *>(sX + li[u] * NPAD + 4 * lane + 128 * v);
            float t = s[u];
            t = accp<P>(t, max3f(x.x - uu.x, ll.x - x.x, 0.f));
            t = accp<P>(t, max3f(x.y - uu.y, ll.y - x.y, 0.f));
            t = accp<P>(t, max3f(x.z - uu.z, ll.z - x.z, 0.f));
            t = accp<P>(t, max3f(x.w - uu.w, ll.w - x.w, 0.f));
            s[u] = t;
        }
    }
    return reduceW<W>(s, lane);
}

// Phase-2 partial sums: beta2 = sum_i max(y_i - max(U(x)_i, LU_i), min(L(x)_i, UL_i) - y_i, 0)^p.
template <int W, int P, int NV, int NPAD, int V0 = 0, int V1 = NV>
__device__ __forceinline__ float p2_group(const float *sU, const float *sL, const int (&li)[8],
                                          const float4 (&yq)[NV], const float4 (&luq)[NV],
                                          const float4 (&ulq)[NV], int lane) {
    float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int v = V0; v < V1; ++v) {
        const float4 y = yq[v], lu = luq[v], ul = ulq[v];
#pragma unroll
        for (int u = 0; u < W; ++u) {
            const int off = li[u] * NPAD + 4 * lane + 128 * v;
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
    return reduceW<W>(s, lane);
}

// Read the W list entries at g (g % W == 0).
template <int W>
__device__ __forceinline__ void read_group(const int *lst, int g, int (&li)[8]) {
    if constexpr (W == 8) {
        const int4 v = *reinterpret_cast<const int4 *>(lst + g);
        const int4 u = *reinterpret_cast<const int4 *>(lst + g + 4);
        li[0] = v.x; li[1] = v.y; li[2] = v.z; li[3] = v.w;
        li[4] = u.x; li[5] = u.y; li[6] = u.z; li[7] = u.w;
    } else if constexpr (W == 4) {
        const int4 v = *reinterpret_cast<const int4 *>(lst + g);
        li[0] = v.x; li[1] = v.y; li[2] = v.z; li[3] = v.w;
    } else if constexpr (W == 2) {
        const int2 v = *reinterpret_cast<const int2 *>(lst + g);
        li[0] = v.x; li[1] = v.y; li[2] = v.x; li[3] = v.y;
    } else {
        li[0] = li[1] = li[2] = li[3] = lst[g];
    }
}

// Append the keys of the lanes with `pass` (one lane per survivor) to query q's list.
// Returns the key's list position on the passing lanes (-1 elsewhere).
__device__ __forceinline__ int append_keys(const ImprovedArgs &a, int64_t q, bool pass, float beta, int64_t c,
                                           int lane) {
    const unsigned bal = __ballot_sync(0xffffffffu, pass);
    if (!bal) return -1;
    int base = 0;
    if (lane == 0) base = atomicAdd(a.list_len + q, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, 0);
    int pos = -1;
    if (pass) {
        pos = base + __popc(bal & ((1u << lane) - 1));
        DCHECK(a.loff ? a.loff[q] + pos < a.loff[q + 1] : pos < a.cap, "list append q=%lld pos=%d", (long long)q, pos);
        a.list[list_base(a.loff, a.cap, q) + pos] = pack_list_key(beta, (uint32_t)c, pos);
    }
    return pos;
}

// Column part of the DTW walk's abandon schedule for one appended pair (DESIGN.md reading
// c22), written to dst[0..32) as fp16: dst[0] = rd(sum_{c >= 4 c0b} beta2_c) and, for
// k = 0..30, dst[1 + k] = ru(E[k]), E[k] = sum_{c in [8k, 8k + 8) + 4 c0b} beta2_c, with
// beta2_c = d(y_c, [L(H)_c, U(H)_c])^p (the closed form above) and 4 c0b >= w.  The walk adds
// dst[0] to its row cascade (+-beta1 minus the computed rows' LB_Keogh terms) at its first
// test and subtracts E[k] after rows 8k .. 8k+7: after 8(k+1) rows the column part is <= the
// sum over columns >= 8(k+1) + w, which every completion visits (no computed row reaches
// them), and each of its cells (r, c) costs at least the row term of r plus the column term
// of c (Theorem 1's split), so rowmin + rest bounds DTW^p.  cb0 / cb1: this lane's
// column terms of the 4-sample blocks lane and lane + 32 (phase 2's per-block partials).
// p2_group keeping this lane's per-block partials: c0[u] / c1[u] = the column terms of
// survivor u over the lane's blocks lane / lane + 32 (REC, NV <= 2); hd: like the return value
// (lane l: survivor l >> (5 - log2 W)) but over the head blocks [0, c0b) only
template <int W, int P, int NV, int NPAD>
__device__ __forceinline__ float p2_group_keep(const float *sU, const float *sL, const int (&li)[8],
                                               const float4 (&yq)[NV], const float4 (&luq)[NV],
                                               const float4 (&ulq)[NV], float (&c0)[4], float (&c1)[4],
                                               int c0b, float &hd, int lane) {
    static_assert(W <= 4 && NV <= 2, "REC groups are at most 4 wide");
    float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float h[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const float4 y = yq[v], lu = luq[v], ul = ulq[v];
#pragma unroll
        for (int u = 0; u < W; ++u) {
            const int off = li[u] * NPAD + 4 * lane + 128 * v;
            const float4 ux = *reinterpret_cast<const float4 *>(sU + off);
            const float4 lx = *reinterpret_cast<const float4 *>(sL + off);
            float t = 0.f;
            t = accp<P>(t, max3f(y.x - fmaxf(ux.x, lu.x), fminf(lx.x, ul.x) - y.x, 0.f));
            t = accp<P>(t, max3f(y.y - fmaxf(ux.y, lu.y), fminf(lx.y, ul.y) - y.y, 0.f));
            t = accp<P>(t, max3f(y.z - fmaxf(ux.z, lu.z), fminf(lx.z, ul.z) - y.z, 0.f));
            t = accp<P>(t, max3f(y.w - fmaxf(ux.w, lu.w), fminf(lx.w, ul.w) - y.w, 0.f));
            if (v == 0) { c0[u] = t; h[u] = lane < c0b ? t : 0.f; } else { c1[u] = t; }
            s[u] += t;
        }
    }
    if constexpr (NV == 1) {
#pragma unroll
        for (int u = 0; u < W; ++u) c1[u] = 0.f;
    }
    hd = reduceW<W>(h, lane);
    return reduceW<W>(s, lane);
}

// Column part of the DTW walk's abandon schedule for one appended pair (DESIGN.md reading
// c22), written to dst[0..32) as fp16: dst[0] = h0 = rd(sum_{c >= 4 c0b} beta2_c) and, for
// k = 0..30, dst[1 + k] = ru(E[k]), E[k] = sum_{c in [8k, 8k + 8) + 4 c0b} beta2_c, with
// beta2_c = d(y_c, [L(H)_c, U(H)_c])^p (the closed form above) and 4 c0b >= w.  The walk adds
// dst[0] to its row cascade (+-beta1 minus the computed rows' LB_Keogh terms) at its first
// test and subtracts E[k] after rows 8k .. 8k+7: after 8(k+1) rows the column part is <= the
// sum over columns >= 8(k+1) + w, which every completion visits (no computed row reaches
// them), and each of its cells (r, c) costs at least the row term of r plus the column term
// of c (Theorem 1's split), so rowmin + rest bounds DTW^p.  pc0 / pc1: this lane's
// pair sums of the 4-sample blocks (b, b + 1), b = lane + 32 v; block b starts word
// 1 + (b - c0b) / 2 when b - c0b is even; the words past the last block are 0.
template <int NV>
__device__ __forceinline__ void write_col_schedule(float pc0, float pc1, float h0, int c0b, __half *dst, int lane) {
    const int d0 = lane - c0b;
    if (d0 >= 0 && !(d0 & 1)) dst[1 + (d0 >> 1)] = __float2half_ru(pc0);
    if constexpr (NV == 2) {
        const int d1 = d0 + 32;
        if (!(d1 & 1) && d1 <= 60) dst[1 + (d1 >> 1)] = __float2half_ru(pc1);
    }
    if (lane >= 1 && 2 * (lane - 1) + c0b >= 32 * NV) dst[lane] = __float2half_rz(0.f);
    if (lane == 0) dst[0] = __float2half_rd(h0);
}

// the look-ahead entry's 64-bit survivor mask as two words, loaded by volatile asm straight into the
// loop-carried registers (a C++ load went to a scratch pair and was moved into place at once)
__device__ __forceinline__ void ld_mask2(const unsigned *p, unsigned &lo, unsigned &hi) {
    asm volatile("ld.global.v2.u32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "l"(p));
}

template <int P, int EPL, bool B1X, bool KO, bool DENSE, bool REC>
__global__ void __launch_bounds__(ImpCfg<EPL, B1X>::NT, 1)
improved_kernel(ImprovedArgs a, int Ct) {
    constexpr int NT = ImpCfg<EPL, B1X>::NT;
    constexpr bool PREFETCH = ImpCfg<EPL, B1X>::PREFETCH;
    constexpr int NW = NT / 32;
    constexpr int NV = EPL / 4;
    constexpr int NPAD = 32 * EPL;
    extern __shared__ __align__(16) float sm[];
    // [Ct][NPAD] blocks: x (B1X), U(x), L(x) (!KO); then per warp: the survivor list of
    // the current phase (local rows, 68 ints), the phase-2 list (68 ints) and its beta1 (64)
    float *sX = sm;
    float *sU = sm + (B1X ? (size_t)Ct * NPAD : 0);
    float *sL = sU + (KO ? 0 : (size_t)Ct * NPAD);
    int *sW = reinterpret_cast<int *>(sL + (KO ? 0 : (size_t)Ct * NPAD));

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int subs = 64 / Ct;
    const int64_t tile = blockIdx.x / subs;
    const int sub = (int)(blockIdx.x - tile * subs);
    const int64_t c0t = tile * 64;               // first candidate of the 64-tile
    const int64_t c0 = c0t + (int64_t)sub * Ct;  // first candidate staged by this CTA
    if (c0 >= a.N) return;
    const int cnt = a.tile_cnt[tile];
    if (cnt == 0) return;
    if (a.n_entries && sub == 0 && threadIdx.x == 0) atomicAdd(a.n_entries, (unsigned long long)cnt);
    const int ct = (int)((a.N - c0) < Ct ? (a.N - c0) : Ct);
    const int n = a.n;
    const unsigned long long ctmask = Ct == 64 ? ~0ull : ((1ull << Ct) - 1);

    // stage the tile: x padded with 0 (the query's padded U = +inf, L = -inf give d = 0);
    // U(x) = +inf, L(x) = -inf padding gives d = 0 in phase 2.  n % 4 == 0: 16-byte cp.async
    // copies (all of a thread's copies in flight at once), pads by plain stores
    if (n % 4 == 0) {
        constexpr int V = NPAD / 4;
        for (int t = threadIdx.x; t < Ct * V; t += NT) {
            const int r = t / V, i = 4 * (t - r * V);
            const int o = r * NPAD + i;
            if (r < ct && i < n) {
                const int64_t g = (c0 + r) * (int64_t)n + i;
                if constexpr (B1X) cp_async16(sX + o, a.xdb + g, 16);
                if constexpr (!KO) {
                    cp_async16(sU + o, a.Ux + g, 16);
                    cp_async16(sL + o, a.Lx + g, 16);
                }
            } else {
                if constexpr (B1X) *reinterpret_cast<float4 *>(sX + o) = make_float4(0.f, 0.f, 0.f, 0.f);
                if constexpr (!KO) {
                    *reinterpret_cast<float4 *>(sU + o) = make_float4(kInf, kInf, kInf, kInf);
                    *reinterpret_cast<float4 *>(sL + o) = make_float4(-kInf, -kInf, -kInf, -kInf);
                }
            }
        }
        cp_commit();
        cp_wait<0>();
    } else
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

    int *lst1 = sW + warp * 296;   // 72 ints (phase 1; reused for the phase-2b list)
    int *lst2 = lst1 + 72;         // 72 ints
    float *b1v = reinterpret_cast<float *>(lst2 + 72);  // 72 floats
    float *b1w = b1v + 72;                              // 72 floats (phase 2a partial bounds)
    unsigned long long evals1 = 0, evals2 = 0;
    const int *eq = a.tile_q + tile * a.Qb;
    const unsigned long long *em = a.tile_m + tile * a.Qb;
    const int u_me = lane >> 3;  // survivor slot this lane ends up holding after reduce4
    const bool lead8 = (lane & 7) == 0;
    const unsigned lt = (1u << lane) - 1u;
    // this warp's entries are e = warp, warp + NW, ...; with several CTAs per 64-tile
    // (Ct < 64) an entry may have no survivor in this CTA's part: seek skips those 32
    // entries at a time (one coalesced read of their masks, one ballot)
    auto seek = [&](int e0, unsigned long long &m) -> int {
        while (e0 < cnt) {
            const int ee = e0 + NW * lane;
            const unsigned long long mm = ee < cnt ? (em[ee] >> (sub * Ct)) & ctmask : 0ull;
            const unsigned bal = __ballot_sync(0xffffffffu, mm != 0ull);
            if (bal) {
                const int src = __ffs(bal) - 1;
                m = __shfl_sync(0xffffffffu, mm, src);
                return e0 + NW * src;
            }
            e0 += NW * 32;
        }
        return cnt;
    };
    // n <= 256: Ct = 64, one CTA per 64-tile and every listed entry has survivors here
    constexpr bool ONE_CTA = NPAD * 64 <= 16384;
    unsigned long long mcur = 0;
    int e = warp;
    if (ONE_CTA || subs == 1) {
        if (e >= cnt) return;
        mcur = em[e];
    } else {
        e = seek(warp, mcur);
        if (e >= cnt) return;
    }
    QRegs<NV, B1X, KO> cur, nxt;
    int64_t qe = eq[e];
    load_p1<EPL, B1X, KO>(cur, a, qe, c0t, lane);
    // one CTA per tile: the (query, mask) of the entry after next is loaded one iteration
    // ahead, so the next entry's query-row loads do not wait on its index load
    constexpr bool IDX_AHEAD = ONE_CTA;
    int q_ah = 0;
    unsigned m_ah_lo = 0, m_ah_hi = 0;  // (two 32-bit words: see below)
    // (the mask as two 32-bit words at a clamped index: as one 64-bit value the compiler loaded it into
    // a scratch pair and moved it into place at once -- a full L2 wait per entry, 9.8 % of the kernel's
    // stall samples on that one MOV, `profiles/r02zl_C5_improved_kernel_1_sass_top.txt`)
    const unsigned *em32 = reinterpret_cast<const unsigned *>(em);
    if (IDX_AHEAD) { const int ia = min(e + NW, cnt - 1); q_ah = eq[ia]; ld_mask2(em32 + 2 * ia, m_ah_lo, m_ah_hi); }
    while (true) {
        unsigned long long mn = 0;
        unsigned t_lo = 0, t_hi = 0;  // the look-ahead mask in flight; becomes m_ah at the end of the iteration
        int en = e + NW;
        if (!ONE_CTA && subs != 1) en = seek(en, mn);
        const bool more = en < cnt;
        int64_t qn = 0;
        if (more) {
            if constexpr (IDX_AHEAD) {
                qn = q_ah;
                mn = ((unsigned long long)m_ah_hi << 32) | m_ah_lo;
                { const int ia = min(en + NW, cnt - 1); q_ah = eq[ia]; ld_mask2(em32 + 2 * ia, t_lo, t_hi); }
            } else {
                qn = eq[en];
                if (ONE_CTA || subs == 1) mn = em[en];
            }
            if constexpr (PREFETCH) load_p1<EPL, B1X, KO>(nxt, a, qn, c0t, lane);
        }
        if (PREFETCH && mcur) load_p2<EPL, B1X, KO>(cur, a, qe, lane);  // in flight during phase 1
        const int64_t q = qe;
        // (REC) the query's schedule offset: issued here so that phase 1 covers its latency (read
        // at the start of phase 2 it was a dependent L2 load per entry, 6.8 % of the stall samples)
        // (32 bits: the host enables schedules only below 2^31 keys per range)
        int roff_c = 0;
        if constexpr (REC) roff_c = (int)__ldg(a.rec_off + q);
        __half *gq = a.gate_w ? a.gate_w + q * a.ldb + c0 : nullptr;
        // ---------------- phase 1: beta1 (B1X) of the gate survivors -> phase-2 list
        // groups of 4 survivors; a tail of 1 or 2 runs as a 1- or 2-wide group (lane l then
        // holds slot l >> 5-log2(W)), so few slots are spent on padding
        int n2 = 0;
        if constexpr (B1X) {
            const int n1 = compact_mask(mcur, lst1, lane);
            __syncwarp();
            evals1 += n1;
            auto phase1 = [&](auto wc, int g) {
                constexpr int W = decltype(wc)::value;
                constexpr int SH = W == 8 ? 2 : (W == 4 ? 3 : (W == 2 ? 4 : 5));
                int li[8];
                read_group<W>(lst1, g, li);
                const float b1 = p1_group<W, P, NV, NPAD>(sX, li, cur.u, cur.l, lane);
                const int us = lane >> SH;
                const int myl = W == 1 ? li[0] : lst1[g + us];
                const bool pass = (lane & ((1 << SH) - 1)) == 0 && g + us < n1 && (DENSE || b1 <= cur.thr);
                if constexpr (!DENSE) {
                    // keep beta1 for the DTW walk's cascading abandon: the gate slot (beta0,
                    // already consumed by this range's mask) takes -beta1 (<= 0, so no later
                    // range re-selects it; the walk reads |.|)
                    if (pass) gq[myl] = __hneg(__float2half_rd(b1));
                }
                if constexpr (KO) {
                    if constexpr (DENSE) {
                        if (pass) a.dense[q * a.ldd + c0 + myl] = rootp<P>(b1);
                    } else {
                        append_keys(a, q, pass, b1, c0 + myl, lane);
                    }
                } else {
                    const unsigned bal = __ballot_sync(0xffffffffu, pass);
                    if (pass) {
                        const int pos = n2 + __popc(bal & lt);
                        lst2[pos] = myl;
                        b1v[pos] = b1;
                    }
                    n2 += __popc(bal);
                }
            };
            int g = 0;
            for (; n1 - g >= 7; g += 8) phase1(std::integral_constant<int, 8>{}, g);
            for (; n1 - g >= 3; g += 4) phase1(std::integral_constant<int, 4>{}, g);
            if (n1 - g == 2) phase1(std::integral_constant<int, 2>{}, g);
            else if (n1 - g == 1) phase1(std::integral_constant<int, 1>{}, g);
            if constexpr (!KO) {
                if (lane < ((8 - (n2 & 7)) & 7)) lst2[n2 + lane] = 0;
            }
            __syncwarp();
        } else {
            n2 = compact_mask(mcur, lst2, lane);
            __syncwarp();
        }
        // ---------------- phase 2: beta2, LB_Improved^p = beta1 + beta2
        // LIST mode, n > 256: in two halves.  2a: beta1 + beta2 over the first half of the
        // samples (a lower bound of LB_Improved^p, so pruning on it is exact) for every
        // phase-2 survivor; 2b: the second half only for the pairs 2a kept (~half of them
        // fail already at 2a on C5: saves ~1/4 of the phase-2 work)
        // (n <= 256, NV = 2: the extra reduction per group costs more than it saves -- measured)
        constexpr bool SPLIT = !DENSE && !KO && NV >= 4;
        if constexpr (SPLIT) {
            if (!PREFETCH && n2) load_p2<EPL, B1X, KO>(cur, a, q, lane);
            evals2 += n2;
            int n3 = 0;
            auto phase2a = [&](auto wc, int g) {
                constexpr int W = decltype(wc)::value;
                constexpr int SH = W == 8 ? 2 : (W == 4 ? 3 : (W == 2 ? 4 : 5));
                int li[8];
                read_group<W>(lst2, g, li);
                const float b2 = p2_group<W, P, NV, NPAD, 0, NV / 2>(sU, sL, li, cur.y, cur.lu, cur.ul, lane);
                const int us = lane >> SH;
                const int myl = W == 1 ? li[0] : lst2[g + us];
                float b1;
                if constexpr (B1X) {
                    b1 = b1v[min(g + us, n2 - 1)];
                } else {
                    const int t64 = sub * Ct + myl;  // slot in the 64-tile
                    const float va = __shfl_sync(0xffffffffu, cur.b1a, t64 & 31);
                    const float vb = __shfl_sync(0xffffffffu, cur.b1b, t64 & 31);
                    b1 = t64 < 32 ? va : vb;
                }
                const float part = b1 + b2;
                const bool alive = (lane & ((1 << SH) - 1)) == 0 && g + us < n2 && part <= cur.thr;
                const unsigned bal = __ballot_sync(0xffffffffu, alive);
                if (alive) {
                    const int pos = n3 + __popc(bal & lt);
                    lst1[pos] = myl;
                    b1w[pos] = part;
                }
                n3 += __popc(bal);
            };
            int g = 0;
            for (; n2 - g >= 7; g += 8) phase2a(std::integral_constant<int, 8>{}, g);
            for (; n2 - g >= 3; g += 4) phase2a(std::integral_constant<int, 4>{}, g);
            if (n2 - g == 2) phase2a(std::integral_constant<int, 2>{}, g);
            else if (n2 - g == 1) phase2a(std::integral_constant<int, 1>{}, g);
            if (lane < ((8 - (n3 & 7)) & 7)) lst1[n3 + lane] = 0;
            __syncwarp();
            auto phase2b = [&](auto wc, int g) {
                constexpr int W = decltype(wc)::value;
                constexpr int SH = W == 8 ? 2 : (W == 4 ? 3 : (W == 2 ? 4 : 5));
                int li[8];
                read_group<W>(lst1, g, li);
                const float b2 = p2_group<W, P, NV, NPAD, NV / 2, NV>(sU, sL, li, cur.y, cur.lu, cur.ul, lane);
                const int us = lane >> SH;
                const int myl = W == 1 ? li[0] : lst1[g + us];
                const float beta = b1w[min(g + us, n3 - 1)] + b2;
                const bool lead = (lane & ((1 << SH) - 1)) == 0 && g + us < n3;
                append_keys(a, q, lead && beta <= cur.thr, beta, c0 + myl, lane);
            };
            g = 0;
            for (; n3 - g >= 7; g += 8) phase2b(std::integral_constant<int, 8>{}, g);
            for (; n3 - g >= 3; g += 4) phase2b(std::integral_constant<int, 4>{}, g);
            if (n3 - g == 2) phase2b(std::integral_constant<int, 2>{}, g);
            else if (n3 - g == 1) phase2b(std::integral_constant<int, 1>{}, g);
        } else if constexpr (!KO) {
            if (!PREFETCH && n2) load_p2<EPL, B1X, KO>(cur, a, q, lane);
            evals2 += n2;
            // abandon schedules (reading c22): the appended pairs' (local row, list position)
            // go to lst1 / b1w (free after phase 1), then one warp pass per pair
            static_assert(!REC || (B1X && !DENSE && NV <= 2), "abandon schedules: pre-filtered LIST mode, n <= 256");
            __half *rq = nullptr;  // (REC) this query's schedules
            if constexpr (REC) rq = a.rec + (int64_t)roff_c * 32;
            auto phase2 = [&](auto wc, int g) {
                constexpr int W = decltype(wc)::value;
                constexpr int SH = W == 8 ? 2 : (W == 4 ? 3 : (W == 2 ? 4 : 5));
                int li[8];
                read_group<W>(lst2, g, li);
                float kc0[4], kc1[4], hd = 0.f;  // (REC) per-block column partials, head sums
                float b2;
                if constexpr (REC)
                    b2 = p2_group_keep<W, P, NV, NPAD>(sU, sL, li, cur.y, cur.lu, cur.ul, kc0, kc1, a.rec_c0b, hd, lane);
                else
                    b2 = p2_group<W, P, NV, NPAD>(sU, sL, li, cur.y, cur.lu, cur.ul, lane);
                const int us = lane >> SH;
                const int myl = W == 1 ? li[0] : lst2[g + us];
                float b1;
                if constexpr (B1X) {
                    b1 = b1v[min(g + us, n2 - 1)];
                } else {
                    const int t64 = sub * Ct + myl;  // slot in the 64-tile
                    const float va = __shfl_sync(0xffffffffu, cur.b1a, t64 & 31);
                    const float vb = __shfl_sync(0xffffffffu, cur.b1b, t64 & 31);
                    b1 = t64 < 32 ? va : vb;
                }
                const float beta = b1 + b2;
                const bool lead = (lane & ((1 << SH) - 1)) == 0 && g + us < n2;
                if constexpr (DENSE) {
                    if (lead) a.dense[q * a.ldd + c0 + myl] = rootp<P>(beta);
                } else {
                    const bool pass = lead && beta <= cur.thr;
                    if constexpr (REC) {
                        // append_keys inlined: the pair-sum shuffles (independent of the list
                        // position) issue between the atomic and the first use of its result, and
                        // the list base reuses the schedule offset when both are the exact-count
                        // offsets (no second dependent load)
                        unsigned bal = __ballot_sync(0xffffffffu, pass);
                        if (bal) {
                            int base = 0;
                            if (lane == 0) base = atomicAdd(a.list_len + q, __popc(bal));
                            // pair sums of adjacent blocks for the whole group (independent shuffles)
                            const int nx = (lane + 1) & 31;
#pragma unroll
                            for (int t = 0; t < W; ++t) {
                                const float n0 = __shfl_sync(0xffffffffu, kc0[t], nx);
                                const float n1 = NV == 2 ? __shfl_sync(0xffffffffu, kc1[t], nx) : 0.f;
                                kc0[t] += lane == 31 ? n1 : n0;
                                kc1[t] += lane == 31 ? 0.f : n1;
                            }
                            const float h0 = b2 - hd;  // (lead lanes: their survivor's column suffix)
                            base = __shfl_sync(0xffffffffu, base, 0);
                            int pos = -1;
                            if (pass) {
                                pos = base + __popc(bal & lt);
                                const int64_t lb = a.loff == a.rec_off ? (int64_t)roff_c : list_base(a.loff, a.cap, q);
                                DCHECK(a.loff ? a.loff[q] + pos < a.loff[q + 1] : pos < a.cap, "list append q=%lld pos=%d", (long long)q, pos);
                                a.list[lb + pos] = pack_list_key(beta, (uint32_t)(c0 + myl), pos);
                            }
                            // the passing survivors' schedules, one warp pass each, from the
                            // partials every lane still holds
                            do {
                                const int src = __ffs(bal) - 1;
                                bal &= bal - 1;
                                const int u = src >> SH;
                                const int ps = __shfl_sync(0xffffffffu, pos, src);
                                const float hu = __shfl_sync(0xffffffffu, h0, src);
                                float v0 = kc0[0], v1 = kc1[0];
#pragma unroll
                                for (int t = 1; t < W; ++t)
                                    if (u == t) { v0 = kc0[t]; v1 = kc1[t]; }
                                write_col_schedule<NV>(v0, v1, hu, a.rec_c0b, rq + (int64_t)ps * 32, lane);
                            } while (bal);
                        }
                    } else {
                        append_keys(a, q, pass, beta, c0 + myl, lane);
                    }
                }
            };
            int g = 0;
            if constexpr (!REC)
                for (; n2 - g >= 7; g += 8) phase2(std::integral_constant<int, 8>{}, g);
            for (; n2 - g >= 3; g += 4) phase2(std::integral_constant<int, 4>{}, g);
            if (n2 - g == 2) phase2(std::integral_constant<int, 2>{}, g);
            else if (n2 - g == 1) phase2(std::integral_constant<int, 1>{}, g);
        } else if constexpr (!B1X) {
            // Alg. 2 (keogh-only) over the dense beta1 block: the gate survivors are the keys
            for (int g = 0; g < n2; g += 4) {
                const int4 li = *reinterpret_cast<const int4 *>(lst2 + g);
                const int nb = min(4, n2 - g);
                const int myl = pick4(li, u_me);
                const int t64 = sub * Ct + myl;
                const float va = __shfl_sync(0xffffffffu, cur.b1a, t64 & 31);
                const float vb = __shfl_sync(0xffffffffu, cur.b1b, t64 & 31);
                const float b1 = t64 < 32 ? va : vb;
                const bool lead = lead8 && u_me < nb;
                if constexpr (DENSE) {
                    if (lead) a.dense[q * a.ldd + c0 + myl] = rootp<P>(b1);
                } else {
                    append_keys(a, q, lead && b1 <= cur.thr, b1, c0 + myl, lane);
                }
            }
        }
        __syncwarp();
        if (!more) break;
        if constexpr (PREFETCH) {
            if constexpr (B1X) {
#pragma unroll
                for (int v = 0; v < NV; ++v) { cur.u[v] = nxt.u[v]; cur.l[v] = nxt.l[v]; }
            } else {
                cur.b1a = nxt.b1a;
                cur.b1b = nxt.b1b;
            }
            cur.thr = nxt.thr;
        } else {
            load_p1<EPL, B1X, KO>(cur, a, qn, c0t, lane);
        }
        e = en;
        qe = qn;
        mcur = mn;
        if constexpr (IDX_AHEAD) { m_ah_lo = t_lo; m_ah_hi = t_hi; }
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
    const size_t smem = (size_t)arrays * Ct * NPAD * sizeof(float) + (size_t)(NT / 32) * 296 * sizeof(int);
    auto k = improved_kernel<P, EPL, B1X, KO, DENSE, false>;
    if constexpr (B1X && !KO && !DENSE && EPL <= 8) {
        if (a.rec) k = improved_kernel<P, EPL, B1X, KO, DENSE, true>;  // + abandon schedules (c22)
    }
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

namespace {

// Any n (the dense lb_improved entry point for n > 1024, beyond the survivor kernel's register
// layout): one warp per (query, candidate) pair, lanes striding over i, the same closed form
// for the envelope of H; out = rooted(beta1 + beta2) with beta1 from the dense LB_Keogh pass.
template <int P>
__global__ void __launch_bounds__(256) improved_generic_kernel(const float *__restrict__ y, const float *__restrict__ LU,
                                                               const float *__restrict__ UL, const float *__restrict__ Ux,
                                                               const float *__restrict__ Lx, const float *__restrict__ beta1,
                                                               int64_t ldb, int64_t Q, int64_t N, int n,
                                                               float *__restrict__ out, int64_t ldd) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t pr = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; pr < Q * N; pr += nw) {
        const int64_t q = pr / N, c = pr - q * N;
        const float *yr = y + q * n, *lur = LU + q * n, *ulr = UL + q * n;
        const float *uxr = Ux + c * n, *lxr = Lx + c * n;
        float acc = 0.f;
        for (int i = lane; i < n; i += 32)
            acc = accp<P>(acc, max3f(yr[i] - fmaxf(__ldg(uxr + i), lur[i]), fminf(__ldg(lxr + i), ulr[i]) - yr[i], 0.f));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) out[q * ldd + c] = rootp<P>(__ldg(beta1 + q * ldb + c) + acc);
    }
}

}  // namespace

int launch_improved_generic(const float *y, const float *LU, const float *UL, const float *Ux, const float *Lx,
                            const float *beta1, int64_t ldb, int64_t Q, int64_t N, int n, int p, float *out,
                            int64_t ldd, cudaStream_t st) {
    if (Q == 0 || N == 0) return DTWLB_OK;
    const int64_t warps = Q * N;
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(warps * 32, 256), 148 * 64);
    if (p == 1)
        improved_generic_kernel<1><<<grid, 256, 0, st>>>(y, LU, UL, Ux, Lx, beta1, ldb, Q, N, n, out, ldd);
    else
        improved_generic_kernel<2><<<grid, 256, 0, st>>>(y, LU, UL, Ux, Lx, beta1, ldb, Q, N, n, out, ldd);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

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

int launch_select(const ImprovedArgs &a, bool dense, cudaStream_t st) {
    if (a.Qb == 0 || a.N == 0) return DTWLB_OK;
    const int64_t ntiles = ceil_div(a.N, 64);
    // per-tile (query, survivor mask) lists into the caller-provided scratch
    DTWLB_CUDA(cudaMemsetAsync(a.tile_cnt, 0, sizeof(int) * ntiles, st));
    const int64_t warps = ntiles * ceil_div(a.Qb, 32);
    if (a.gate_half && a.ldb % 8 == 0) {
        const int64_t warps8 = ceil_div(ntiles, 4) * ceil_div(a.Qb, 32);
        select_mask8_kernel<<<(unsigned)ceil_div(warps8 * 32, 256), 256, 0, st>>>(
            static_cast<const __half *>(a.gate), a.ldb, a.Qb, a.N, a.lo, a.hi, a.thr, dense, a.tile_m, a.tile_q,
            a.tile_cnt, ntiles, a.q_count);
    } else if (a.gate_half)
        select_mask_kernel<__half><<<(unsigned)ceil_div(warps * 32, 256), 256, 0, st>>>(
            static_cast<const __half *>(a.gate), a.ldb, a.Qb, a.N, a.lo, a.hi, a.thr, dense, a.tile_m, a.tile_q,
            a.tile_cnt, ntiles, a.q_count);
    else
        select_mask_kernel<float><<<(unsigned)ceil_div(warps * 32, 256), 256, 0, st>>>(
            static_cast<const float *>(a.gate), a.ldb, a.Qb, a.N, a.lo, a.hi, a.thr, dense, a.tile_m, a.tile_q,
            a.tile_cnt, ntiles, a.q_count);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

int launch_survivor(const ImprovedArgs &a, int p, bool keogh_only, bool dense, cudaStream_t st) {
    if (a.Qb == 0 || a.N == 0) return DTWLB_OK;
    const int64_t ntiles = ceil_div(a.N, 64);
    const int epl = a.npadE / 32;
    if (a.ev0) DTWLB_CUDA(cudaEventRecord(a.ev0, st));
    const int rc = p == 1 ? launch_imp_p<1>(a, epl, keogh_only, dense, ntiles, st)
                          : launch_imp_p<2>(a, epl, keogh_only, dense, ntiles, st);
    if (a.ev1) DTWLB_CUDA(cudaEventRecord(a.ev1, st));
    return rc;
}

int launch_improved(const ImprovedArgs &a, int p, bool keogh_only, bool dense, cudaStream_t st) {
    DTWLB_TRY(launch_select(a, dense, st));
    return launch_survivor(a, p, keogh_only, dense, st);
}

}  // namespace dtwlb
