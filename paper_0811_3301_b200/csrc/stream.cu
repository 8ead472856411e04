// stream.cu -- the LB_Keogh pass (a2) for a FEW queries: one streaming pass over the
// database (SURVEY 8(d) "C5-stream": Q <= 8, the regime where the bound pass is
// HBM-bound).  P:453-464, Alg. 2/3 lines P:507-514 / P:589-597:
//
//   beta1(q, c) = sum_i d(x_c,i, [L_q,i, U_q,i])^p,  d(v,[a,b]) = max(v - b, a - v, 0)
//
// This is the paper's own per-query scan shape -- Alg. 2/3 stream the whole database
// for one query, (2N+3)n comparisons -- with up to QB = 8
// queries sharing one read of the database.
//
// B200 design: thread = candidate.  A persistent CTA of 256 threads walks tiles of 256
// database rows; each row is copied chunk by chunk (KCH floats) from HBM into the
// thread's own shared-memory slot by a TMA bulk copy (cp.async.bulk, no tensor map:
// a row chunk is contiguous) that completes on the thread's own mbarrier, D stages
// deep, so ~D-1 chunks per row (~100 KB per SM) are in flight while the thread
// computes on the oldest one.  Every thread reads only the slot it filled itself, so
// there is no CTA-wide synchronisation in the loop.  The QB query envelopes sit in
// shared memory and are read as 128-bit broadcasts (every lane the same address);
// per pair-element the minimal FADD2 (two subtractions of two elements), FMNMX3,
// FFMA|FADD (3 issue slots per element, the x value reused by all QB queries).
// Per-chunk partial sums are folded into the total at each chunk end (two-level
// summation, as the tile kernel).  Output beta1 (p-th power, fp32) [Q][ldo].
// A cp.async (LDGSTS) variant of the same loop (COPY = 1: each warp copies its 32 rows
// cooperatively, 128-byte coalesced segments) is kept for comparison.
#include <cudaTypedefs.h>  // CUtensorMap, PFN_cuTensorMapEncodeTiled (driver entry point, no -lcuda)

#include "kernels.cuh"

namespace dtwlb {

namespace {

constexpr int kStreamNT = 256;  // threads (= candidate rows) per CTA
constexpr int kKch = 32;        // floats per row chunk (128-byte copies)
constexpr int kSlot = kKch + 4; // padded slot pitch (floats): conflict-free 128-bit reads

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// TMA bulk copy global -> shared (1D, bytes % 16 == 0, both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// 128-bit shared-memory load by 32-bit shared address (forces LDS: pointers derived from the
// dynamic shared array through address arithmetic otherwise compile to generic loads)
__device__ __forceinline__ float4 lds128(unsigned a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
// order this thread's earlier generic-proxy reads of its slot before the next async write
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

template <int P>
__device__ __forceinline__ float lb4(float acc, const float4 &x, const float4 &u, const float4 &l) {
    // d = max(x - U, L - x, 0) on two elements at a time (packed f32x2 subtractions)
    const float2 a0 = __fadd2_rn(make_float2(x.x, x.y), make_float2(-u.x, -u.y));
    const float2 b0 = __fadd2_rn(make_float2(l.x, l.y), make_float2(-x.x, -x.y));
    const float2 a1 = __fadd2_rn(make_float2(x.z, x.w), make_float2(-u.z, -u.w));
    const float2 b1 = __fadd2_rn(make_float2(l.z, l.w), make_float2(-x.z, -x.w));
    acc = accp<P>(acc, max3f(a0.x, b0.x, 0.f));
    acc = accp<P>(acc, max3f(a0.y, b0.y, 0.f));
    acc = accp<P>(acc, max3f(a1.x, b1.x, 0.f));
    acc = accp<P>(acc, max3f(a1.y, b1.y, 0.f));
    return acc;
}

// COPY: 0 = TMA bulk copies (per thread, own mbarrier), 1 = cp.async per warp.
template <int P, int QB, int COPY>
__global__ void __launch_bounds__(kStreamNT, 1)
keogh_stream_kernel(const float *__restrict__ U, const float *__restrict__ L, const float *__restrict__ db,
                    int64_t N, int n, int Q, int D, bool rooted, float *__restrict__ out, int64_t ldo) {
    extern __shared__ __align__(128) unsigned char smraw[];
    const int npad = (n + kKch - 1) / kKch * kKch;
    const int nch = npad / kKch;
    float *sU = reinterpret_cast<float *>(smraw);       // [QB][npad]
    float *sL = sU + (size_t)QB * npad;                 // [QB][npad]
    float *slots = sL + (size_t)QB * npad;              // [D][NT][kSlot]
    uint64_t *bars = reinterpret_cast<uint64_t *>(slots + (size_t)D * kStreamNT * kSlot);  // [D][NT]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // query envelopes; pad columns (i >= n) and missing queries: U = +inf, L = -inf (d = 0)
    for (int t = tid; t < QB * npad; t += kStreamNT) {
        const int q = t / npad, i = t - q * npad;
        const bool ok = q < Q && i < n;
        sU[t] = ok ? U[(int64_t)q * n + i] : kInf;
        sL[t] = ok ? L[(int64_t)q * n + i] : -kInf;
    }
    for (int t = tid; t < D * kStreamNT * kSlot; t += kStreamNT) slots[t] = 0.f;
    if constexpr (COPY == 0) {
        for (int s = 0; s < D; ++s) mbar_init(bars + s * kStreamNT + tid, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    const int64_t ntiles = (N + kStreamNT - 1) / kStreamNT;
    const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t steps = my_tiles * nch;  // (tile, chunk) steps of this CTA, same for every thread

    // issue the copy of step g into stage g % D
    auto issue = [&](int64_t g) {
        const int64_t ti = g / nch;
        const int ch = (int)(g - ti * nch);
        const int64_t tile = blockIdx.x + ti * gridDim.x;
        const int s = (int)(g % D);
        const int k0 = ch * kKch;
        const int len = min(kKch, n - k0);  // floats (n % 4 == 0: a multiple of 4)
        if constexpr (COPY == 0) {
            const int64_t c = tile * kStreamNT + tid;
            if (c < N) {
                float *dst = slots + ((size_t)s * kStreamNT + tid) * kSlot;
                fence_proxy_async();
                mbar_expect_tx(bars + s * kStreamNT + tid, (unsigned)len * 4u);
                bulk_g2s(dst, db + c * (int64_t)n + k0, (unsigned)len * 4u, bars + s * kStreamNT + tid);
            }
        } else {
            // warp copies its 32 rows: each instruction moves 4 rows x 128 bytes (8 lanes per row)
            const int sub = lane & 7, rr = lane >> 3;
#pragma unroll
            for (int r0 = 0; r0 < 32; r0 += 4) {
                const int row = warp * 32 + r0 + rr;
                const int64_t c = tile * kStreamNT + row;
                const bool ok = c < N && 4 * sub < len;
                float *dst = slots + ((size_t)s * kStreamNT + row) * kSlot + 4 * sub;
                cp_async16(dst, ok ? db + c * (int64_t)n + k0 + 4 * sub : db, ok ? 16 : 0);
            }
            cp_commit();
        }
    };

    float acc[QB];
#pragma unroll
    for (int q = 0; q < QB; ++q) acc[q] = 0.f;
    const int64_t pro = steps < D - 1 ? steps : D - 1;
    for (int64_t g = 0; g < pro; ++g) issue(g);
    for (int64_t g = 0; g < steps; ++g) {
        if (g + D - 1 < steps) issue(g + D - 1);
        else if constexpr (COPY == 1) cp_commit();  // keep the group count uniform
        const int64_t ti = g / nch;
        const int ch = (int)(g - ti * nch);
        const int64_t c = (blockIdx.x + ti * gridDim.x) * kStreamNT + tid;
        const int s = (int)(g % D);
        if constexpr (COPY == 0) {
            if (c < N) mbar_wait(bars + s * kStreamNT + tid, (unsigned)((g / D) & 1));
        } else {
            switch (D - 1) {  // (wait_group takes an immediate)
                case 1: cp_wait<1>(); break;
                case 2: cp_wait<2>(); break;
                case 3: cp_wait<3>(); break;
                case 4: cp_wait<4>(); break;
                case 5: cp_wait<5>(); break;
                default: cp_wait<0>(); break;
            }
            __syncwarp();
        }
        const float *xs = slots + ((size_t)s * kStreamNT + tid) * kSlot;
        const int k0 = ch * kKch;
        float part[QB];
#pragma unroll
        for (int q = 0; q < QB; ++q) part[q] = 0.f;
#pragma unroll 2
        for (int e = 0; e < kKch; e += 4) {
            const float4 xv = *reinterpret_cast<const float4 *>(xs + e);
#pragma unroll
            for (int q = 0; q < QB; ++q) {
                const float4 u = *reinterpret_cast<const float4 *>(sU + (size_t)q * npad + k0 + e);
                const float4 l = *reinterpret_cast<const float4 *>(sL + (size_t)q * npad + k0 + e);
                part[q] = lb4<P>(part[q], xv, u, l);
            }
        }
#pragma unroll
        for (int q = 0; q < QB; ++q) acc[q] += part[q];
        if (ch == nch - 1) {
            if (c < N) {
#pragma unroll
                for (int q = 0; q < QB; ++q)
                    if (q < Q) out[(int64_t)q * ldo + c] = rooted ? rootp<P>(acc[q]) : acc[q];
            }
#pragma unroll
            for (int q = 0; q < QB; ++q) acc[q] = 0.f;
        }
        if constexpr (COPY == 1) __syncwarp();  // the slot is rewritten by the warp's next copy
    }
    if constexpr (COPY == 1) cp_wait<0>();
}

// ---------------------------------------------------------------------------------------
// COPY = 2 (default): 2D TMA.  The database is a [N][n] fp32 tensor map; a warp owns tiles of
// 32 rows and streams them through its own ring of D boxes of 32 rows x 32 floats (4 KB, one
// cp.async.bulk.tensor per box issued by lane 0, completing on the warp's mbarrier of that
// stage; out-of-range rows / columns are zero-filled by the TMA unit).  The boxes are written
// with the TMA 128-byte swizzle (16-byte chunk c of row r lands at chunk c ^ (r & 7)): lane t
// owns row t and reads logical chunk k at physical chunk k ^ (t & 7), so the 8 lanes of a
// quarter-warp hit 8 distinct bank groups, while every lane reads the SAME query-envelope
// chunk -- a shared-memory broadcast.  (An unswizzled, lane-rotated layout measured 0.55 ms at
// Q = 8, bound by the non-broadcast envelope reads.)
// R > 1: lane t owns rows t, t+32, .. of a 32R-row box, so every envelope chunk read from
// shared memory serves R rows (a 128-bit read costs 4 shared-memory wavefronts, broadcast or
// not: with R = 1 and Q >= 2 the envelope reads, not HBM, bounded the kernel).
constexpr int kBoxCols = 32;

template <int P, int QB, int R, int W>
__global__ void __launch_bounds__(W * 32, 1)
keogh_stream_tma_kernel(const __grid_constant__ CUtensorMap tmap, const float *__restrict__ U,
                        const float *__restrict__ L, int64_t N, int n, int Q, int D, bool rooted,
                        float *__restrict__ out, int64_t ldo) {
    extern __shared__ __align__(128) unsigned char smraw[];
    constexpr int ROWS = 32 * R;
    const int npad = (n + kBoxCols - 1) / kBoxCols * kBoxCols;
    const int nch = npad / kBoxCols;
    constexpr int BOX = ROWS * kBoxCols;  // floats (a multiple of the 1 KB swizzle atom)
    // (the dynamic shared-memory base is only guaranteed 16-byte aligned: round up to 1 KB)
    // (offset arithmetic on the shared array itself, not a uintptr_t round trip: the compiler
    // then keeps the shared address space and emits LDS, not generic loads)
    float *boxes = reinterpret_cast<float *>(smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u));
    float *sU = boxes + (size_t)W * D * BOX;  // [QB][npad]
    float *sL = sU + (size_t)QB * npad;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sL + (size_t)QB * npad);  // [W][D]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int t = tid; t < QB * npad; t += W * 32) {
        const int q = t / npad, i = t - q * npad;
        const bool ok = q < Q && i < n;
        sU[t] = ok ? U[(int64_t)q * n + i] : kInf;
        sL[t] = ok ? L[(int64_t)q * n + i] : -kInf;
    }
    if (lane == 0) {
        for (int s = 0; s < D; ++s) mbar_init(bars + warp * D + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    const int64_t ntiles = (N + ROWS - 1) / ROWS;
    const int64_t gw = (int64_t)blockIdx.x * W + warp, GW = (int64_t)gridDim.x * W;
    const int64_t my_tiles = gw < ntiles ? (ntiles - 1 - gw) / GW + 1 : 0;
    const int64_t steps = my_tiles * nch;
    float *mybox = boxes + (size_t)warp * D * BOX;
    uint64_t *mybar = bars + warp * D;
    auto issue = [&](int64_t g) {
        if (lane == 0) {
            const int64_t ti = g / nch;
            const int ch = (int)(g - ti * nch);
            const int64_t tile = gw + ti * GW;
            const int s = (int)(g % D);
            fence_proxy_async();
            mbar_expect_tx(mybar + s, (unsigned)(BOX * sizeof(float)));
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                "[%4];\n" ::"r"(smem_u32(mybox + (size_t)s * BOX)),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(ch * kBoxCols), "r"((int)(tile * ROWS)),
                "r"(smem_u32(mybar + s))
                : "memory");
        }
    };
    const int pro = (int)(steps < D - 1 ? steps : D - 1);
    for (int g = 0; g < pro; ++g) issue(g);
    const int swz = lane & 7;  // (rows lane + 32 i share lane & 7)
    float acc[QB][R];
#pragma unroll
    for (int q = 0; q < QB; ++q)
#pragma unroll
        for (int i = 0; i < R; ++i) acc[q][i] = 0.f;
    for (int64_t g = 0; g < steps; ++g) {
        if (g + D - 1 < steps) issue(g + D - 1);
        const int64_t ti = g / nch;
        const int ch = (int)(g - ti * nch);
        const int s = (int)(g % D);
        mbar_wait(mybar + s, (unsigned)((g / D) & 1));
        const unsigned xr = smem_u32(mybox) + (unsigned)(s * BOX + lane * kBoxCols) * 4u;
        const unsigned ub = smem_u32(sU) + (unsigned)(ch * kBoxCols) * 4u, lb = smem_u32(sL) + (unsigned)(ch * kBoxCols) * 4u;
        float part[QB][R];
#pragma unroll
        for (int q = 0; q < QB; ++q)
#pragma unroll
            for (int i = 0; i < R; ++i) part[q][i] = 0.f;
#pragma unroll
        for (int k = 0; k < kBoxCols / 4; ++k) {
            float4 xv[R];
#pragma unroll
            for (int i = 0; i < R; ++i) xv[i] = lds128(xr + (unsigned)(i * 32 * kBoxCols + 4 * (k ^ swz)) * 4u);
#pragma unroll
            for (int q = 0; q < QB; ++q) {
                const float4 u = lds128(ub + (unsigned)(q * npad + 4 * k) * 4u);
                const float4 l = lds128(lb + (unsigned)(q * npad + 4 * k) * 4u);
#pragma unroll
                for (int i = 0; i < R; ++i) part[q][i] = lb4<P>(part[q][i], xv[i], u, l);
            }
        }
#pragma unroll
        for (int q = 0; q < QB; ++q)
#pragma unroll
            for (int i = 0; i < R; ++i) acc[q][i] += part[q][i];
        if (ch == nch - 1) {
            const int64_t c0 = (gw + ti * GW) * ROWS + lane;
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const int64_t c = c0 + 32 * i;
                if (c < N) {
#pragma unroll
                    for (int q = 0; q < QB; ++q)
                        if (q < Q) out[(int64_t)q * ldo + c] = rooted ? rootp<P>(acc[q][i]) : acc[q][i];
                }
            }
#pragma unroll
            for (int q = 0; q < QB; ++q)
#pragma unroll
                for (int i = 0; i < R; ++i) acc[q][i] = 0.f;
        }
        __syncwarp();  // every lane is done with box s before lane 0 refills it
    }
}

// ---------------------------------------------------------------------------------------
// COPY = 3 (5 <= Q <= 8): split queries, shared boxes.  At Q = 8 the pass does 8 pair-elements
// per database element, so the per-element issue cost, not HBM, decides: the R = 4, one-warp-
// per-scheduler variant above reached 0.24 of HBM.  Here a CTA has G row groups x H query
// groups of warps; the G rings of D boxes (32R rows x 16 floats, 64-byte TMA swizzle) are each
// consumed by the H warps of the row group (QW = 4 queries each), so a box read from HBM once
// serves all Q queries, each lane holds R = 8 rows (an envelope read from shared memory serves
// 8 rows), and two warps per scheduler hide the shared-memory latency.  Ring protocol per row
// group: full[s] completes on the TMA bytes, empty[s] on the H consumer warps' arrivals; lane 0
// of the group's first warp refills a stage once both consumers released it.  Accumulation in
// packed pairs (even / odd elements of a row: one FFMA2 per two pair-elements), so per
// pair-element one FADD2 (two subtractions), one FMNMX3 and half an FFMA2: 2.5 issue slots.
// Two-level summation (as the other bound kernels): the 16 terms of a box per (query, row) in
// two packed partial sums, folded into the row total after every box.
constexpr int kSqCols = 16;  // box columns (64-byte rows)

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

template <int P>
__device__ __forceinline__ float2 lb4x2(float2 acc, const float4 &x, const float4 &u, const float4 &l) {
    const float2 a0 = __fadd2_rn(make_float2(x.x, x.y), make_float2(-u.x, -u.y));
    const float2 b0 = __fadd2_rn(make_float2(l.x, l.y), make_float2(-x.x, -x.y));
    const float2 a1 = __fadd2_rn(make_float2(x.z, x.w), make_float2(-u.z, -u.w));
    const float2 b1 = __fadd2_rn(make_float2(l.z, l.w), make_float2(-x.z, -x.w));
    const float2 d0 = make_float2(max3f(a0.x, b0.x, 0.f), max3f(a0.y, b0.y, 0.f));
    const float2 d1 = make_float2(max3f(a1.x, b1.x, 0.f), max3f(a1.y, b1.y, 0.f));
    if constexpr (P == 1) {
        acc = __fadd2_rn(acc, d0);
        return __fadd2_rn(acc, d1);
    } else {
        acc = __ffma2_rn(d0, d0, acc);
        return __ffma2_rn(d1, d1, acc);
    }
}

template <int P, int H, int G, int R>
__global__ void __launch_bounds__(G * H * 32, 1)
keogh_stream_sq_kernel(const __grid_constant__ CUtensorMap tmap, const float *__restrict__ U,
                       const float *__restrict__ L, int64_t N, int n, int Q, int D, bool rooted,
                       float *__restrict__ out, int64_t ldo) {
    constexpr int QW = 4;  // queries per warp
    constexpr int QB = QW * H;
    constexpr int ROWS = 32 * R;
    constexpr int BOX = ROWS * kSqCols;  // floats
    extern __shared__ __align__(128) unsigned char smraw[];
    const int npad = (n + kSqCols - 1) / kSqCols * kSqCols;
    const int nch = npad / kSqCols;
    // (offset arithmetic on the shared array itself, not a uintptr_t round trip: the compiler
    // then keeps the shared address space and emits LDS, not generic loads)
    float *boxes = reinterpret_cast<float *>(smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u));
    float *sU = boxes + (size_t)G * D * BOX;  // [QB][npad]
    float *sL = sU + (size_t)QB * npad;
    uint64_t *full = reinterpret_cast<uint64_t *>(sL + (size_t)QB * npad);  // [G][D]
    uint64_t *empty = full + G * D;                                        // [G][D]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = warp / H, h = warp - g * H;  // row group, query group
    for (int t = tid; t < QB * npad; t += G * H * 32) {
        const int q = t / npad, i = t - q * npad;
        const bool ok = q < Q && i < n;
        sU[t] = ok ? U[(int64_t)q * n + i] : kInf;
        sL[t] = ok ? L[(int64_t)q * n + i] : -kInf;
    }
    if (tid == 0) {
        for (int s = 0; s < G * D; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, H);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    const int64_t ntiles = (N + ROWS - 1) / ROWS;
    const int64_t gw = (int64_t)blockIdx.x * G + g, GW = (int64_t)gridDim.x * G;
    const int64_t my_tiles = gw < ntiles ? (ntiles - 1 - gw) / GW + 1 : 0;
    const int64_t steps = my_tiles * nch;
    float *mybox = boxes + (size_t)g * D * BOX;
    uint64_t *myfull = full + g * D, *myempty = empty + g * D;
    const bool producer = h == 0 && lane == 0;
    auto issue = [&](int64_t st) {
        const int64_t ti = st / nch;
        const int ch = (int)(st - ti * nch);
        const int64_t tile = gw + ti * GW;
        const int s = (int)(st % D);
        if (st >= D) mbar_wait(myempty + s, (unsigned)(((st / D) - 1) & 1));  // both consumers done
        fence_proxy_async();
        mbar_expect_tx(myfull + s, (unsigned)(BOX * sizeof(float)));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
            "[%4];\n" ::"r"(smem_u32(mybox + (size_t)s * BOX)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(ch * kSqCols), "r"((int)(tile * ROWS)),
            "r"(smem_u32(myfull + s))
            : "memory");
    };
    if (producer) {
        const int pro = (int)(steps < D - 1 ? steps : D - 1);
        for (int st = 0; st < pro; ++st) issue(st);
    }
    const int swz = (lane >> 1) & 3;  // 64-byte swizzle: chunk c of row r sits at c ^ ((r >> 1) & 3)
    const unsigned ub_a = smem_u32(sU + (size_t)h * QW * npad), lb_a = smem_u32(sL + (size_t)h * QW * npad);
    const unsigned box_a = smem_u32(mybox);
    float2 acc[QW][R];
    float tot[QW][R];
#pragma unroll
    for (int q = 0; q < QW; ++q)
#pragma unroll
        for (int i = 0; i < R; ++i) {
            acc[q][i] = make_float2(0.f, 0.f);
            tot[q][i] = 0.f;
        }
    for (int64_t st = 0; st < steps; ++st) {
        if (producer && st + D - 1 < steps) issue(st + D - 1);
        const int64_t ti = st / nch;
        const int ch = (int)(st - ti * nch);
        const int s = (int)(st % D);
        mbar_wait(myfull + s, (unsigned)((st / D) & 1));
        const unsigned xr = box_a + (unsigned)(s * BOX + lane * kSqCols) * 4u;
        const unsigned ua = ub_a + (unsigned)(ch * kSqCols) * 4u, la = lb_a + (unsigned)(ch * kSqCols) * 4u;
#pragma unroll
        for (int k = 0; k < kSqCols / 4; ++k) {
            float4 xv[R];
#pragma unroll
            for (int i = 0; i < R; ++i) xv[i] = lds128(xr + (unsigned)(i * 32 * kSqCols + 4 * (k ^ swz)) * 4u);
#pragma unroll
            for (int q = 0; q < QW; ++q) {
                const float4 u = lds128(ua + (unsigned)(q * npad + 4 * k) * 4u);
                const float4 l = lds128(la + (unsigned)(q * npad + 4 * k) * 4u);
#pragma unroll
                for (int i = 0; i < R; ++i) acc[q][i] = lb4x2<P>(acc[q][i], xv[i], u, l);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(myempty + s);  // this warp is done with box s
        // two-level summation: the box's 8 + 8 terms per (query, row) fold into the row total
#pragma unroll
        for (int q = 0; q < QW; ++q)
#pragma unroll
            for (int i = 0; i < R; ++i) {
                tot[q][i] += acc[q][i].x + acc[q][i].y;
                acc[q][i] = make_float2(0.f, 0.f);
            }
        if (ch == nch - 1) {
            const int64_t c0 = (gw + ti * GW) * ROWS + lane;
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const int64_t c = c0 + 32 * i;
                if (c < N) {
#pragma unroll
                    for (int q = 0; q < QW; ++q) {
                        const int qq = h * QW + q;
                        const float v = tot[q][i];
                        if (qq < Q) out[(int64_t)qq * ldo + c] = rooted ? rootp<P>(v) : v;
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < QW; ++q)
#pragma unroll
                for (int i = 0; i < R; ++i) tot[q][i] = 0.f;
        }
    }
}

using EncodeTiledFn = PFN_cuTensorMapEncodeTiled_v12000;
EncodeTiledFn get_encode_tiled() {
    static EncodeTiledFn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            p = nullptr;
        }
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

template <int P, int QB, int R, int W>
int launch_stream_tma_t(const float *U, const float *L, const float *db, int64_t Q, int64_t N, int n, bool rooted,
                        float *out, int64_t ldo, cudaStream_t st) {
    EncodeTiledFn enc = get_encode_tiled();
    if (!enc) {
        set_error(DTWLB_ECUDA, "stream LB_Keogh pass: cuTensorMapEncodeTiled unavailable");
        return DTWLB_ECUDA;
    }
    constexpr int ROWS = 32 * R;
    CUtensorMap tmap;
    const cuuint64_t gdim[2] = {(cuuint64_t)n, (cuuint64_t)N};
    const cuuint64_t gstride[1] = {(cuuint64_t)n * sizeof(float)};
    const cuuint32_t box[2] = {kBoxCols, ROWS};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(db), gdim, gstride, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error(DTWLB_ECUDA, "stream LB_Keogh pass: cuTensorMapEncodeTiled failed (%d)", (int)r);
        return DTWLB_ECUDA;
    }
    const int npad = (n + kBoxCols - 1) / kBoxCols * kBoxCols;
    const size_t env = (size_t)2 * QB * npad * sizeof(float);
    int dev = 0, smem_max = 0, nsm = 148;
    DTWLB_CUDA(cudaGetDevice(&dev));
    DTWLB_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    DTWLB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const size_t per_stage = (size_t)W * (ROWS * kBoxCols * sizeof(float) + sizeof(uint64_t));
    static const int env_d = [] { const char *e = getenv("DTWLB_STREAM_STAGES"); return e ? atoi(e) : 0; }();
    // ~192 KB of boxes per SM: D - 1 boxes per warp in flight while it computes on one
    int D = env_d > 1 ? std::min(env_d, 12) : (int)std::max<size_t>(2, (192 * 1024) / per_stage);
    while (D > 2 && env + D * per_stage + 1024 > (size_t)smem_max) --D;
    const size_t smem = env + D * per_stage + 1024;
    if (smem > (size_t)smem_max) {
        set_error(DTWLB_EUNSUPPORTED, "stream LB_Keogh pass: n = %d too long for shared memory", n);
        return DTWLB_EUNSUPPORTED;
    }
    auto k = keogh_stream_tma_kernel<P, QB, R, W>;
    DTWLB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t ntiles = ceil_div(N, ROWS);
    const int grid = (int)std::min<int64_t>(ceil_div(ntiles, W), nsm);  // persistent
    k<<<grid, W * 32, smem, st>>>(tmap, U, L, N, n, (int)Q, D, rooted, out, ldo);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

template <int P, int H, int G, int R>
int launch_stream_sq_t(const float *U, const float *L, const float *db, int64_t Q, int64_t N, int n, bool rooted,
                       float *out, int64_t ldo, cudaStream_t st) {
    EncodeTiledFn enc = get_encode_tiled();
    if (!enc) {
        set_error(DTWLB_ECUDA, "stream LB_Keogh pass: cuTensorMapEncodeTiled unavailable");
        return DTWLB_ECUDA;
    }
    constexpr int ROWS = 32 * R;
    CUtensorMap tmap;
    const cuuint64_t gdim[2] = {(cuuint64_t)n, (cuuint64_t)N};
    const cuuint64_t gstride[1] = {(cuuint64_t)n * sizeof(float)};
    const cuuint32_t box[2] = {kSqCols, ROWS};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(db), gdim, gstride, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error(DTWLB_ECUDA, "stream LB_Keogh pass: cuTensorMapEncodeTiled failed (%d)", (int)r);
        return DTWLB_ECUDA;
    }
    const int npad = (n + kSqCols - 1) / kSqCols * kSqCols;
    const size_t env = (size_t)2 * 4 * H * npad * sizeof(float);
    int dev = 0, smem_max = 0, nsm = 148;
    DTWLB_CUDA(cudaGetDevice(&dev));
    DTWLB_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    DTWLB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const size_t per_stage = (size_t)G * (ROWS * kSqCols * sizeof(float) + 2 * sizeof(uint64_t));
    static const int env_d = [] { const char *e = getenv("DTWLB_STREAM_STAGES"); return e ? atoi(e) : 0; }();
    int D = env_d > 1 ? std::min(env_d, 8) : 8;
    while (D > 2 && env + D * per_stage + 1024 > (size_t)smem_max) --D;
    const size_t smem = env + D * per_stage + 1024;
    if (smem > (size_t)smem_max) {
        set_error(DTWLB_EUNSUPPORTED, "stream LB_Keogh pass: n = %d too long for shared memory", n);
        return DTWLB_EUNSUPPORTED;
    }
    auto k = keogh_stream_sq_kernel<P, H, G, R>;
    DTWLB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t ntiles = ceil_div(N, ROWS);
    const int grid = (int)std::min<int64_t>(ceil_div(ntiles, G), nsm);  // persistent
    k<<<grid, G * H * 32, smem, st>>>(tmap, U, L, N, n, (int)Q, D, rooted, out, ldo);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

template <int P>
int launch_stream_tma_p(const float *U, const float *L, const float *db, int64_t Q, int64_t N, int n, bool rooted,
                        float *out, int64_t ldo, cudaStream_t st) {
    // rows per lane R grows with Q: each envelope read serves R rows (see the kernel)
    if (Q <= 1) return launch_stream_tma_t<P, 1, 1, 8>(U, L, db, Q, N, n, rooted, out, ldo, st);
    if (Q <= 2) return launch_stream_tma_t<P, 2, 2, 8>(U, L, db, Q, N, n, rooted, out, ldo, st);
    // split-query shared-box kernel (DTWLB_STREAM_SQ=0 keeps the per-warp-ring kernel): 5..8
    // queries as two query groups, 3..4 queries as one (eight row groups of 4 rows per lane:
    // C5s4 0.243 vs 0.256 ms for the per-warp-ring kernel)
    static const int env_sq = [] { const char *e = getenv("DTWLB_STREAM_SQ"); return e ? atoi(e) : 1; }();
    if (Q <= 4) {
        if (env_sq && Q >= 3) return launch_stream_sq_t<P, 1, 8, 4>(U, L, db, Q, N, n, rooted, out, ldo, st);
        return launch_stream_tma_t<P, 4, 4, 4>(U, L, db, Q, N, n, rooted, out, ldo, st);
    }
    if (env_sq == 3) return launch_stream_sq_t<P, 2, 6, 8>(U, L, db, Q, N, n, rooted, out, ldo, st);
    if (env_sq) return launch_stream_sq_t<P, 2, 4, 8>(U, L, db, Q, N, n, rooted, out, ldo, st);
    return launch_stream_tma_t<P, 8, 4, 4>(U, L, db, Q, N, n, rooted, out, ldo, st);
}

template <int P, int QB, int COPY>
int launch_stream_t(const float *U, const float *L, const float *db, int64_t Q, int64_t N, int n, bool rooted,
                    float *out, int64_t ldo, cudaStream_t st) {
    const int npad = (n + kKch - 1) / kKch * kKch;
    const size_t env = (size_t)2 * QB * npad * sizeof(float);
    int dev = 0, smem_max = 0, nsm = 148;
    DTWLB_CUDA(cudaGetDevice(&dev));
    DTWLB_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    DTWLB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const size_t per_stage = (size_t)kStreamNT * (kSlot * sizeof(float) + sizeof(uint64_t));
    static const int env_d = [] { const char *e = getenv("DTWLB_STREAM_STAGES"); return e ? atoi(e) : 0; }();
    int D = env_d > 1 ? std::min(env_d, 6) : 5;
    while (D > 2 && env + D * per_stage > (size_t)smem_max) --D;
    const size_t smem = env + D * per_stage;
    if (smem > (size_t)smem_max) {
        set_error(DTWLB_EUNSUPPORTED, "stream LB_Keogh pass: n = %d too long for shared memory", n);
        return DTWLB_EUNSUPPORTED;
    }
    auto k = keogh_stream_kernel<P, QB, COPY>;
    DTWLB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t ntiles = ceil_div(N, kStreamNT);
    const int grid = (int)std::min<int64_t>(ntiles, nsm);  // persistent: one CTA per SM
    k<<<grid, kStreamNT, smem, st>>>(U, L, db, N, n, (int)Q, D, rooted, out, ldo);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

template <int P, int COPY>
int launch_stream_p(const float *U, const float *L, const float *db, int64_t Q, int64_t N, int n, bool rooted,
                    float *out, int64_t ldo, cudaStream_t st) {
    if (Q <= 1) return launch_stream_t<P, 1, COPY>(U, L, db, Q, N, n, rooted, out, ldo, st);
    if (Q <= 2) return launch_stream_t<P, 2, COPY>(U, L, db, Q, N, n, rooted, out, ldo, st);
    if (Q <= 4) return launch_stream_t<P, 4, COPY>(U, L, db, Q, N, n, rooted, out, ldo, st);
    return launch_stream_t<P, 8, COPY>(U, L, db, Q, N, n, rooted, out, ldo, st);
}

}  // namespace

bool keogh_stream_ok(int64_t Q, int n, const void *db) {
    return Q >= 1 && Q <= kStreamMaxQ && n % 4 == 0 && (reinterpret_cast<uintptr_t>(db) % 16) == 0;
}

int launch_keogh_stream(const float *U, const float *L, const float *db, int64_t Q, int64_t N, int n, int p,
                        bool rooted, float *out, int64_t ldo, cudaStream_t st) {
    if (Q == 0 || N == 0) return DTWLB_OK;
    if (!keogh_stream_ok(Q, n, db)) {
        set_error(DTWLB_EINVAL, "internal: stream LB_Keogh pass needs 1 <= Q <= %d, n %% 4 == 0, aligned rows",
                  kStreamMaxQ);
        return DTWLB_EINVAL;
    }
    // copy engine: 2 = 2D TMA boxes (default; n >= 32), 0 = per-row TMA bulk copies, 1 = cp.async
    static const int env_copy = [] { const char *e = getenv("DTWLB_STREAM_COPY"); return e ? atoi(e) : 2; }();
    if (env_copy == 2 && n >= kBoxCols)
        return p == 1 ? launch_stream_tma_p<1>(U, L, db, Q, N, n, rooted, out, ldo, st)
                      : launch_stream_tma_p<2>(U, L, db, Q, N, n, rooted, out, ldo, st);
    if (env_copy != 0)
        return p == 1 ? launch_stream_p<1, 1>(U, L, db, Q, N, n, rooted, out, ldo, st)
                      : launch_stream_p<2, 1>(U, L, db, Q, N, n, rooted, out, ldo, st);
    return p == 1 ? launch_stream_p<1, 0>(U, L, db, Q, N, n, rooted, out, ldo, st)
                  : launch_stream_p<2, 0>(U, L, db, Q, N, n, rooted, out, ldo, st);
}

}  // namespace dtwlb
