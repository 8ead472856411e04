// envelope.cu -- batched warping envelope, the a1 step of the cascade.
//
//   U_i = max{x_k : |k-i| <= w},  L_i = min{x_k : |k-i| <= w}   (window clipped)
//
// Design (B200): HBM-bound streaming kernel.  Each CTA stages a few rows in
// shared memory with edge replication (x_{-t} := x_0, x_{n-1+t} := x_{n-1}:
// replicated edge values always lie inside the clipped window, so max/min are
// unchanged and the result is exact).  Each thread produces four consecutive
// outputs from one scan of their common window [i+3-w, i+w] plus three extra
// values on each side: 2w+4 shared-memory reads per 4 outputs instead of
// 4(2w+1).  min/max never round, so the output is bit-identical to the
// definition.  Rows too long for shared memory use the global-memory variant.
#include "kernels.cuh"

namespace dtwlb {

__device__ __forceinline__ void env_quad(const float *P, int i0, int w, float *mx, float *mn) {
    // P is the padded row: P[t] = x[clamp(t - pad, 0, n-1)], pad = w.
    // Output k of the quad (i = i0 + k) covers padded [i0 + k, i0 + k + 2w].
    if (w <= 1) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float a = P[i0 + k], b = P[i0 + k + w], c = P[i0 + k + 2 * w];
            mx[k] = max3f(a, b, c);
            mn[k] = min3f(a, b, c);
        }
        return;
    }
    // common window of the 4 outputs: padded [i0+3, i0+2w]
    float cmx = P[i0 + 3], cmn = cmx;
    int t = i0 + 4;
    const int te = i0 + 2 * w;
    for (; t + 1 <= te; t += 2) {
        float a = P[t], b = P[t + 1];
        cmx = max3f(cmx, a, b);
        cmn = min3f(cmn, a, b);
    }
    if (t <= te) {
        float a = P[t];
        cmx = fmaxf(cmx, a);
        cmn = fminf(cmn, a);
    }
    float a = P[i0], b = P[i0 + 1], c = P[i0 + 2];
    float d = P[i0 + 2 * w + 1], e = P[i0 + 2 * w + 2], f = P[i0 + 2 * w + 3];
    mx[0] = fmaxf(cmx, max3f(a, b, c));
    mn[0] = fminf(cmn, min3f(a, b, c));
    mx[1] = fmaxf(cmx, max3f(b, c, d));
    mn[1] = fminf(cmn, min3f(b, c, d));
    mx[2] = fmaxf(cmx, max3f(c, d, e));
    mn[2] = fminf(cmn, min3f(c, d, e));
    mx[3] = fmaxf(cmx, max3f(d, e, f));
    mn[3] = fminf(cmn, min3f(d, e, f));
}

// env_quad with 128-bit shared-memory reads: P 16-byte aligned and i0 % 4 == 0, so the four
// outputs' common window [i0+3, i0+2w] is read as aligned float4 vectors (a quarter-warp reads
// 8 consecutive vectors: conflict-free) -- the scalar version's stride-4 reads were 4-way bank
// conflicted.  Same comparisons, same (exact) result.
__device__ __forceinline__ void env_quad4(const float *P, int i0, int w, float *mx, float *mn) {
    const float4 h = *reinterpret_cast<const float4 *>(P + i0);  // P[i0 .. i0+3]
    float cmx = h.w, cmn = h.w;                                  // P[i0+3]
    const int te = i0 + 2 * w;                                   // last index of the common window
    int t = i0 + 4;
    for (; t + 3 <= te; t += 4) {
        const float4 v = *reinterpret_cast<const float4 *>(P + t);
        cmx = max3f(cmx, v.x, v.y);
        cmx = max3f(cmx, v.z, v.w);
        cmn = min3f(cmn, v.x, v.y);
        cmn = min3f(cmn, v.z, v.w);
    }
    for (; t <= te; ++t) {
        const float v = P[t];
        cmx = fmaxf(cmx, v);
        cmn = fminf(cmn, v);
    }
    const float a = h.x, b = h.y, c = h.z;
    const float d = P[te + 1], e = P[te + 2], f = P[te + 3];
    mx[0] = fmaxf(cmx, max3f(a, b, c));
    mn[0] = fminf(cmn, min3f(a, b, c));
    mx[1] = fmaxf(cmx, max3f(b, c, d));
    mn[1] = fminf(cmn, min3f(b, c, d));
    mx[2] = fmaxf(cmx, max3f(c, d, e));
    mn[2] = fminf(cmn, min3f(c, d, e));
    mx[3] = fmaxf(cmx, max3f(d, e, f));
    mn[3] = fminf(cmn, min3f(d, e, f));
}

// rows_per_cta rows per CTA; padded row length plen >= n + 2w + 4 (a multiple of 4).
__global__ void envelope_smem_kernel(const float *__restrict__ x, int n, int w, float *__restrict__ U,
                                     float *__restrict__ L, int64_t count, int rows_per_cta, int plen,
                                     bool vec_out) {
    extern __shared__ float sm[];
    const int nq = (n + 3) >> 2;  // quads per row
    for (int64_t r0 = (int64_t)blockIdx.x * rows_per_cta; r0 < count;
         r0 += (int64_t)gridDim.x * rows_per_cta) {
        const int rows = (int)((count - r0) < rows_per_cta ? (count - r0) : rows_per_cta);
        // stage: padded rows, edge-replicated
        for (int t = threadIdx.x; t < rows * plen; t += blockDim.x) {
            int r = t / plen, j = t - r * plen - w;
            j = j < 0 ? 0 : (j > n - 1 ? n - 1 : j);
            sm[t] = __ldg(x + (r0 + r) * (int64_t)n + j);
        }
        __syncthreads();
        for (int t = threadIdx.x; t < rows * nq; t += blockDim.x) {
            int r = t / nq, i0 = (t - r * nq) * 4;
            float mx[4], mn[4];
            float *u = U + (r0 + r) * (int64_t)n, *l = L + (r0 + r) * (int64_t)n;
            if (w >= 2 && (plen & 3) == 0) env_quad4(sm + r * plen, i0, w, mx, mn);
            else env_quad(sm + r * plen, i0, w, mx, mn);
            if ((n & 3) == 0 && vec_out) {  // 16-byte stores: a warp writes 512 contiguous bytes
                *reinterpret_cast<float4 *>(u + i0) = make_float4(mx[0], mx[1], mx[2], mx[3]);
                *reinterpret_cast<float4 *>(l + i0) = make_float4(mn[0], mn[1], mn[2], mn[3]);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (i0 + k < n) { u[i0 + k] = mx[k]; l[i0 + k] = mn[k]; }
            }
        }
        __syncthreads();
    }
}

// Fallback for rows that do not fit in shared memory: direct window scan from global.
__global__ void envelope_global_kernel(const float *__restrict__ x, int n, int w, float *__restrict__ U,
                                       float *__restrict__ L, int64_t count) {
    const int64_t total = count * (int64_t)n;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = t / n;
        int i = (int)(t - r * n);
        int lo = max(0, i - w), hi = min(n - 1, i + w);
        const float *row = x + r * n;
        float mx = row[lo], mn = mx;
        for (int k = lo + 1; k <= hi; ++k) { float v = __ldg(row + k); mx = fmaxf(mx, v); mn = fminf(mn, v); }
        U[t] = mx;
        L[t] = mn;
    }
}

int launch_envelope(const float *x, int n, int w, float *U, float *L, int64_t count, cudaStream_t st) {
    if (count == 0) return DTWLB_OK;
    w = w > n - 1 ? n - 1 : w;
    const int plen = (n + 2 * w + 4 + 3) & ~3;  // (a multiple of 4: 16-byte aligned rows)
    const size_t row_bytes = (size_t)plen * sizeof(float);
    const size_t max_smem = 160 * 1024;
    if (row_bytes <= max_smem) {
        // ~32 KB of staged rows per CTA (several CTAs per SM); one long row may use more
        const int rows = (int)std::max<size_t>(1, std::min<size_t>(64, (32 * 1024) / row_bytes));
        size_t smem = rows * row_bytes;
        if (smem > 48 * 1024)
            DTWLB_CUDA(cudaFuncSetAttribute(envelope_smem_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int64_t ctas = ceil_div(count, rows);
        int grid = (int)std::min<int64_t>(ctas, 148 * 64);
        const bool vec_out = ((reinterpret_cast<uintptr_t>(U) | reinterpret_cast<uintptr_t>(L)) & 15) == 0;
        envelope_smem_kernel<<<grid, 256, smem, st>>>(x, n, w, U, L, count, rows, plen, vec_out);
    } else {
        int64_t total = count * (int64_t)n;
        int grid = (int)std::min<int64_t>(ceil_div(total, 256), 148 * 32);
        envelope_global_kernel<<<grid, 256, 0, st>>>(x, n, w, U, L, count);
    }
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

}  // namespace dtwlb
