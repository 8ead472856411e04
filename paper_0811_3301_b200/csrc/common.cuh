// common.cuh -- shared plumbing of libdtwlb (error model, small device helpers).
// Product code only: nothing here is shared with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/dtwlb.h"

namespace dtwlb {

// ---- error model: thread-local message, status codes never exceptions ----
void set_error(int code, const char *fmt, ...);
int cuda_fail(cudaError_t e, const char *what, const char *file, int line);

#define DTWLB_CUDA(call)                                                           \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess) return ::dtwlb::cuda_fail(e_, #call, __FILE__, __LINE__); \
    } while (0)

// every kernel launch site is followed by DTWLB_LAUNCH_CHECK(), which also counts
// the launch (nn_stats.kernel_launches reports the count of one nn_search call)
extern unsigned long long g_launches;
#define DTWLB_LAUNCH_CHECK()                                   \
    do {                                                       \
        __atomic_fetch_add(&::dtwlb::g_launches, 1ull, __ATOMIC_RELAXED); \
        DTWLB_CUDA(cudaGetLastError());                        \
    } while (0)

#define DTWLB_TRY(expr)            \
    do {                           \
        int s_ = (expr);           \
        if (s_ != DTWLB_OK) return s_; \
    } while (0)

// Device-side bounds checks of the debug build (build.py --checked): printf + trap.
#ifdef DTWLB_CHECKED
#define DCHECK(cond, ...)                                                  \
    do {                                                                   \
        if (!(cond)) {                                                     \
            printf("DCHECK %s:%d (%s): ", __FILE__, __LINE__, #cond);       \
            printf(__VA_ARGS__);                                           \
            printf("\n");                                                  \
            __trap();                                                      \
        }                                                                  \
    } while (0)
#else
#define DCHECK(cond, ...) \
    do {                  \
    } while (0)
#endif

// One-time device check: an sm_100 device must be current.
int require_device();

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr float kInf = __builtin_huge_valf();

// ---- device helpers ----
__device__ __forceinline__ float min3f(float a, float b, float c) { return fminf(fminf(a, b), c); }
__device__ __forceinline__ float max3f(float a, float b, float c) { return fmaxf(fmaxf(a, b), c); }

// |t|^P for P in {1,2}: the cost term |x_i - y_j|^p of P:207 and the bound terms.
template <int P>
__device__ __forceinline__ float powp(float t) {
    if constexpr (P == 1) return fabsf(t);
    else return t * t;
}
// acc + d^P with d >= 0 (one FADD or one FFMA).
template <int P>
__device__ __forceinline__ float accp(float acc, float d) {
    if constexpr (P == 1) return acc + d;
    else return fmaf(d, d, acc);
}
template <int P>
__device__ __forceinline__ float rootp(float v) {
    if constexpr (P == 2) return sqrtf(v);
    else if constexpr (P == 4) return sqrtf(sqrtf(v));  // (dtw_band's DTW_4, Appendix C)
    else return v;  // p = 1, and p = 0 (DTW_inf, a max: no root)
}

// (dist, idx) ordering key: non-negative float bits are monotone (reading c17: -0 -> +0).
__device__ __forceinline__ unsigned long long pack_key(float d, uint32_t idx) {
    d = fmaxf(d, 0.0f);
    return (static_cast<unsigned long long>(__float_as_uint(d)) << 32) | idx;
}

// Candidate-list keys (survivor kernel -> sort -> DTW walk) carry, in the low kKeyPosBits bits
// of their bound word, the key's append position within its sort run (runs are kRun =
// 2^kKeyPosBits keys), so the walk can find the pair's abandon schedule after the sort.  The
// bound is the word with those bits cleared: a truncation of a non-negative float, so never
// above the exact bound (reading c22).
constexpr int kKeyPosBits = 12;
constexpr uint32_t kKeyPosMask = (1u << kKeyPosBits) - 1u;
__device__ __forceinline__ unsigned long long pack_list_key(float d, uint32_t idx, int pos) {
    d = fmaxf(d, 0.0f);
    const uint32_t hi = (__float_as_uint(d) & ~kKeyPosMask) | ((uint32_t)pos & kKeyPosMask);
    return (static_cast<unsigned long long>(hi) << 32) | idx;
}
__device__ __forceinline__ float key_bound(unsigned long long key) {
    return __uint_as_float((uint32_t)(key >> 32) & ~kKeyPosMask);
}
__device__ __forceinline__ int key_pos(unsigned long long key) { return (int)((uint32_t)(key >> 32) & kKeyPosMask); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Start of query q's key list: exact-count lists (per-query offsets) or fixed capacity.
__device__ __forceinline__ int64_t list_base(const int64_t *loff, int64_t cap, int64_t q) {
    return loff ? __ldg(loff + q) : q * cap;
}

// ---- cp.async (global -> shared, no register staging); src_bytes < size zero-fills ----
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

}  // namespace dtwlb
