// search.cu -- nn_search: exact k-NN under banded DTW_p by the paper's cascade
// (Alg. 3), generalised to p in {1,2}, k >= 1 and many queries.
//
// Host runtime (per block of Qb queries, all device-side data):
//   a1  envelopes U,L of the queries (+ LU = U(L), UL = L(U) for LB_Improved) and
//       U(x), L(x) of the database (once per call)                  [envelope.cu]
//   a2  beta1 = LB_Keogh^p for every (query, candidate) pair          [keogh.cu]
//   a3  best-first ordering:  a sampled quantile t_S of each query's beta1 row
//       splits its candidates into a small first range (beta1 <= t_S, ~S pairs)
//       and the rest.  Range 1 is bounded, sorted by LB_Improved and walked in
//       ascending order with growing DTW batches; this drives tau (the k-th best)
//       down to ~its final value.  Range 2 (t_S < beta1 <= tau(1+eps)) is then
//       filtered by LB_Improved against that tau, sorted, and walked the same way.
//       Correctness never depends on the order: every candidate with
//       beta1 <= tau_final(1+eps) is in range 1 or range 2.
//   a4  LB_Improved on each range's survivors -> per-query key lists (beta_lb, c)
//                                                                     [improved.cu]
//   a5  DTW walk: rounds of (plan -> DTW batch with early abandon -> top-k merge);
//       a query stops when its next sorted bound exceeds tau(1+eps)     [dtw.cu]
//   a6  finalize: k smallest by (DTW^p, index), rooted.
// Pruning rule (reading c3/c13): a bound prunes only if bound > tau^p (1 + eps).
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <tuple>
#include <vector>

#include <cub/block/block_radix_sort.cuh>

#include "kernels.cuh"

namespace dtwlb {

int launch_dtw_generic(const DtwArgs &a, const float *yraw, float *scratch, int p, bool walk,
                       cudaStream_t st);

// ------------------------------------------------------------------ workspace
namespace {

// One workspace per CUDA device ordinal: a process may call the library on several devices
// (each call uses the workspace of the device current on the calling thread).
struct Workspace {
    int device = -1;  // owner ordinal (set on first allocation)
    std::vector<void *> ptr;
    std::vector<size_t> size;
    ~Workspace() { release(); }
    cudaStream_t copy_stream = nullptr;  // host->device database chunks of the e2e path
    cudaStream_t get_copy_stream() {
        if (!copy_stream && cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking) != cudaSuccess) {
            cudaGetLastError();
            copy_stream = nullptr;
        }
        return copy_stream;
    }
    void release() {
        qb_cache.clear();
        if (copy_stream) { cudaStreamDestroy(copy_stream); copy_stream = nullptr; }
        if (ptr.empty()) return;
        int cur = -1;
        cudaGetDevice(&cur);
        if (device >= 0 && device != cur) cudaSetDevice(device);
        for (void *p : ptr)
            if (p) cudaFree(p);
        if (device >= 0 && device != cur) cudaSetDevice(cur);
        ptr.clear();
        size.clear();
    }
    size_t cur_size(int slot) const { return slot < (int)size.size() ? size[slot] : 0; }
    // query-block size chosen for a problem shape (Q, N, n, mode): cudaMemGetInfo is asked once
    // per shape -- it contends with NVML clients (nvidia-smi) for a driver lock, and a call of
    // it inside the pipeline showed up as 5-50 ms device-idle gaps before the bound pass
    std::vector<std::tuple<int64_t, int64_t, int, int, int64_t>> qb_cache;
    int64_t cached_qb(int64_t Q, int64_t N, int n, int mode) const {
        for (auto &t : qb_cache)
            if (std::get<0>(t) == Q && std::get<1>(t) == N && std::get<2>(t) == n && std::get<3>(t) == mode)
                return std::get<4>(t);
        return 0;
    }
    int get(int slot, size_t bytes, void **out) {
        if ((int)ptr.size() <= slot) { ptr.resize(slot + 1, nullptr); size.resize(slot + 1, 0); }
        bytes = std::max<size_t>(bytes, 256);
        if (size[slot] < bytes) {
            if (ptr[slot]) { cudaDeviceSynchronize(); cudaFree(ptr[slot]); ptr[slot] = nullptr; size[slot] = 0; }
            if (device < 0) cudaGetDevice(&device);
            cudaError_t e = cudaMalloc(&ptr[slot], bytes);
            if (e != cudaSuccess) {
                cudaGetLastError();
                set_error(DTWLB_ENOMEM, "device workspace: cannot allocate %zu bytes (%s)", bytes,
                          cudaGetErrorString(e));
                return DTWLB_ENOMEM;
            }
            size[slot] = bytes;
        }
        *out = ptr[slot];
        return DTWLB_OK;
    }
};

constexpr int kMaxDevices = 64;
Workspace *ws_all() {
    static Workspace w[kMaxDevices];
    return w;
}
Workspace &ws() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) { cudaGetLastError(); d = 0; }
    return ws_all()[d];
}
std::mutex &ws_mutex() {
    static std::mutex m;
    return m;
}

enum Slot {
    S_QSTAGE, S_DBSTAGE, S_ENV, S_QPAD, S_YSH, S_DBENV, S_BETA1, S_LIST, S_RES, S_STATE, S_TOPK,
    S_OUTSTAGE, S_SCRATCH, S_TMP, S_MASK, S_PAA, S_QPAA, S_RPAA, S_SNAP, S_COUNT, S_REC
};

template <typename T>
int wsget(int slot, size_t count, T **out) {
    void *p = nullptr;
    DTWLB_TRY(ws().get(slot, count * sizeof(T), &p));
    *out = static_cast<T *>(p);
    return DTWLB_OK;
}

// ------------------------------------------------------------------ kernels
// Padded copies of the query-side LB_Improved arrays: [Q][npadE], zero padded.
__global__ void pad_rows_kernel(const float *__restrict__ src, int64_t rows, int n, float *__restrict__ dst,
                                int npad, float padv) {
    const int64_t total = rows * (int64_t)npad;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = t / npad;
        int i = (int)(t - r * npad);
        dst[t] = i < n ? src[r * n + i] : padv;
    }
}

// Sampled quantiles of each query's gate-bound row: t_r (r = 0..R-2) such that ~S*G^r
// candidates have gate <= t_r.  They split the candidates into R ranges processed in
// ascending order (selection thresholds only -- correctness does not depend on them).
constexpr int kSample = 2048;
constexpr int kMaxRanges = 8;
__device__ __forceinline__ float gate_at(const float *g, int64_t i) { return g[i]; }
__device__ __forceinline__ float gate_at(const __half *g, int64_t i) { return __half2float(g[i]); }

template <typename T>
__global__ void __launch_bounds__(512) sample_threshold_kernel(const T *__restrict__ beta1, int64_t ldb,
                                                               int64_t N, int64_t S, int R, int G,
                                                               float *__restrict__ tS, int Qb) {
    __shared__ float v[kSample];
    const int64_t q = blockIdx.x;
    const int M = N < kSample ? (int)N : kSample;
    for (int s = threadIdx.x; s < kSample; s += blockDim.x) {
        int64_t c = (int64_t)s * N / M;
        v[s] = s < M ? gate_at(beta1, q * ldb + c) : kInf;
    }
    __syncthreads();
    // bitonic sort of kSample floats
    for (int k = 2; k <= kSample; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int t = threadIdx.x; t < kSample; t += blockDim.x) {
                int u = t ^ j;
                if (u > t) {
                    bool up = (t & k) == 0;
                    float a = v[t], b = v[u];
                    if ((a > b) == up) { v[t] = b; v[u] = a; }
                }
            }
            __syncthreads();
        }
    if (threadIdx.x < R - 1) {
        int64_t Sr = S;
        for (int i = 0; i < (int)threadIdx.x; ++i) Sr *= G;
        float t;
        if (Sr >= N) t = kInf;
        else {
            int64_t r = (Sr * M + N - 1) / N;  // rank in the sample
            r = r < 1 ? 1 : (r > M ? M : r);
            t = v[r - 1];
        }
        tS[(int64_t)threadIdx.x * Qb + q] = t;
    }
}

// Sort runs of kRun keys of each query list by their bound (the walk's best-first order):
// a block-wide LSD radix sort (CUB BlockRadixSort, in this kernel's shared memory) of the
// 32-bit bound bits with the candidate index as payload; 512 threads x 8 keys = one run.
// Non-negative float bits order like the floats; equal bounds keep their list order.
constexpr int kRun = 4096;
static_assert(kRun == 1 << kKeyPosBits, "list keys carry their position within a sort run");
constexpr int kSortThreads = 512, kSortItems = kRun / kSortThreads;
// Runs of the range's lists, built on the device (no host round trip): run t = (query,
// index) with t over sum_q ceil(len_q / kRun); the count goes to *nruns.  One CTA.
__global__ void __launch_bounds__(1024) make_runs_kernel(const int *__restrict__ len, int Qb, int *__restrict__ run_q,
                                                         int *__restrict__ run_idx, int *__restrict__ nruns) {
    __shared__ int warp_sums[32];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int base = 0; base < Qb; base += blockDim.x) {
        const int q = base + threadIdx.x;
        const int m = q < Qb ? (len[q] + kRun - 1) / kRun : 0;
        int v = m;  // inclusive scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        if (lane == 31) warp_sums[wid] = v;
        __syncthreads();
        if (wid == 0) {
            int u = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, u, o);
                if (lane >= o) u += t;
            }
            warp_sums[lane] = u;
        }
        __syncthreads();
        const int off = carry + v - m + (wid ? warp_sums[wid - 1] : 0);
        for (int r = 0; r < m; ++r) { run_q[off + r] = q; run_idx[off + r] = r; }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = off + m;
        __syncthreads();
    }
    if (threadIdx.x == 0) *nruns = carry;
}

// Exact-count key lists: off[q] = sum_{q' < q} cnt[q'] (int64), off[Qb] = the total, off[Qb + 1] =
// the largest count.  One CTA.
__global__ void __launch_bounds__(1024) list_offsets_kernel(const int *__restrict__ cnt, int Qb,
                                                            int64_t *__restrict__ off) {
    __shared__ long long warp_sums[32];
    __shared__ long long carry;
    __shared__ int mx;
    if (threadIdx.x == 0) { carry = 0; mx = 0; }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int base = 0; base < Qb; base += blockDim.x) {
        const int q = base + threadIdx.x;
        const long long m = q < Qb ? cnt[q] : 0;
        if (m) atomicMax(&mx, (int)m);
        long long v = m;  // inclusive scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
        }
        if (lane == 31) warp_sums[wid] = v;
        __syncthreads();
        if (wid == 0) {
            long long u = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long t = __shfl_up_sync(0xffffffffu, u, o);
                if (lane >= o) u += t;
            }
            warp_sums[lane] = u;
        }
        __syncthreads();
        const long long ex = carry + v - m + (wid ? warp_sums[wid - 1] : 0);
        if (q < Qb) off[q] = ex;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = ex + m;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        off[Qb] = carry;
        off[Qb + 1] = mx;
    }
}

__global__ void __launch_bounds__(kSortThreads) sort_runs_kernel(unsigned long long *__restrict__ list, int64_t cap,
                                                                 const int64_t *__restrict__ loff,
                                                                 const int *__restrict__ run_q,
                                                                 const int *__restrict__ run_idx,
                                                                 const int *__restrict__ len,
                                                                 const int *__restrict__ nruns) {
    using BRS = cub::BlockRadixSort<unsigned, kSortThreads, kSortItems, unsigned>;
    __shared__ typename BRS::TempStorage tmp;
    const int nr = *nruns;
    for (int t = blockIdx.x; t < nr; t += gridDim.x) {
    const int q = run_q[t], r = run_idx[t];
    const int64_t base = list_base(loff, cap, q) + (int64_t)r * kRun;
    const int m = min(kRun, len[q] - r * kRun);
    DCHECK(m > 0 && (loff ? base + m <= loff[q + 1] : (int64_t)r * kRun + m <= cap), "sort q=%d r=%d m=%d cap=%lld",
           q, r, m, (long long)cap);
    unsigned key[kSortItems], val[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const int i = threadIdx.x * kSortItems + j;
        const unsigned long long k = i < m ? list[base + i] : ~0ull;
        key[j] = (unsigned)(k >> 32);
        val[j] = (unsigned)(k & 0xffffffffu);
    }
    BRS(tmp).Sort(key, val);
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const int i = threadIdx.x * kSortItems + j;
        if (i < m) list[base + i] = ((unsigned long long)key[j] << 32) | val[j];
    }
    __syncthreads();  // temp storage reuse
    }
}

// Row+column cascade start values (reading c21) of the keys appended in this
// range: the gate slot of pair (q, c) takes -rd(LB_Improved^p - sum_{j < c0} beta2_j), beta2_j
// = d(y_j, [L(H)_j, U(H)_j])^p by the closed form of improved.cu.  One CTA per sorted run;
// a warp takes four keys at a time, lane l & 7 covers the columns 4 (l & 7) .. + 3 (c0 <= 32).
template <int P>
__global__ void __launch_bounds__(256) rest0_kernel(const unsigned long long *__restrict__ list, int64_t cap,
                                                    const int64_t *__restrict__ loff, const int *__restrict__ run_q, const int *__restrict__ run_idx,
                                                    const int *__restrict__ len, const int *__restrict__ nruns,
                                                    const float *__restrict__ yq,
                                                    const float *__restrict__ LUq, const float *__restrict__ ULq,
                                                    const float *__restrict__ Ux, const float *__restrict__ Lx, int n,
                                                    int c0, __half *__restrict__ gate, int64_t ldb) {
    const int nr = *nruns;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, src = lane & 7, grp = lane >> 3;
    for (int t = blockIdx.x; t < nr; t += gridDim.x) {
    const int q = run_q[t], r = run_idx[t];
    const int m = min(kRun, len[q] - r * kRun);
    const bool mine = 4 * src < c0;
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f), lu = y, ul = y;
    if (mine) {
        y = __ldg(reinterpret_cast<const float4 *>(yq + (int64_t)q * n + 4 * src));
        lu = __ldg(reinterpret_cast<const float4 *>(LUq + (int64_t)q * n + 4 * src));
        ul = __ldg(reinterpret_cast<const float4 *>(ULq + (int64_t)q * n + 4 * src));
    }
    const unsigned long long *lq = list + list_base(loff, cap, q) + (int64_t)r * kRun;
    for (int j0 = warp * 4; j0 < m; j0 += (blockDim.x >> 5) * 4) {
        const int j = j0 + grp;
        float s = 0.f, beta = 0.f;
        uint32_t c = 0;
        if (j < m) {
            const unsigned long long key = lq[j];
            c = (uint32_t)(key & 0xffffffffu);
            beta = key_bound(key);
            if (mine) {
                const float4 ux = __ldg(reinterpret_cast<const float4 *>(Ux + (int64_t)c * n + 4 * src));
                const float4 lx = __ldg(reinterpret_cast<const float4 *>(Lx + (int64_t)c * n + 4 * src));
                s = accp<P>(s, max3f(y.x - fmaxf(ux.x, lu.x), fminf(lx.x, ul.x) - y.x, 0.f));
                s = accp<P>(s, max3f(y.y - fmaxf(ux.y, lu.y), fminf(lx.y, ul.y) - y.y, 0.f));
                s = accp<P>(s, max3f(y.z - fmaxf(ux.z, lu.z), fminf(lx.z, ul.z) - y.z, 0.f));
                s = accp<P>(s, max3f(y.w - fmaxf(ux.w, lu.w), fminf(lx.w, ul.w) - y.w, 0.f));
            }
        }
        s += __shfl_xor_sync(0xffffffffu, s, 4);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        if (j < m && src == 0) gate[(int64_t)q * ldb + c] = __hneg(__float2half_rd(fmaxf(__fsub_rd(beta, s), 0.f)));
    }
    }
}

struct QState {
    float *thr;      // tau^p (1+eps) (+inf until k results)
    float *lo, *hi;  // current range of beta1
    float *tS;
    int *len, *pos, *rnd, *active;
    int *item_off;   // [Qb+1] first result slot of each query this round
    int *chunk_off;  // [Qb+1] first warp chunk of each query this round
    int *counters;   // [0] total items of the round, [1] total warp chunks
    unsigned long long *topk;  // [Qb][k] keys (DTW^p bits, index), ascending; ~0 = empty
    int *lock;                 // [Qb] top-k insertion locks (dtw.cu walk_result)
    int *prev_cnt;             // [Qb] items of the query in the previous walk round
    unsigned long long *stat;  // [0] improved evals, [1] dtw items started, [2] cells, [3] abandoned
    int *q_count;              // [Qb] the range's gate survivors per query (select kernel)
    int64_t *loff;             // [Qb + 1] offsets of the range's exact-count key lists
};

__global__ void init_state_kernel(QState s, int Qb, int k) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < Qb; q += gridDim.x * blockDim.x) {
        s.thr[q] = kInf;
        s.lock[q] = 0;
        for (int j = 0; j < k; ++j) s.topk[(int64_t)q * k + j] = ~0ull;
    }
}

__global__ void set_range_kernel(QState s, int Qb, int macro, int R) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < Qb; q += gridDim.x * blockDim.x) {
        s.lo[q] = macro == 0 ? -kInf : s.tS[(int64_t)(macro - 1) * Qb + q];
        s.hi[q] = macro == R - 1 ? kInf : s.tS[(int64_t)macro * Qb + q];
        s.len[q] = 0;
        s.q_count[q] = 0;
    }
}

__global__ void start_walk_kernel(QState s, int Qb) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < Qb; q += gridDim.x * blockDim.x) {
        s.pos[q] = 0;
        s.rnd[q] = 0;
        s.prev_cnt[q] = 0;
        s.active[q] = s.len[q] > 0;
    }
}

// Per-round plan: items of each active query = min(D0 * 2^round, remaining), and
// the warp chunks (kDtwIpw items each, never spanning two queries) that hold them.
// Two exclusive scans: item_off (results layout) and chunk_off (warp -> query).
constexpr int kD0 = 128, kDMax = 65536;
constexpr int kSeedCap = 2048;   // cap of the best-first seed range size S (nn_search)
constexpr int kRoundBatch = 8;  // walk rounds queued per host check (w <= 64 DTW kernels)
__device__ __forceinline__ int2 block_scan2(int2 v, int2 *warp_sums, int2 &total) {
    // inclusive block-wide scan of two ints; returns the inclusive value, sets total
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int tx = __shfl_up_sync(0xffffffffu, v.x, o), ty = __shfl_up_sync(0xffffffffu, v.y, o);
        if (lane >= o) { v.x += tx; v.y += ty; }
    }
    if (lane == 31) warp_sums[wid] = v;
    __syncthreads();
    if (wid == 0) {
        int2 w = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : make_int2(0, 0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int tx = __shfl_up_sync(0xffffffffu, w.x, o), ty = __shfl_up_sync(0xffffffffu, w.y, o);
            if (lane >= o) { w.x += tx; w.y += ty; }
        }
        warp_sums[lane] = w;
    }
    __syncthreads();
    if (wid) { v.x += warp_sums[wid - 1].x; v.y += warp_sums[wid - 1].y; }
    total = warp_sums[(blockDim.x >> 5) - 1];
    __syncthreads();
    return v;
}

// The previous round's items are consumed first (the DTW kernel merged its results
// into the top-k and tau directly): the walk advances past them and skips the rest of
// a sorted run once its next bound exceeds tau (1+eps).
__global__ void __launch_bounds__(1024) plan_kernel(QState s, int Qb, const unsigned long long *__restrict__ list,
                                                    int64_t cap, const int64_t *__restrict__ loff, bool sorted, int d0,
                                                    int gs) {
    __shared__ int2 warp_sums[32];
    int2 carry = make_int2(0, 0);
    for (int base = 0; base < Qb; base += blockDim.x) {
        const int q = base + threadIdx.x;
        int cnt = 0;
        if (q < Qb && s.active[q]) {
            int pos = s.pos[q] + s.prev_cnt[q];
            const int len = s.len[q];
            if (s.prev_cnt[q] > 0 && sorted) {
                s.rnd[q] += 1;
                const float thr = *reinterpret_cast<volatile float *>(s.thr + q);
                const unsigned long long *lq = list + list_base(loff, cap, q);
                while (pos < len && key_bound(lq[pos]) > thr)
                    pos = (pos / kRun + 1) * kRun;
            }
            s.pos[q] = pos;
            if (pos < len) {
                const long long d = min((long long)d0 << min(s.rnd[q] * gs, 11), (long long)kDMax);
                cnt = (int)min(d, (long long)(len - pos));
            } else {
                s.active[q] = 0;
            }
            s.prev_cnt[q] = cnt;
        }
        const int2 mine = make_int2(cnt, (cnt + kDtwIpw - 1) / kDtwIpw);
        int2 tot;
        const int2 inc = block_scan2(mine, warp_sums, tot);
        if (q < Qb) {
            s.item_off[q] = carry.x + inc.x - mine.x;
            s.chunk_off[q] = carry.y + inc.y - mine.y;
        }
        carry.x += tot.x;
        carry.y += tot.y;
    }
    if (threadIdx.x == 0) {
        s.item_off[Qb] = carry.x;
        s.chunk_off[Qb] = carry.y;
        s.counters[0] = carry.x;
        s.counters[1] = carry.y;
    }
}

__global__ void finalize_kernel(const unsigned long long *__restrict__ topk, int Qb, int k, int p,
                                int64_t index_base, int64_t *__restrict__ out_idx, float *__restrict__ out_dist) {
    const int64_t total = (int64_t)Qb * k;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = topk[t];
        if (key == ~0ull) { out_idx[t] = -1; out_dist[t] = kInf; continue; }
        const float d = __uint_as_float((uint32_t)(key >> 32));
        out_dist[t] = p == 1 ? d : sqrtf(d);
        out_idx[t] = index_base + (int64_t)(key & 0xffffffffu);
    }
}

// k-way shard merge: k smallest by (dist, idx) of G lists per query.
__global__ void nn_merge_kernel(const int64_t *__restrict__ in_idx, const float *__restrict__ in_dist, int G,
                                int64_t Q, int k, int64_t *__restrict__ out_idx, float *__restrict__ out_dist) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= Q) return;
    // G-way merge of sorted lists (each list ascending in (dist, idx))
    int head[64];
    for (int g = 0; g < G; ++g) head[g] = 0;
    for (int r = 0; r < k; ++r) {
        int best = -1;
        float bd = kInf;
        int64_t bi = 0x7fffffffffffffffLL;
        for (int g = 0; g < G; ++g) {
            if (head[g] >= k) continue;
            const int64_t o = ((int64_t)g * Q + q) * k + head[g];
            const int64_t ii = in_idx[o];
            if (ii < 0) continue;
            const float dd = in_dist[o];
            if (best < 0 || dd < bd || (dd == bd && ii < bi)) { best = g; bd = dd; bi = ii; }
        }
        if (best < 0) { out_idx[q * k + r] = -1; out_dist[q * k + r] = kInf; continue; }
        ++head[best];
        out_idx[q * k + r] = bi;
        out_dist[q * k + r] = bd;
    }
}

bool is_device_ptr(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

struct Timer {
    bool on;
    cudaStream_t st;
    cudaEvent_t e[8];
    int n = 0;
    Timer(bool on_, cudaStream_t s) : on(on_), st(s) {
        if (on) for (auto &x : e) cudaEventCreate(&x);
    }
    ~Timer() { if (on) for (auto &x : e) cudaEventDestroy(x); }
    void mark() { if (on && n < 8) cudaEventRecord(e[n++], st); }
    double ms(int a, int b) {
        float v = 0;
        if (on && b < n) cudaEventElapsedTime(&v, e[a], e[b]);
        return v;
    }
};

}  // namespace

int comm_allreduce_min(void *comm, float *thr, int64_t count, cudaStream_t st);  // comm.cu

// ------------------------------------------------------------------ pipeline
int nn_search_impl(const float *queries_in, int64_t Q, const float *db_in, int64_t N, int n, int w, int p,
                   int k, int64_t *out_idx_in, float *out_dist_in, const nn_opts *opts, nn_stats *stats,
                   cudaStream_t st) {
    std::lock_guard<std::mutex> lock(ws_mutex());
    const float eps = opts ? opts->eps : 1e-3f;
    const int64_t index_base = opts ? opts->index_base : 0;
    bool keogh_only = opts && (opts->flags & DTWLB_KEOGH_ONLY);
    // piecewise-sum pre-filter as the dense gate pass, LB_Keogh on its survivors;
    // not with few queries (stream mode below: the LB_Keogh pass is then memory-bound)
    bool prefilter = !(opts && (opts->flags & DTWLB_NO_PREFILTER));
    if (improved_epl(n) == 0) {
        // n > 1024: the survivor kernel keeps a pair's samples in one warp's registers (<= 1024),
        // so the search runs Alg. 2: LB_Keogh over every pair, then DTW -- exact,
        // without the LB_Improved pass (the key lists come from the dense LB_Keogh values)
        keogh_only = true;
        prefilter = false;
    }
    // DTW early abandon on rowmin + LB_Keogh terms of the remaining rows (reading c19)
    const bool cascade = !(opts && (opts->flags & DTWLB_NO_CASCADE));
    const bool no_abandon = opts && (opts->flags & DTWLB_NO_ABANDON);
    w = std::min(w, n - 1);
    Timer tm(stats != nullptr, st);
    tm.mark();  // 0
    const unsigned long long launches0 = __atomic_load_n(&g_launches, __ATOMIC_RELAXED);

    // ---- stage host inputs (e2e path) ----
    const float *queries = queries_in, *db = db_in;
    if (!is_device_ptr(queries_in)) {
        float *d;
        DTWLB_TRY(wsget(S_QSTAGE, (size_t)Q * n, &d));
        DTWLB_CUDA(cudaMemcpyAsync(d, queries_in, sizeof(float) * Q * n, cudaMemcpyHostToDevice, st));
        queries = d;
    }
    const float *db_host = nullptr;
    if (!is_device_ptr(db_in)) {
        float *d;
        DTWLB_TRY(wsget(S_DBSTAGE, (size_t)N * n, &d));
        db = d;
        db_host = db_in;
    }
    // stream mode (Q <= kStreamMaxQ): LB_Keogh of all Q queries in one streaming pass over the
    // database (stream.cu), no pre-filter
    const bool stream_mode = !(opts && (opts->flags & DTWLB_NO_STREAM)) && keogh_stream_ok(Q, n, db);
    if (stream_mode) prefilter = false;
    // A host database with the pre-filter (the e2e path): it is copied in chunks on a side stream
    // and the database-side setup and the first block's gate run chunk by chunk as the chunks
    // land, so the host->device copy hides behind the gate (bench e2e); else one copy up front
    const bool chunked = db_host && prefilter && !(opts && opts->db_env) &&
                         ws().get_copy_stream() != nullptr;
    if (db_host && !chunked)
        DTWLB_CUDA(cudaMemcpyAsync(const_cast<float *>(db), db_host, sizeof(float) * N * n, cudaMemcpyHostToDevice, st));
    const bool out_dev = is_device_ptr(out_idx_in) && is_device_ptr(out_dist_in);
    int64_t *out_idx = out_idx_in;
    float *out_dist = out_dist_in;
    if (!out_dev) {
        char *d;
        DTWLB_TRY(wsget(S_OUTSTAGE, (size_t)Q * k * 12, &d));
        out_idx = reinterpret_cast<int64_t *>(d);
        out_dist = reinterpret_cast<float *>(d + (size_t)Q * k * 8);
    }

    // ---- a1: envelopes ----
    const int epl = improved_epl(n);
    const int npadE = 32 * std::max(epl, 4);

    float *env;  // U, L, LU, UL, scratch: [5][Q][n]
    DTWLB_TRY(wsget(S_ENV, (size_t)5 * Q * n, &env));
    float *U = env, *L = env + (size_t)Q * n, *LU = env + 2 * (size_t)Q * n, *UL = env + 3 * (size_t)Q * n,
          *scr = env + 4 * (size_t)Q * n;
    DTWLB_TRY(launch_envelope(queries, n, w, U, L, Q, st));
    DTWLB_TRY(launch_envelope(L, n, w, LU, scr, Q, st));   // LU = U(L(y))
    DTWLB_TRY(launch_envelope(U, n, w, scr, UL, Q, st));   // UL = L(U(y))
    float *qpad;  // y, LU, UL (zero padded), U (+inf padded), L (-inf padded): [5][Q][npadE]
    DTWLB_TRY(wsget(S_QPAD, (size_t)5 * Q * npadE, &qpad));
    {
        const int grid = (int)std::min<int64_t>(ceil_div(Q * npadE, 256), 148 * 8);
        const float *src[5] = {queries, LU, UL, U, L};
        const float padv[5] = {0.f, 0.f, 0.f, kInf, -kInf};
        for (int a = 0; a < (prefilter ? 5 : 3); ++a) {
            pad_rows_kernel<<<grid, 256, 0, st>>>(src[a], Q, n, qpad + (size_t)a * Q * npadE, npadE, padv[a]);
            DTWLB_LAUNCH_CHECK();
        }
    }
    // piecewise sums in midpoint-radius form (the fused gate's operands, launch_paa_mid):
    // database sums [2][N][Dp] (m, r), query envelope boxes [2][Q][Dp] (m, r)
    const int Dp = paa_pitch(n);
    float *xpaa = nullptr, *qpaa = nullptr;
    if (prefilter) {
        DTWLB_TRY(wsget(S_PAA, (size_t)2 * N * Dp, &xpaa));
        DTWLB_TRY(wsget(S_QPAA, (size_t)2 * Q * Dp, &qpaa));
        if (!chunked) DTWLB_TRY(launch_paa_mid(db, db, N, n, xpaa, xpaa + (size_t)N * Dp, false, st));
        DTWLB_TRY(launch_paa_mid(L, U, Q, n, qpaa, qpaa + (size_t)Q * Dp, true, st));
    }
    const bool generic_dtw = w > 64;
    // row+column cascade of the w <= 32 DTW kernel (reading c21; C(i) = i + col_c0).  Off by
    // default: at C5 it cuts the computed DTW cells by 31 % but the per-step column work and
    // the rest0 pass cost as much as the cells save; DTWLB_COLCASC=1 enables it.
    static const bool env_col = [] { const char *e = getenv("DTWLB_COLCASC"); return e && atoi(e); }();
    const int col_c0 =
        (prefilter && !keogh_only && cascade && env_col && w <= 32 && n % 4 == 0) ? (w + 3) / 4 * 4 : 0;
    // abandon schedules (reading c22): the survivor kernel writes each appended pair's
    // precomputed row + column suffix bounds, the w <= 64 walk kernel abandons on them (no
    // per-step envelope gathers).  DTWLB_NO_SCHEDULE=1 keeps the row-only cascade (b1h)
    static const bool env_nosched = [] { const char *e = getenv("DTWLB_NO_SCHEDULE"); return e && atoi(e); }();
    const bool sched = prefilter && !keogh_only && cascade && !env_nosched && !generic_dtw && col_c0 == 0 &&
                       n % 4 == 0 && n <= 256 && (p == 1 || p == 2);
    const int LP = dtw_padded_len(n);
    float *ysh = nullptr;
    if (!generic_dtw) {
        DTWLB_TRY(wsget(S_YSH, (size_t)4 * Q * LP, &ysh));
        DTWLB_TRY(launch_build_ysh(queries, Q, n, ysh, LP, st));
    }
    // w > 64: the four-lanes-per-pair kernel (dtw_wide.cu) where instantiated, else the generic one
    int wide_S = 0, wide_padL = 0, wide_LPW = 0;
    const int wide_mode = generic_dtw ? dtw_wide_plan(n, w, &wide_S) : 0;
    float *ywide = nullptr;
    if (wide_mode) {
        wide_LPW = dtw_wide_padded(n, w, wide_S, &wide_padL);
        DTWLB_TRY(wsget(S_YSH, (size_t)Q * wide_LPW, &ywide));
        DTWLB_TRY(launch_build_ywide(queries, Q, n, ywide, wide_LPW, wide_padL, st));
    }
    // U(x), L(x): [2][N][n] -- the caller's database index (nn_opts.db_env) or computed here
    const float *dbenv = opts ? opts->db_env : nullptr;
    if (!dbenv && (!keogh_only || prefilter)) {
        float *e;
        DTWLB_TRY(wsget(S_DBENV, (size_t)2 * N * n, &e));
        if (!chunked) DTWLB_TRY(launch_envelope(db, n, w, e, e + (size_t)N * n, N, st));
        dbenv = e;
    }
    // symmetric gate (reading c20): the candidate envelope boxes [P(L(x)), P(U(x))] [2][N][Dp] and
    // the query sums P(y) [2][Q][Dp], midpoint-radius form
    float *rpaa = nullptr;
    if (prefilter) {
        DTWLB_TRY(wsget(S_RPAA, (size_t)2 * N * Dp + (size_t)2 * Q * Dp, &rpaa));
        if (!chunked)
            DTWLB_TRY(launch_paa_mid(dbenv + (size_t)N * n, dbenv, N, n, rpaa, rpaa + (size_t)N * Dp, true, st));
        float *yp = rpaa + (size_t)2 * N * Dp;
        DTWLB_TRY(launch_paa_mid(queries, queries, Q, n, yp, yp + (size_t)Q * Dp, false, st));
    }
    tm.mark();  // 1

    // ---- query block size from free memory ----
    const int qb_mode = (prefilter ? 1 : 0) | (keogh_only ? 2 : 0) | (stream_mode ? 4 : 0);
    const int64_t qb_hit = (opts && opts->query_block > 0) ? 0 : ws().cached_qb(Q, N, n, qb_mode);
    size_t free_b = 0, total_b = 0;
    if (!qb_hit) {
        DTWLB_CUDA(cudaMemGetInfo(&free_b, &total_b));
        // the block-sized slots this call would reuse count as free: the block size (hence the
        // pipeline) is then the same on every call of a given problem, not smaller after the first
        for (int sl : {S_BETA1, S_LIST, S_RES, S_MASK, S_COUNT}) free_b += ws().cur_size(sl);
    }
    // per query of the block: gate bound (2 B fp16 with the pre-filter, else 4 B) per pair, a
    // walk round's completed-pair slots (12 B per item, <= min(N, kDMax) items), the survivor
    // pass's (query, mask) entries (12 B per 64-candidate tile), and a budget for the key lists:
    // those are sized per range by the exact survivor count (8 B per gate survivor of the range,
    // list pool below); the budget assumes <= 1/8 of the pairs survive a range's gate on
    // average (C5: 3.8 %) -- a block whose lists do not fit is redone as two half blocks
    const size_t gate_elem = prefilter ? 2 : 4;
    const int64_t round_items = std::min<int64_t>(N, kDMax);
    const size_t per_q = (size_t)N * gate_elem + (size_t)N + (size_t)round_items * 12 + (size_t)ceil_div(N, 64) * 12 +
                         (size_t)ceil_div(N, kRun) * 8 + 4096;
    static const double env_mem = [] { const char *e = getenv("DTWLB_BLOCK_MEM_FRAC"); return e ? atof(e) : 0.0; }();
    // (0.6 of the free memory: one 8192-query block at C5, measured 274 vs 281 ms for 2 x 4096)
    const double mem_frac = env_mem > 0 ? env_mem : 0.6;
    int64_t Qb = opts && opts->query_block > 0 ? opts->query_block
                 : qb_hit                     ? qb_hit
                                              : (int64_t)(free_b * mem_frac / per_q);
    // a walk round holds <= Qb * min(N, kDMax) items, counted in int32 (plan_kernel, dtw4_kernel)
    Qb = std::min<int64_t>(Qb, (int64_t)(0x7fffffff - 1024) / round_items);
    Qb = std::max<int64_t>(1, std::min<int64_t>(Qb, Q));
    if (Qb >= 64) Qb = Qb / 64 * 64;
    if (!(opts && opts->query_block > 0) && Qb >= 64) {  // balance the blocks (e.g. 2 x 4096, not 7168 + 1024)
        const int64_t nb = ceil_div(Q, Qb);
        Qb = std::min<int64_t>(Qb, ceil_div(ceil_div(Q, nb), 64) * 64);
    }
    if (!qb_hit && !(opts && opts->query_block > 0)) ws().qb_cache.emplace_back(Q, N, n, qb_mode, Qb);
    const int64_t cap = N;
    const int64_t ldb = (N + 7) / 8 * 8;  // 16-byte rows of the fp16 gate block

    float *beta1;
    unsigned long long *list = nullptr;  // the range's exact-count key lists (pool, S_LIST)
    __half *srec = nullptr;              // the range's abandon schedules (S_REC), or NULL
    {   // float, or __half with the pre-filter
        void *g = nullptr;
        DTWLB_TRY(ws().get(S_BETA1, (size_t)Qb * ldb * gate_elem, &g));
        beta1 = static_cast<float *>(g);
    }
    const int64_t res_cap = Qb * round_items;  // items of one walk round (< 2^31, see Qb)
    char *rbuf;  // completed pairs of a round: keys [res_cap] u64 + queries [res_cap] int
    DTWLB_TRY(wsget(S_RES, (size_t)res_cap * 12 + 64, &rbuf));
    char *imp_scratch;
    DTWLB_TRY(wsget(S_MASK, improved_scratch_bytes(Qb, N), &imp_scratch));
    char *stb;
    const size_t st_bytes = (size_t)Qb * 4 * (11 + kMaxRanges) + (Qb + 2) * 8 * 2 + 64 + 64 + 16 * 16;
    DTWLB_TRY(wsget(S_STATE, st_bytes, &stb));
    QState s;
    {
        char *p_ = stb;
        auto take = [&](size_t bytes) { char *r = p_; p_ += (bytes + 15) / 16 * 16; return r; };
        s.stat = reinterpret_cast<unsigned long long *>(take(8 * 8));
        s.counters = reinterpret_cast<int *>(take(64));
        s.thr = reinterpret_cast<float *>(take(Qb * 4));
        s.lo = reinterpret_cast<float *>(take(Qb * 4));
        s.hi = reinterpret_cast<float *>(take(Qb * 4));
        s.tS = reinterpret_cast<float *>(take(Qb * 4 * (kMaxRanges - 1)));
        s.len = reinterpret_cast<int *>(take(Qb * 4));
        s.pos = reinterpret_cast<int *>(take(Qb * 4));
        s.rnd = reinterpret_cast<int *>(take(Qb * 4));
        s.active = reinterpret_cast<int *>(take(Qb * 4));
        s.lock = reinterpret_cast<int *>(take(Qb * 4));
        s.prev_cnt = reinterpret_cast<int *>(take(Qb * 4));
        s.item_off = reinterpret_cast<int *>(take((Qb + 1) * 4));
        s.chunk_off = reinterpret_cast<int *>(take((Qb + 1) * 4));
        s.q_count = reinterpret_cast<int *>(take(Qb * 4));
        s.loff = reinterpret_cast<int64_t *>(take((Qb + 2) * 8));
    }
    DTWLB_TRY(wsget(S_TOPK, (size_t)Qb * k, &s.topk));
    DTWLB_CUDA(cudaMemsetAsync(s.stat, 0, 8 * 8, st));

    // target size of the first (best-first) range: ~kSeedCap candidates per query.  Measured at
    // C5 (ms/step): 8192 -> 323, 4096 -> 310, 2048 -> 304, 1536 -> 303, 1024 -> 302-322; three
    // ranges were slower (326-338): the seed range's survivor pass is dominated by per-entry
    // cost (about one survivor per (query, 64-tile) entry), so a smaller seed is cheaper
    static const int env_S = [] { const char *e = getenv("DTWLB_SEED"); return e ? atoi(e) : 0; }();
    // (a database shard seeds from 1/G of the whole database's seed range, nn_opts.shards)
    const int64_t shards = opts && opts->shards > 1 ? opts->shards : 1;
    // the shard threshold exchange: the caller's callback, or the library's NCCL all-reduce MIN
    const bool has_exchange = opts && (opts->exchange || opts->nccl_comm);
    auto exchange_thr = [&](float *thr, int64_t count) -> int {
        if (opts->exchange) {
            opts->exchange(thr, count, opts->exchange_user);
            DTWLB_CUDA(cudaGetLastError());
            return DTWLB_OK;
        }
        return comm_allreduce_min(opts->nccl_comm, thr, count, st);
    };
    // (N / 768: measured seed sweeps, profiles/r02n_seed_sweep.txt -- C5 (N = 10^6) is flat for
    // S in 512..2048, C3 (10^5) and C4 (2 10^5) are 7-9 % faster at 256 than at the old N/64)
    const int64_t S = std::max<int64_t>(std::max<int64_t>(256, 4LL * k),
                                        std::min<int64_t>((env_S > 0 ? env_S : kSeedCap) / shards,
                                                          env_S > 0 ? (int64_t)env_S : N / 768));
    // number of ranges R and the growth G of their sampled sizes (S, S*G, S*G^2, ..., rest)
    static const int env_R = [] { const char *e = getenv("DTWLB_RANGES"); return e ? atoi(e) : 0; }();
    static const int env_G = [] { const char *e = getenv("DTWLB_RANGE_GROWTH"); return e ? atoi(e) : 0; }();
    const int R = std::min(kMaxRanges, std::max(2, env_R > 0 ? env_R : 2));
    const int G = std::max(2, env_G > 0 ? env_G : 8);

    // run lists of the sort: at most sum_q ceil(len_q / kRun) <= Qb + total / kRun runs of
    // (query, index), + the count; sized per range with the lists
    int64_t max_runs = 0;
    int *d_runs = nullptr, *d_nruns = nullptr;
    double ms_keogh = 0, ms_select = 0, ms_improved = 0, ms_dtw = 0, ms_survivor = 0, ms_dtw_kernel = 0;
    int64_t walk_rounds = 0;
    // stats: CUDA-event spans resolved after the call's final synchronisation (no host waits
    // inside the pipeline); the range-1 counters are device-to-device snapshots
    std::vector<cudaEvent_t> evpool;
    std::vector<std::tuple<cudaEvent_t, cudaEvent_t, double *>> spans;
    auto new_ev = [&]() { cudaEvent_t e; cudaEventCreate(&e); evpool.push_back(e); return e; };
    auto rec = [&]() { cudaEvent_t e = new_ev(); cudaEventRecord(e, st); return e; };
    auto span = [&](cudaEvent_t a, cudaEvent_t b, double *acc) { spans.emplace_back(a, b, acc); };
    // blocks actually run (a block whose key lists do not fit is redone as two half blocks)
    const int64_t snap_cap = 4 * ceil_div(Q, Qb) + 64;
    int64_t nblocks = 0;
    unsigned long long *snap = nullptr;  // [blocks][2][4]: stat after range 1, after the last range
    if (stats) DTWLB_TRY(wsget(S_SNAP, (size_t)snap_cap * 8 + 8, &snap));
    unsigned long long *stat_save = stats ? snap + snap_cap * 8 : nullptr;  // stat at the block start
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_s0 = nullptr, ev_s1 = nullptr;

    int64_t gate0_qn = -1;  // rows of the first block whose gate ran with the chunked copy
    if (chunked) {
        cudaStream_t cs = ws().get_copy_stream();
        cudaEvent_t e_in;
        DTWLB_CUDA(cudaEventCreateWithFlags(&e_in, cudaEventDisableTiming));
        DTWLB_CUDA(cudaEventRecord(e_in, st));  // the staging buffer is free once st gets here
        DTWLB_CUDA(cudaStreamWaitEvent(cs, e_in, 0));
        cudaEventDestroy(e_in);
        const int64_t qn0 = std::min<int64_t>(Qb, Q);
        const int64_t rows_per = std::max<int64_t>(1, std::min<int64_t>(131072, ceil_div(N, 4)));
        const float *yp = rpaa + (size_t)2 * N * Dp;
        float *dbs = const_cast<float *>(db);
        float *ex = const_cast<float *>(dbenv);
        for (int64_t r0 = 0; r0 < N; r0 += rows_per) {
            const int64_t cnt = std::min<int64_t>(rows_per, N - r0);
            cudaEvent_t e_c;
            DTWLB_CUDA(cudaEventCreateWithFlags(&e_c, cudaEventDisableTiming));
            DTWLB_CUDA(cudaMemcpyAsync(dbs + r0 * n, db_host + r0 * n, sizeof(float) * cnt * n,
                                       cudaMemcpyHostToDevice, cs));
            DTWLB_CUDA(cudaEventRecord(e_c, cs));
            DTWLB_CUDA(cudaStreamWaitEvent(st, e_c, 0));
            cudaEventDestroy(e_c);
            DTWLB_TRY(launch_paa_mid(db + r0 * n, db + r0 * n, cnt, n, xpaa + r0 * Dp, xpaa + (size_t)N * Dp + r0 * Dp,
                                     false, st));
            DTWLB_TRY(launch_envelope(db + r0 * n, n, w, ex + r0 * n, ex + (size_t)N * n + r0 * n, cnt, st));
            DTWLB_TRY(launch_paa_mid(ex + (size_t)N * n + r0 * n, ex + r0 * n, cnt, n, rpaa + r0 * Dp,
                                     rpaa + (size_t)N * Dp + r0 * Dp, true, st));
            const cudaEvent_t g0 = stats ? rec() : nullptr;
            DTWLB_TRY(launch_paa_bound_sym(qpaa, qpaa + (size_t)Q * Dp, yp, yp + (size_t)Q * Dp, xpaa + r0 * Dp,
                                           xpaa + (size_t)N * Dp + r0 * Dp, rpaa + r0 * Dp,
                                           rpaa + (size_t)N * Dp + r0 * Dp, qn0, cnt, n, p, false,
                                           reinterpret_cast<__half *>(beta1) + r0, ldb, st));
            if (stats) span(g0, rec(), &ms_keogh);
        }
        gate0_qn = qn0;
    }
    int64_t Qcur = Qb;  // current block size
    int64_t rcap = cap;               // the range's list capacity per query (uniform lists)
    const int64_t *loff_r = nullptr;  // or its exact per-query offsets
    for (int64_t qb0 = 0; qb0 < Q;) {
        const int64_t qn = std::min<int64_t>(Qcur, Q - qb0);
        bool redo = false;  // the range's key lists did not fit: redo this block as two halves
        if (stats) DTWLB_CUDA(cudaMemcpyAsync(stat_save, s.stat, 64, cudaMemcpyDeviceToDevice, st));
        // ---- dense gate pass for the block: the piecewise-sum bound beta0 (pre-filter,
        //      LB_Keogh then runs on its survivors inside the survivor pass), or a2 itself ----
        if (stats) ev0 = rec();
        if (prefilter) {
            // symmetric gate: max of the forward and the reverse piecewise-sum bounds (readings c18,
            // c20), one fused tile pass
            const float *yp = rpaa + (size_t)2 * N * Dp;
            if (qb0 == 0 && qn == gate0_qn) {
                // (computed chunk by chunk with the database copy, above)
            } else {
                DTWLB_TRY(launch_paa_bound_sym(qpaa + qb0 * Dp, qpaa + (size_t)Q * Dp + qb0 * Dp, yp + qb0 * Dp,
                                               yp + (size_t)Q * Dp + qb0 * Dp, xpaa, xpaa + (size_t)N * Dp, rpaa,
                                               rpaa + (size_t)N * Dp, qn, N, n, p, false, beta1, ldb, st));
            }
        } else if (stream_mode)
            DTWLB_TRY(launch_keogh_stream(U + qb0 * n, L + qb0 * n, db, qn, N, n, p, false, beta1, ldb, st));
        else
            DTWLB_TRY(launch_keogh(U + qb0 * n, L + qb0 * n, db, qn, N, n, p, false, beta1, ldb, st));
        if (stats) ev1 = rec();
        init_state_kernel<<<(unsigned)ceil_div(qn, 256), 256, 0, st>>>(s, (int)qn, k);
        DTWLB_LAUNCH_CHECK();
        if (prefilter)
            sample_threshold_kernel<__half><<<(unsigned)qn, 512, 0, st>>>(reinterpret_cast<const __half *>(beta1),
                                                                         ldb, N, S, R, G, s.tS, (int)qn);
        else
            sample_threshold_kernel<float><<<(unsigned)qn, 512, 0, st>>>(beta1, ldb, N, S, R, G, s.tS, (int)qn);
        DTWLB_LAUNCH_CHECK();
        if (stats) {
            const cudaEvent_t e2 = rec();
            span(ev0, ev1, &ms_keogh);
            span(ev1, e2, &ms_select);
        }

        for (int macro = 0; macro < R; ++macro) {
            set_range_kernel<<<(unsigned)ceil_div(qn, 256), 256, 0, st>>>(s, (int)qn, macro, R);
            DTWLB_LAUNCH_CHECK();
            if (stats) ev0 = rec();
            // ---- a4: LB_Improved on the range's LB_Keogh survivors ----
            {
                ImprovedArgs ia{};
                ia.yq = qpad + qb0 * npadE;
                ia.LUq = qpad + (size_t)Q * npadE + qb0 * npadE;
                ia.ULq = qpad + 2 * (size_t)Q * npadE + qb0 * npadE;
                if (prefilter) {
                    ia.Uq = qpad + 3 * (size_t)Q * npadE + qb0 * npadE;
                    ia.Lq = qpad + 4 * (size_t)Q * npadE + qb0 * npadE;
                    ia.xdb = db;
                    ia.gate_w = reinterpret_cast<__half *>(beta1);
                    ia.gate_half = true;
                    ia.n_eval_keogh = s.stat + 4;
                }
                ia.Ux = dbenv;
                ia.Lx = dbenv ? dbenv + (size_t)N * n : nullptr;
                ia.gate = beta1;
                ia.ldb = ldb;
                ia.Qb = qn;
                ia.N = N;
                ia.n = n;
                ia.npadE = npadE;
                ia.lo = s.lo;
                ia.hi = s.hi;
                ia.thr = s.thr;
                ia.cap = cap;
                ia.loff = nullptr;  // (set below with the lists)
                ia.q_count = s.q_count;
                ia.list_len = s.len;
                ia.n_eval = s.stat + 0;
                ia.n_entries = s.stat + 5;
                if (stats) { ev_s0 = new_ev(); ev_s1 = new_ev(); ia.ev0 = ev_s0; ia.ev1 = ev_s1; }
                improved_scratch_bind(ia, imp_scratch);
                DTWLB_TRY(launch_select(ia, false, st));
                // exact-count key lists: the range's gate survivors per query bound its keys
                list_offsets_kernel<<<1, 1024, 0, st>>>(s.q_count, (int)qn, s.loff);
                DTWLB_LAUNCH_CHECK();
                int64_t tm2[2] = {0, 0};  // total keys, largest count
                DTWLB_CUDA(cudaMemcpyAsync(tm2, s.loff + qn, sizeof(tm2), cudaMemcpyDeviceToHost, st));
                DTWLB_CUDA(cudaStreamSynchronize(st));
                const int64_t total = tm2[0];
                // lists of a uniform capacity (the range's largest count: the survivor kernel's
                // append then needs no per-query offset load, measured 84 vs 92 ms at C5), or
                // exact per-query offsets when the uniform ones do not fit
                rcap = std::max<int64_t>(tm2[1], 1);
                loff_r = nullptr;
                if (wsget(S_LIST, (size_t)qn * rcap, &list) != DTWLB_OK) {
                    cudaGetLastError();
                    loff_r = s.loff;
                }
                const int64_t nkeys = loff_r ? total : qn * rcap;
                max_runs = qn + nkeys / kRun + 1;
                // (DTWLB_LIST_POOL_MAX: a cap on the pool in keys, to exercise the redo path in tests)
                static const long long pool_max = [] { const char *e = getenv("DTWLB_LIST_POOL_MAX"); return e ? atoll(e) : 0LL; }();
                const bool over = pool_max > 0 && nkeys > pool_max;
                if (over) set_error(DTWLB_ENOMEM, "key lists of %lld keys exceed DTWLB_LIST_POOL_MAX", (long long)total);
                if (over || (loff_r && wsget(S_LIST, (size_t)std::max<int64_t>(total, 1), &list) != DTWLB_OK) ||
                    wsget(S_COUNT, (size_t)max_runs * 2 + 64, &d_runs) != DTWLB_OK) {
                    if (qn == 1 || has_exchange) return DTWLB_ENOMEM;  // (error set by wsget)
                    redo = true;
                    break;
                }
                d_nruns = d_runs + 2 * max_runs;
                ia.list = list;
                ia.cap = rcap;
                ia.loff = loff_r;
                // schedules at the exact per-query offsets s.loff (gate survivors), whatever the
                // key lists' layout
                srec = nullptr;
                if (sched && total < (1LL << 31) && wsget(S_REC, (size_t)std::max<int64_t>(total, 1) * 32, &srec) != DTWLB_OK) {
                    cudaGetLastError();  // no room: this range keeps the row-only cascade
                    srec = nullptr;
                }
                ia.rec = srec;
                ia.rec_off = s.loff;
                ia.rec_c0b = (w + 3) / 4;  // (w <= 64: <= 16)
                DTWLB_TRY(launch_survivor(ia, p, keogh_only, false, st));
            }
            // ---- a3: sort each query's list in runs (run list built on the device) ----
            if (stats) span(ev_s0, ev_s1, &ms_survivor);
            {
                static const bool dbg_keys = [] { const char *e = getenv("DTWLB_DEBUG_ROUNDS"); return e && atoi(e); }();
                if (stats && dbg_keys) {  // (debug: the range's appended keys; syncs)
                    std::vector<int> lens((size_t)qn);
                    DTWLB_CUDA(cudaMemcpyAsync(lens.data(), s.len, sizeof(int) * qn, cudaMemcpyDeviceToHost, st));
                    DTWLB_CUDA(cudaStreamSynchronize(st));
                    long long sum = 0;
                    for (int v : lens) sum += v;
                    fprintf(stderr, "[dtwlb] range %d: %lld keys appended, schedules %s\n", macro, sum,
                            srec ? "on" : "off");
                }
            }
            static const bool nosort2 = [] { const char *e = getenv("DTWLB_NOSORT2"); return e && atoi(e); }();
            const bool sorted = !(nosort2 && macro > 0);
            if (sorted || col_c0 > 0) {
                make_runs_kernel<<<1, 1024, 0, st>>>(s.len, (int)qn, d_runs, d_runs + max_runs, d_nruns);
                DTWLB_LAUNCH_CHECK();
                const unsigned grid = (unsigned)std::min<int64_t>(max_runs, 148 * 8);
                if (sorted) {
                    sort_runs_kernel<<<grid, kSortThreads, 0, st>>>(list, rcap, loff_r, d_runs, d_runs + max_runs,
                                                                    s.len, d_nruns);
                    DTWLB_LAUNCH_CHECK();
                }
                if (col_c0 > 0) {  // row+column cascade start values (reading c21)
                    auto rk = p == 1 ? rest0_kernel<1> : rest0_kernel<2>;
                    rk<<<grid, 256, 0, st>>>(list, rcap, loff_r, d_runs, d_runs + max_runs, s.len, d_nruns, queries + qb0 * n,
                                             LU + qb0 * n, UL + qb0 * n, dbenv, dbenv + (size_t)N * n, n, col_c0,
                                             reinterpret_cast<__half *>(beta1), ldb);
                    DTWLB_LAUNCH_CHECK();
                }
            }
            if (stats) ev1 = rec();
            // ---- a5: DTW walk ----
            start_walk_kernel<<<(unsigned)ceil_div(qn, 256), 256, 0, st>>>(s, (int)qn);
            DTWLB_LAUNCH_CHECK();
            // The w <= 64 DTW kernels read each round's item count from device memory (written by
            // the plan kernel), so rounds are queued in batches of kRoundBatch with one host
            // check per batch; the generic kernel sizes its grid from it (one check per round).
            const bool dev_rounds = !generic_dtw;  // (w <= 64: the dtw4 kernels)
            const int batch = dev_rounds ? kRoundBatch : 1;
            // shard threshold exchanges inside the last range's walk (nn_opts.exchange_walk):
            // after its rounds 2, 4, .., 2 * ex_walk; calls left when the walk ends early are made
            // after it, so every shard makes the same number of calls per block
            const int ex_walk = (has_exchange && macro == R - 1 && macro > 0)
                                    ? std::max(0, std::min(3, (int)opts->exchange_walk)) : 0;
            int range_round = 0, ex_done = 0;
            for (bool walking = true; walking;) {
                for (int b = 0; b < batch && walking; ++b) {
                    ++walk_rounds;
                    ++range_round;
                    static const int env_d0 = [] { const char *e = getenv("DTWLB_D0"); return e ? atoi(e) : 0; }();
                    // batch per query and round: kD0 << (round * gs).  The first round stays small (its
                    // pairs run with tau = +inf: none is abandoned, and every completed pair is merged
                    // into the query's top-k under its lock); later batches grow 8x per round: a round
                    // costs its launches, its merge and the tail of its longest pair (a ~n-step
                    // chain), so fewer, fuller rounds win although tau tightens less often between
                    // them (measured, DESIGN.md a3: C5 267.8 -> 265.5 ms, C4 43.0 -> 41.7, C3 w = 100
                    // 56.6 -> 47.3; 2x growth was the default for more than 64 queries before)
                    const int d0 = env_d0 > 0 ? env_d0 : kD0;
                    static const int env_gs = [] { const char *e = getenv("DTWLB_WALK_GS"); return e ? atoi(e) : 0; }();
                    const int gs = env_gs > 0 ? env_gs : 3;
                    plan_kernel<<<1, 1024, 0, st>>>(s, (int)qn, list, rcap, loff_r, sorted, d0, gs);
                    DTWLB_LAUNCH_CHECK();
                    int tot2[2] = {0, 0};
                    if (!dev_rounds) {
                        DTWLB_CUDA(cudaMemcpyAsync(tot2, s.counters, sizeof(tot2), cudaMemcpyDeviceToHost, st));
                        DTWLB_CUDA(cudaStreamSynchronize(st));
                        if (tot2[0] == 0) { walking = false; break; }
                    }
                    DtwArgs da{};
                    da.no_abandon = no_abandon;
                    da.ysh = ysh;
                    da.ysh_stride_s = (int64_t)Q * LP;
                    da.LP = LP;
                    da.db = db;
                    da.Ndb = N;
                    da.n = n;
                    da.w = w;
                    da.item_off = s.item_off;
                    da.chunk_off = s.chunk_off;
                    da.nchunks = tot2[1];
                    da.pos = s.pos;
                    da.list = list;
                    da.cap = rcap;
                    da.loff = loff_r;
                    da.Qb = (int)qn;
                    da.thr = s.thr;
                    da.topk = s.topk;
                    da.topk_lock = s.lock;
                    da.k = k;
                    da.eps = eps;
                    da.rkey = reinterpret_cast<unsigned long long *>(rbuf);
                    da.rq = reinterpret_cast<int *>(rbuf + (size_t)res_cap * 8);
                    da.rcount = reinterpret_cast<unsigned *>(s.counters + 6);
                    da.rcap = res_cap;
                    DTWLB_CUDA(cudaMemsetAsync(da.rcount, 0, sizeof(unsigned), st));
                    da.total = dev_rounds ? res_cap : tot2[0];  // (dev_rounds: grid bound only)
                    da.dev_total = dev_rounds ? s.counters : nullptr;
                    da.cells = s.stat + 2;
                    da.abandoned = s.stat + 3;
                    da.started = s.stat + 1;
                    da.queue = reinterpret_cast<unsigned *>(s.counters + 4);
                    da.rec = srec;  // (the schedules of this range's keys, or NULL)
                    da.rec_off = s.loff;
                    if (cascade) {  // cascading abandon with the pair's LB_Keogh row terms
                        if (prefilter) da.b1h = reinterpret_cast<const __half *>(beta1);
                        else da.b1 = beta1;
                        da.ldb = ldb;
                        da.Uq = U + qb0 * n;
                        da.Lq = L + qb0 * n;
                        if (col_c0 > 0) {
                            da.col_c0 = col_c0;
                            da.yq = queries + qb0 * n;
                            da.LUq = LU + qb0 * n;
                            da.ULq = UL + qb0 * n;
                            da.Uxdb = dbenv;
                            da.Lxdb = dbenv + (size_t)N * n;
                        }
                    }
                    if (wide_mode) {
                        const cudaEvent_t d0 = stats ? rec() : nullptr;
                        DTWLB_TRY(launch_dtw_wide(da, ywide + (size_t)qb0 * wide_LPW, wide_LPW, wide_padL, p, true, st));
                        if (stats) span(d0, rec(), &ms_dtw_kernel);
                    } else if (generic_dtw) {
                        // global band scratch only when 128 bands do not fit in shared memory,
                        // sized by this round's item count
                        float *scratch = nullptr;
                        if (dtw_generic_needs_scratch(w))
                            DTWLB_TRY(wsget(S_SCRATCH, (size_t)tot2[0] * (2 * w + 2), &scratch));
                        const cudaEvent_t d0 = stats ? rec() : nullptr;
                        DTWLB_TRY(launch_dtw_generic(da, queries + qb0 * n, scratch, p, true, st));
                        if (stats) span(d0, rec(), &ms_dtw_kernel);
                    }
                    else {
                        da.ysh = ysh + qb0 * LP;
                        const cudaEvent_t d0 = stats ? rec() : nullptr;
                        DTWLB_TRY(launch_dtw(da, p, true, st));
                        if (stats) span(d0, rec(), &ms_dtw_kernel);
                        static const bool dbg_rounds = [] { const char *e = getenv("DTWLB_DEBUG_ROUNDS"); return e && atoi(e); }();
                        if (stats && dbg_rounds) {  // per-round items, time and cells (debug: syncs)
                            const cudaEvent_t d1 = evpool.back();
                            DTWLB_CUDA(cudaStreamSynchronize(st));
                            float ms_r = 0;
                            cudaEventElapsedTime(&ms_r, d0, d1);
                            int c2[2];
                            unsigned long long h4[4];
                            DTWLB_CUDA(cudaMemcpy(c2, s.counters, sizeof(c2), cudaMemcpyDeviceToHost));
                            DTWLB_CUDA(cudaMemcpy(h4, s.stat, sizeof(h4), cudaMemcpyDeviceToHost));
                            static unsigned long long prev[4] = {0, 0, 0, 0};
                            if (h4[1] < prev[1]) prev[0] = prev[1] = prev[2] = prev[3] = 0;  // a new call
                            fprintf(stderr, "[dtwlb] range %d round %lld: items %d, %.3f ms, started %llu, cells %llu, abandoned %llu, %.3g cells/s\n",
                                    macro, (long long)walk_rounds, c2[0], ms_r, h4[1] - prev[1], h4[2] - prev[2],
                                    h4[3] - prev[3], ms_r > 0 ? (double)(h4[2] - prev[2]) / (ms_r * 1e-3) : 0.0);
                            for (int j = 0; j < 4; ++j) prev[j] = h4[j];
                        }
                    }
                    DTWLB_TRY(launch_topk_merge(da, st));  // a6: the round's completed pairs -> top-k, tau
                    if (ex_done < ex_walk && range_round == 2 * (ex_done + 1)) {
                        DTWLB_TRY(exchange_thr(s.thr, qn));  // (stream-ordered)
                        ++ex_done;
                    }
                }
                if (dev_rounds && walking) {  // one host check per batch: did the last round have items?
                    int tot0 = 0;
                    DTWLB_CUDA(cudaMemcpyAsync(&tot0, s.counters, sizeof(int), cudaMemcpyDeviceToHost, st));
                    DTWLB_CUDA(cudaStreamSynchronize(st));
                    walking = tot0 > 0;
                }
            }
            for (; ex_done < ex_walk; ++ex_done)  // the walk ended before its scheduled exchanges
                DTWLB_TRY(exchange_thr(s.thr, qn));
            if (has_exchange && macro + 1 < R) {
                // a7: shard threshold exchange after the best-first range (stream-ordered)
                DTWLB_TRY(exchange_thr(s.thr, qn));
            }
            if (stats) {
                const cudaEvent_t e2 = rec();
                span(ev0, ev1, &ms_improved);
                span(ev1, e2, &ms_dtw);
                if (macro == 0 || macro == R - 1)  // cumulative counters after range 1 / the block
                    if (nblocks < snap_cap)
                    DTWLB_CUDA(cudaMemcpyAsync(snap + nblocks * 8 + (macro == 0 ? 0 : 4), s.stat, 32,
                                               cudaMemcpyDeviceToDevice, st));
            }
        }
        if (redo) {  // undo the block's counters, then redo it as two half blocks
            if (stats) DTWLB_CUDA(cudaMemcpyAsync(s.stat, stat_save, 64, cudaMemcpyDeviceToDevice, st));
            cudaGetLastError();
            Qcur = std::max<int64_t>(1, qn / 2);
            continue;
        }
        finalize_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(qn * k, 256), 4096)), 256, 0, st>>>(
            s.topk, (int)qn, k, p, index_base, out_idx + qb0 * k, out_dist + qb0 * k);
        DTWLB_LAUNCH_CHECK();
        qb0 += qn;
        ++nblocks;
    }
    if (!out_dev) {
        DTWLB_CUDA(cudaMemcpyAsync(out_idx_in, out_idx, sizeof(int64_t) * Q * k, cudaMemcpyDeviceToHost, st));
        DTWLB_CUDA(cudaMemcpyAsync(out_dist_in, out_dist, sizeof(float) * Q * k, cudaMemcpyDeviceToHost, st));
    }
    tm.mark();  // 2
    DTWLB_CUDA(cudaStreamSynchronize(st));
    static const bool dbg_spans = [] { const char *e = getenv("DTWLB_DEBUG_SPANS"); return e && atoi(e); }();
    if (stats && dbg_spans) fprintf(stderr, "[dtwlb] Q %lld N %lld: query block %lld\n", (long long)Q, (long long)N, (long long)Qb);
    if (stats && dbg_spans && !evpool.empty()) {
        float g0 = 0, g1 = 0;
        cudaEventElapsedTime(&g0, tm.e[1], evpool.front());
        cudaEventElapsedTime(&g1, evpool.back(), tm.e[2]);
        float gfl = 0, g12 = 0;
        cudaEventElapsedTime(&gfl, evpool.front(), evpool.back());
        cudaEventElapsedTime(&g12, tm.e[1], tm.e[2]);
        fprintf(stderr, "[dtwlb] setup->first span %.2f ms, last span->end %.2f ms, envelope %.2f ms, first->last %.2f, "
                "mark1->mark2 %.2f, total %.2f, %zu events\n", g0, g1, tm.ms(0, 1), gfl, g12, tm.ms(0, 2), evpool.size());
    }
    if (stats && dbg_spans) {  // uncovered device time between consecutive spans (debug)
        for (size_t t = 0; t + 1 < evpool.size(); ++t) {
            float g = 0;
            if (cudaEventElapsedTime(&g, evpool[t], evpool[t + 1]) == cudaSuccess && g > 0.02f)
                fprintf(stderr, "[dtwlb] events %zu -> %zu: %.2f ms\n", t, t + 1, g);
        }
    }
    if (stats) {
        for (auto &sp : spans) {
            float t = 0;
            cudaEventElapsedTime(&t, std::get<0>(sp), std::get<1>(sp));
            *std::get<2>(sp) += t;
        }
        for (auto &e : evpool) cudaEventDestroy(e);
        const int64_t nsnap = std::min(nblocks, snap_cap);
        std::vector<unsigned long long> hs((size_t)std::max<int64_t>(nsnap, 1) * 8);
        if (nsnap) DTWLB_CUDA(cudaMemcpy(hs.data(), snap, (size_t)nsnap * 64, cudaMemcpyDeviceToHost));
        unsigned long long r1[3] = {0, 0, 0};
        for (int64_t b = 0; b < nsnap; ++b)
            for (int j = 0; j < 3; ++j) r1[j] += hs[b * 8 + j] - (b ? hs[(b - 1) * 8 + 4 + j] : 0ull);
        unsigned long long h[8];
        DTWLB_CUDA(cudaMemcpy(h, s.stat, sizeof(h), cudaMemcpyDeviceToHost));
        stats->pairs = Q * N;
        stats->keogh_evaluated = prefilter ? (int64_t)h[4] : Q * N;
        stats->prefilter_evaluated = prefilter ? Q * N : 0;
        stats->prefilter_segment = prefilter ? kSeg : 0;
        stats->improved_evaluated = (int64_t)h[0];
        stats->dtw_cells_computed = (int64_t)h[2];
        stats->dtw_abandoned = (int64_t)h[3];
        stats->dtw_evaluated = (int64_t)h[1];
        stats->dtw_cells_nominal = (int64_t)h[1] * (int64_t)(n * (2 * w + 1) - w * (w + 1));
        stats->ms_envelope = tm.ms(0, 1);
        stats->ms_keogh = ms_keogh;
        stats->ms_select = ms_select;
        stats->ms_improved = ms_improved;
        stats->ms_survivor_kernel = ms_survivor;
        stats->ms_dtw_kernel = ms_dtw_kernel;
        stats->ms_dtw = ms_dtw;
        stats->ms_total = tm.ms(0, 2);
        stats->kernel_launches = (int64_t)(__atomic_load_n(&g_launches, __ATOMIC_RELAXED) - launches0);
        stats->range1_improved = (int64_t)r1[0];
        stats->range1_dtw = (int64_t)r1[1];
        stats->range1_cells = (int64_t)r1[2];
        stats->walk_rounds = walk_rounds;
        stats->survivor_entries = (int64_t)h[5];
    }
    return DTWLB_OK;
}

int nn_merge_impl(const int64_t *in_idx, const float *in_dist, int G, int64_t Q, int k, int64_t *out_idx,
                  float *out_dist, cudaStream_t st) {
    if (Q == 0) return DTWLB_OK;
    nn_merge_kernel<<<(unsigned)ceil_div(Q, 128), 128, 0, st>>>(in_idx, in_dist, G, Q, k, out_idx, out_dist);
    DTWLB_LAUNCH_CHECK();
    return DTWLB_OK;
}

// workspace access for abi.cu (dense entry points)
int ws_get_bytes(int slot, size_t bytes, void **out) {
    return ws().get(S_COUNT + 1 + slot, bytes, out);
}
std::mutex &api_mutex() { return ws_mutex(); }
void release_workspace() {
    std::lock_guard<std::mutex> lock(ws_mutex());
    cudaDeviceSynchronize();
    for (int d = 0; d < kMaxDevices; ++d) ws_all()[d].release();
}

}  // namespace dtwlb
