// abi.cu -- the extern "C" boundary of libdtwlb (declared in include/dtwlb.h):
// argument validation, the thread-local error model, and dispatch to the kernels.
#include <cstring>
#include <mutex>

#include "kernels.cuh"

namespace dtwlb {

int nn_search_impl(const float *queries, int64_t Q, const float *db, int64_t N, int n, int w, int p, int k,
                   int64_t *out_idx, float *out_dist, const nn_opts *opts, nn_stats *stats, cudaStream_t st);
int nn_merge_impl(const int64_t *in_idx, const float *in_dist, int G, int64_t Q, int k, int64_t *out_idx,
                  float *out_dist, cudaStream_t st);
int launch_dtw_generic(const DtwArgs &a, const float *yraw, float *scratch, int p, bool walk, cudaStream_t st);
int ws_get_bytes(int slot, size_t bytes, void **out);
std::mutex &api_mutex();
void release_workspace();

unsigned long long g_launches = 0;
static thread_local char g_err[512] = "";

void set_error(int code, const char *fmt, ...) {
    (void)code;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int cuda_fail(cudaError_t e, const char *what, const char *file, int line) {
    set_error(DTWLB_ECUDA, "CUDA error %s (%s) at %s:%d in %s", cudaGetErrorName(e), cudaGetErrorString(e),
              file, line, what);
    return DTWLB_ECUDA;
}

int require_device() {
    // checked once per device ordinal (the current device of the calling thread)
    constexpr int kMaxDev = 64;
    static int state[kMaxDev + 1];  // 0 unknown, 1 ok, else 1 + status
    static char msg[kMaxDev + 1][256];
    static std::mutex m;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    const int slot = (e != cudaSuccess || dev < 0 || dev >= kMaxDev) ? kMaxDev : dev;
    std::lock_guard<std::mutex> lock(m);
    if (state[slot] == 0) {
        cudaDeviceProp prop;
        if (e == cudaSuccess) e = cudaGetDeviceProperties(&prop, dev);
        if (e != cudaSuccess) {
            cudaGetLastError();
            snprintf(msg[slot], sizeof(msg[slot]), "no usable CUDA device: %s", cudaGetErrorString(e));
            state[slot] = 1 + DTWLB_ECUDA;
        } else if (prop.major != 10) {
            snprintf(msg[slot], sizeof(msg[slot]), "device %s is sm_%d%d; libdtwlb is built for sm_100a only",
                     prop.name, prop.major, prop.minor);
            state[slot] = 1 + DTWLB_ECUDA;
        } else {
            state[slot] = 1;
        }
    }
    const int st = state[slot] - 1;
    if (st != DTWLB_OK) set_error(st, "%s", msg[slot]);
    return st;
}

}  // namespace dtwlb

using namespace dtwlb;

#define CHECK_ARG(cond, ...)                      \
    do {                                          \
        if (!(cond)) {                            \
            set_error(DTWLB_EINVAL, __VA_ARGS__); \
            return DTWLB_EINVAL;                  \
        }                                         \
    } while (0)

static int check_p(int p) {
    if (p != 1 && p != 2) {
        set_error(DTWLB_EUNSUPPORTED, "p = %d unsupported (p must be 1 or 2)", p);
        return DTWLB_EUNSUPPORTED;
    }
    return DTWLB_OK;
}

extern "C" {

const char *dtwlb_last_error(void) { return g_err; }

void dtwlb_release_workspace(void) { release_workspace(); }

int lb_envelope(const float *x, int32_t n, int32_t w, float *U, float *L, int64_t count, void *stream) {
    g_err[0] = 0;
    CHECK_ARG(n >= 1, "lb_envelope: n = %d < 1", n);
    CHECK_ARG(w >= 0, "lb_envelope: w = %d < 0", w);
    CHECK_ARG(count >= 0, "lb_envelope: count < 0");
    if (count == 0) return DTWLB_OK;
    CHECK_ARG(x && U && L, "lb_envelope: NULL pointer");
    CHECK_ARG(U != L && (const float *)U != x && (const float *)L != x, "lb_envelope: outputs alias");
    DTWLB_TRY(require_device());
    return launch_envelope(x, n, w, U, L, count, as_stream(stream));
}

int lb_keogh(const float *q_env, const float *db, int64_t Q, int64_t N, int32_t n, int32_t p, float *out,
             void *stream) {
    g_err[0] = 0;
    CHECK_ARG(n >= 1, "lb_keogh: n = %d < 1", n);
    CHECK_ARG(Q >= 0 && N >= 0, "lb_keogh: negative size");
    DTWLB_TRY(check_p(p));
    if (Q == 0 || N == 0) return DTWLB_OK;
    CHECK_ARG(q_env && db && out, "lb_keogh: NULL pointer");
    DTWLB_TRY(require_device());
    if (keogh_stream_ok(Q, n, db))  // few queries: one streaming pass over the database (stream.cu)
        return launch_keogh_stream(q_env, q_env + Q * n, db, Q, N, n, p, true, out, N, as_stream(stream));
    return launch_keogh(q_env, q_env + Q * n, db, Q, N, n, p, true, out, N, as_stream(stream));
}

int lb_piecewise(const float *q_env, const float *db, int64_t Q, int64_t N, int32_t n, int32_t p, float *out,
                 void *stream) {
    g_err[0] = 0;
    CHECK_ARG(n >= 1, "lb_piecewise: n = %d < 1", n);
    CHECK_ARG(Q >= 0 && N >= 0, "lb_piecewise: negative size");
    DTWLB_TRY(check_p(p));
    if (Q == 0 || N == 0) return DTWLB_OK;
    CHECK_ARG(q_env && db && out, "lb_piecewise: NULL pointer");
    DTWLB_TRY(require_device());
    std::lock_guard<std::mutex> lock(api_mutex());
    cudaStream_t st = as_stream(stream);
    const int Dp = paa_pitch(n);
    float *xs, *qs;
    DTWLB_TRY(ws_get_bytes(8, sizeof(float) * 2 * N * Dp, (void **)&xs));
    DTWLB_TRY(ws_get_bytes(9, sizeof(float) * 2 * Q * Dp, (void **)&qs));
    DTWLB_TRY(launch_paa_sums(db, N, n, xs, xs + N * Dp, st));
    DTWLB_TRY(launch_paa_env_sums(q_env, q_env + Q * n, Q, n, qs, qs + Q * Dp, st));
    DTWLB_TRY(launch_paa_bound(qs, qs + Q * Dp, xs, xs + N * Dp, Q, N, n, p, true, out, N, st));
    DTWLB_CUDA(cudaStreamSynchronize(st));  // workspace reuse safety
    return DTWLB_OK;
}

int lb_piecewise_sym(const float *q, const float *q_env, const float *db, int64_t Q, int64_t N, int32_t n,
                     int32_t w, int32_t p, float *out, void *stream) {
    g_err[0] = 0;
    CHECK_ARG(n >= 1, "lb_piecewise_sym: n = %d < 1", n);
    CHECK_ARG(w >= 0, "lb_piecewise_sym: w = %d < 0", w);
    CHECK_ARG(Q >= 0 && N >= 0, "lb_piecewise_sym: negative size");
    DTWLB_TRY(check_p(p));
    if (Q == 0 || N == 0) return DTWLB_OK;
    CHECK_ARG(q && q_env && db && out, "lb_piecewise_sym: NULL pointer");
    DTWLB_TRY(require_device());
    std::lock_guard<std::mutex> lock(api_mutex());
    cudaStream_t st = as_stream(stream);
    const int Dp = paa_pitch(n);
    w = std::min(w, n - 1);
    float *xs, *qs, *dbenv;
    DTWLB_TRY(ws_get_bytes(8, sizeof(float) * 4 * N * Dp, (void **)&xs));
    DTWLB_TRY(ws_get_bytes(9, sizeof(float) * 4 * Q * Dp, (void **)&qs));
    DTWLB_TRY(ws_get_bytes(3, sizeof(float) * 2 * N * n, (void **)&dbenv));
    // forward operands: candidate sums, query envelope boxes (midpoint-radius form)
    DTWLB_TRY(launch_paa_mid(db, db, N, n, xs, xs + N * Dp, false, st));
    DTWLB_TRY(launch_paa_mid(q_env + Q * n, q_env, Q, n, qs, qs + Q * Dp, true, st));
    // reverse operands: candidate envelope boxes, query sums
    DTWLB_TRY(launch_envelope(db, n, w, dbenv, dbenv + N * n, N, st));
    DTWLB_TRY(launch_paa_mid(dbenv + N * n, dbenv, N, n, xs + 2 * N * Dp, xs + 3 * N * Dp, true, st));
    DTWLB_TRY(launch_paa_mid(q, q, Q, n, qs + 2 * Q * Dp, qs + 3 * Q * Dp, false, st));
    // both terms, max-combined, in one pass (the kernel nn_search's gate runs)
    DTWLB_TRY(launch_paa_bound_sym(qs, qs + Q * Dp, qs + 2 * Q * Dp, qs + 3 * Q * Dp, xs, xs + N * Dp, xs + 2 * N * Dp,
                                   xs + 3 * N * Dp, Q, N, n, p, true, out, N, st));
    DTWLB_CUDA(cudaStreamSynchronize(st));  // workspace reuse safety
    return DTWLB_OK;
}

int lb_improved(const float *q, const float *q_env, const float *db, int64_t Q, int64_t N, int32_t n,
                int32_t w, int32_t p, float *out, void *stream) {
    g_err[0] = 0;
    CHECK_ARG(n >= 1, "lb_improved: n = %d < 1", n);
    CHECK_ARG(w >= 0, "lb_improved: w = %d < 0", w);
    CHECK_ARG(Q >= 0 && N >= 0, "lb_improved: negative size");
    DTWLB_TRY(check_p(p));
    if (Q == 0 || N == 0) return DTWLB_OK;
    CHECK_ARG(q && q_env && db && out, "lb_improved: NULL pointer");
    DTWLB_TRY(require_device());
    const int epl = improved_epl(n);
    std::lock_guard<std::mutex> lock(api_mutex());
    cudaStream_t st = as_stream(stream);
    if (epl == 0) {  // n > 1024: the generic warp-per-pair kernel (same closed form)
        const int64_t ldb = N;
        float *beta1, *env, *dbenv;
        DTWLB_TRY(ws_get_bytes(0, sizeof(float) * Q * ldb, (void **)&beta1));
        DTWLB_TRY(ws_get_bytes(1, sizeof(float) * 3 * Q * n, (void **)&env));
        DTWLB_TRY(ws_get_bytes(3, sizeof(float) * 2 * N * n, (void **)&dbenv));
        const float *U = q_env, *L = q_env + Q * n;
        float *LU = env, *UL = env + Q * n, *scr = env + 2 * Q * n;
        DTWLB_TRY(launch_keogh(U, L, db, Q, N, n, p, false, beta1, ldb, st));
        DTWLB_TRY(launch_envelope(L, n, w, LU, scr, Q, st));
        DTWLB_TRY(launch_envelope(U, n, w, scr, UL, Q, st));
        DTWLB_TRY(launch_envelope(db, n, w, dbenv, dbenv + N * n, N, st));
        DTWLB_TRY(launch_improved_generic(q, LU, UL, dbenv, dbenv + N * n, beta1, ldb, Q, N, n, p, out, N, st));
        DTWLB_CUDA(cudaStreamSynchronize(st));  // workspace reuse safety
        return DTWLB_OK;
    }
    const int npadE = 32 * epl;
    const int64_t ldb = (N + 7) / 8 * 8;  // 16-byte rows of the fp16 gate block
    float *beta1, *env, *qpad, *dbenv;
    DTWLB_TRY(ws_get_bytes(0, sizeof(float) * Q * ldb, (void **)&beta1));
    DTWLB_TRY(ws_get_bytes(1, sizeof(float) * 3 * Q * n, (void **)&env));
    DTWLB_TRY(ws_get_bytes(2, sizeof(float) * 3 * Q * npadE, (void **)&qpad));
    DTWLB_TRY(ws_get_bytes(3, sizeof(float) * 2 * N * n, (void **)&dbenv));
    void *imp_scratch;
    DTWLB_TRY(ws_get_bytes(6, improved_scratch_bytes(Q, N), &imp_scratch));
    const float *U = q_env, *L = q_env + Q * n;
    float *LU = env, *UL = env + Q * n, *scr = env + 2 * Q * n;
    DTWLB_TRY(launch_keogh(U, L, db, Q, N, n, p, false, beta1, ldb, st));
    DTWLB_TRY(launch_envelope(L, n, w, LU, scr, Q, st));
    DTWLB_TRY(launch_envelope(U, n, w, scr, UL, Q, st));
    DTWLB_TRY(launch_envelope(db, n, w, dbenv, dbenv + N * n, N, st));
    // padded query-side arrays (host loop of copies: Q*n is small next to Q*N)
    DTWLB_CUDA(cudaMemsetAsync(qpad, 0, sizeof(float) * 3 * Q * npadE, st));
    DTWLB_CUDA(cudaMemcpy2DAsync(qpad, npadE * 4, q, n * 4, n * 4, Q, cudaMemcpyDeviceToDevice, st));
    DTWLB_CUDA(cudaMemcpy2DAsync(qpad + Q * npadE, npadE * 4, LU, n * 4, n * 4, Q, cudaMemcpyDeviceToDevice, st));
    DTWLB_CUDA(cudaMemcpy2DAsync(qpad + 2 * Q * npadE, npadE * 4, UL, n * 4, n * 4, Q, cudaMemcpyDeviceToDevice, st));
    ImprovedArgs a{};
    a.yq = qpad;
    a.LUq = qpad + Q * npadE;
    a.ULq = qpad + 2 * Q * npadE;
    a.Ux = dbenv;
    a.Lx = dbenv + N * n;
    a.gate = beta1;
    a.ldb = ldb;
    a.Qb = Q;
    a.N = N;
    a.n = n;
    a.npadE = npadE;
    a.dense = out;
    a.ldd = N;
    improved_scratch_bind(a, imp_scratch);
    DTWLB_TRY(launch_improved(a, p, false, true, st));
    DTWLB_CUDA(cudaStreamSynchronize(st));  // workspace reuse safety
    return DTWLB_OK;
}

int dtw_band(const float *x, const float *y, int32_t n, int32_t w, int32_t p, float *out, int64_t count,
             void *stream) {
    g_err[0] = 0;
    CHECK_ARG(n >= 1, "dtw_band: n = %d < 1", n);
    CHECK_ARG(w >= 0, "dtw_band: w = %d < 0", w);
    CHECK_ARG(count >= 0, "dtw_band: count < 0");
    CHECK_ARG(count <= 0x7fffffffLL, "dtw_band: count = %lld > 2^31 - 1 (split the call)", (long long)count);
    if (p != 0 && p != 4) DTWLB_TRY(check_p(p));  // p = 0 encodes DTW_inf; p = 4: DTW_4
                                                  // (Appendix C); both dtw_band only
    if (count == 0) return DTWLB_OK;
    CHECK_ARG(x && y && out, "dtw_band: NULL pointer");
    DTWLB_TRY(require_device());
    std::lock_guard<std::mutex> lock(api_mutex());
    cudaStream_t st = as_stream(stream);
    w = w > n - 1 ? n - 1 : w;
    DtwArgs a{};
    a.db = x;
    a.Ndb = count;
    a.n = n;
    a.w = w;
    a.total = count;
    a.res = out;
    int wS = 0;
    const int wide = w > 64 ? dtw_wide_plan(n, w, &wS) : 0;
    if (wide) {  // four lanes per pair, band (or the full row) in registers (dtw_wide.cu)
        int padL = 0;
        const int LPW = dtw_wide_padded(n, w, wS, &padL);
        float *yp;
        DTWLB_TRY(ws_get_bytes(5, sizeof(float) * count * LPW, (void **)&yp));
        DTWLB_TRY(launch_build_ywide(y, count, n, yp, LPW, padL, st));
        unsigned *queue;
        DTWLB_TRY(ws_get_bytes(7, 64, (void **)&queue));
        a.queue = queue;
        DTWLB_TRY(launch_dtw_wide(a, yp, LPW, padL, p, false, st));
    } else if (w > 64) {
        float *scratch = nullptr;
        if (dtw_generic_needs_scratch(w))
            DTWLB_TRY(ws_get_bytes(4, sizeof(float) * count * (2 * w + 2), (void **)&scratch));
        DTWLB_TRY(launch_dtw_generic(a, y, scratch, p, false, st));
    } else {
        const int LP = dtw_padded_len(n);
        float *ysh;
        DTWLB_TRY(ws_get_bytes(5, sizeof(float) * 4 * count * LP, (void **)&ysh));
        DTWLB_TRY(launch_build_ysh(y, count, n, ysh, LP, st));
        unsigned *queue;
        DTWLB_TRY(ws_get_bytes(7, 64, (void **)&queue));
        a.ysh = ysh;
        a.ysh_stride_s = count * LP;
        a.LP = LP;
        a.queue = queue;
        DTWLB_TRY(launch_dtw(a, p, false, st));
    }
    DTWLB_CUDA(cudaStreamSynchronize(st));
    return DTWLB_OK;
}

int nn_search(const float *queries, int64_t Q, const float *db, int64_t N, int32_t n, int32_t w, int32_t p,
              int32_t k, int64_t *out_idx, float *out_dist, const nn_opts *opts, nn_stats *stats, void *stream) {
    g_err[0] = 0;
    if (stats) memset(stats, 0, sizeof(*stats));
    CHECK_ARG(n >= 1, "nn_search: n = %d < 1", n);
    CHECK_ARG(w >= 0, "nn_search: w = %d < 0", w);
    CHECK_ARG(k >= 1, "nn_search: k = %d < 1", k);
    CHECK_ARG(Q >= 0, "nn_search: Q < 0");
    CHECK_ARG(N >= 1, "nn_search: empty database (N = %lld)", (long long)N);
    CHECK_ARG(k <= N, "nn_search: k = %d > N = %lld", k, (long long)N);
    CHECK_ARG(N <= 0xffffffffLL, "nn_search: N above 2^32 per shard");
    DTWLB_TRY(check_p(p));
    if (k > DTWLB_MAX_K) {
        set_error(DTWLB_EUNSUPPORTED, "nn_search: k = %d > DTWLB_MAX_K = %d", k, DTWLB_MAX_K);
        return DTWLB_EUNSUPPORTED;
    }
    if (Q == 0) return DTWLB_OK;
    CHECK_ARG(queries && db && out_idx && out_dist, "nn_search: NULL pointer");
    {   // outputs may not overlap an input or each other (byte ranges)
        auto ov = [](const void *a, size_t na, const void *b, size_t nb) {
            const char *x = static_cast<const char *>(a), *y = static_cast<const char *>(b);
            return x < y + nb && y < x + na;
        };
        const size_t bq = sizeof(float) * (size_t)Q * n, bd = sizeof(float) * (size_t)N * n;
        const size_t bi = sizeof(int64_t) * (size_t)Q * k, bo = sizeof(float) * (size_t)Q * k;
        CHECK_ARG(!ov(out_idx, bi, queries, bq) && !ov(out_idx, bi, db, bd) && !ov(out_dist, bo, queries, bq) &&
                      !ov(out_dist, bo, db, bd) && !ov(out_idx, bi, out_dist, bo),
                  "nn_search: an output aliases an input or the other output");
    }
    CHECK_ARG(opts == nullptr || opts->eps >= 0.f, "nn_search: eps < 0");
    DTWLB_TRY(require_device());
    return nn_search_impl(queries, Q, db, N, n, w, p, k, out_idx, out_dist, opts, stats, as_stream(stream));
}

int nn_merge(const int64_t *in_idx, const float *in_dist, int32_t G, int64_t Q, int32_t k, int64_t *out_idx,
             float *out_dist, void *stream) {
    g_err[0] = 0;
    CHECK_ARG(G >= 1 && G <= 64, "nn_merge: G = %d outside [1, 64]", G);
    CHECK_ARG(Q >= 0 && k >= 1, "nn_merge: bad sizes");
    if (Q == 0) return DTWLB_OK;
    CHECK_ARG(in_idx && in_dist && out_idx && out_dist, "nn_merge: NULL pointer");
    DTWLB_TRY(require_device());
    return nn_merge_impl(in_idx, in_dist, G, Q, k, out_idx, out_dist, as_stream(stream));
}

}  // extern "C"
