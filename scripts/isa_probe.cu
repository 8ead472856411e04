// isa_probe.cu -- measured issue/pipe rates of the SASS ops the bound and DTW
// kernels are built from (sm_100a).  Standalone:  nvcc -arch=sm_100a -O3 -o isa_probe isa_probe.cu
// Each variant runs 8 independent dependency chains per thread, 148*4 CTAs x 256 threads,
// and reports warp-instructions per SM clock and lane-ops per SM clock.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

template <int OP>
__global__ void probe(float *out, float s0, float s1, long long *cycles) {
    float a[8], b[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { a[j] = s0 + j + threadIdx.x * 1e-7f; b[j] = s1 - j; }
    float2 p[8], q2[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { p[j] = make_float2(a[j], b[j]); q2[j] = make_float2(b[j], a[j]); }
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if constexpr (OP == 0) a[j] = a[j] + b[j];                                 // FADD
            if constexpr (OP == 1) a[j] = fmaf(a[j], b[j], s1);                        // FFMA (3 reg)
            if constexpr (OP == 2) a[j] = fmaxf(a[j], b[j]);                            // FMNMX
            if constexpr (OP == 3) a[j] = fmaxf(fmaxf(a[j], b[j]), b[(j + 1) & 7]);     // FMNMX3
            if constexpr (OP == 4) p[j] = __fadd2_rn(p[j], q2[j]);                      // FADD2
            if constexpr (OP == 5) p[j] = __ffma2_rn(p[j], q2[j], q2[(j + 1) & 7]);     // FFMA2
            if constexpr (OP == 6) {  // LB element: FADD, FADD, FMNMX3, FFMA
                float d = fmaxf(fmaxf(b[j] - a[j], a[j] - s1), 0.f);
                a[j] = fmaf(d, d, a[j]);
            }
            if constexpr (OP == 7) {  // packed LB element pair: FADD2, FADD2, 2x FMNMX3, FFMA2
                float2 u = __fadd2_rn(q2[j], make_float2(-p[j].x, -p[j].y));
                float2 l = __fadd2_rn(p[j], make_float2(-s1, -s0));
                float2 d = make_float2(fmaxf(fmaxf(u.x, l.x), 0.f), fmaxf(fmaxf(u.y, l.y), 0.f));
                p[j] = __ffma2_rn(d, d, p[j]);
            }
            if constexpr (OP == 9) {  // FMNMX pair that cannot be folded: max / min swap
                const float t = fmaxf(a[j], b[j]);
                b[j] = fminf(a[j], b[j]);
                a[j] = t + 0.f;
            }
            if constexpr (OP == 10) {  // LB_Improved element: FMNMX, FMNMX, FADD, FADD, FMNMX3, FFMA
                const float d = fmaxf(fmaxf(a[j] - fmaxf(b[j], s0), fminf(b[(j + 1) & 7], s1) - a[j]), 0.f);
                a[j] = fmaf(d, d, a[j]);
            }
            if constexpr (OP == 11) {  // gate / tile-kernel element pair: FADD2, FADD2, 2x FMNMX3, 2x FFMA
                float2 u = __fadd2_rd(q2[j], make_float2(-p[j].x, -p[j].y));
                float2 l = __fadd2_rd(p[j], make_float2(-s1, -s0));
                const float d0 = fmaxf(fmaxf(u.x, l.x), 0.f), d1 = fmaxf(fmaxf(u.y, l.y), 0.f);
                p[j].x = __fmaf_rd(d1, d1, __fmaf_rd(d0, d0, p[j].x));
            }
            if constexpr (OP == 12) {  // midpoint-form gate element: FADD.RZ, FADD.RM |.|, FADD |.|, FFMA.RM
                const float t1 = __fsub_rz(a[j], b[j]);
                const float t2 = __fsub_rd(fabsf(t1), s1);
                const float t3 = t2 + fabsf(t2);
                b[j] = __fmaf_rd(t3, t3, b[j]);
            }
            if constexpr (OP == 8) {  // DTW cell: FADD, FMNMX3, FFMA
                float t = s0 - b[j];
                a[j] = fmaf(t, t, fminf(fminf(a[j], b[(j + 1) & 7]), a[(j + 7) & 7]));
            }
        }
    }
    long long t1 = clock64();
    float acc = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += a[j] + b[j] + p[j].x + p[j].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char *name, double ops_per_iter_per_thread, double lane_ops_per_iter) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int ctas = sms * 4, nt = 256;
    float *out;
    long long *cyc;
    cudaMalloc(&out, sizeof(float) * ctas * nt);
    cudaMalloc(&cyc, sizeof(long long) * ctas);
    probe<OP><<<ctas, nt>>>(out, 1.0f, 2.0f, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<OP><<<ctas, nt>>>(out, 1.0f, 2.0f, cyc);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    long long h[4096];
    cudaMemcpy(h, cyc, sizeof(long long) * ctas, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < ctas; ++i) avg += h[i];
    avg /= ctas;
    // 4 CTAs resident per SM (256 threads each): per-SM warp-instr per clock
    const double warps_per_sm = 4 * nt / 32.0;
    const double winst = warps_per_sm * ITERS * ops_per_iter_per_thread / avg;
    const double lops = warps_per_sm * 32 * ITERS * lane_ops_per_iter / avg;
    // event-timed: whole grid's warp-instructions / (elapsed x SMs x clock) -- independent of
    // what clock64() counts (its per-CTA counts gave > 4 warp-inst/clk/SM, i.e. not SM clocks)
    const double tot_w = (double)ctas * (nt / 32) * ITERS * ops_per_iter_per_thread;
    const double ev_w = tot_w / (ms * 1e-3 * sms * khz * 1e3);
    printf("%-40s %6.2f warp-inst/clk/SM  %7.1f lane-ops/clk/SM (clock64)   event-timed: %5.2f warp-inst/clk/SM %7.1f lane-ops/clk/SM  %.3f ms @ %d MHz\n",
           name, winst, lops, ev_w, ev_w * 32 * lane_ops_per_iter / ops_per_iter_per_thread, ms, khz / 1000);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run<0>("FADD", 8, 8);
    run<1>("FFMA (3-reg)", 8, 8);
    run<2>("FMNMX", 8, 8);
    run<3>("FMNMX3", 8, 8);
    run<4>("FADD2 (f32x2)", 8, 16);
    run<5>("FFMA2 (f32x2)", 8, 16);
    run<6>("LB element (4 ops) [elements]", 32, 8);
    run<7>("packed LB pair (5 ops) [elements]", 40, 16);
    run<8>("DTW cell (3 ops) [cells]", 24, 8);
    run<9>("FMNMX (max/min swap, 2 ops)", 16, 16);
    run<11>("gate element pair (FADD2 x2, FMNMX3 x2, FFMA x2) [elements]", 48, 16);
    run<10>("LB_Improved element (6 ops) [elements]", 48, 8);
    run<12>("midpoint gate element (FADD.RZ, FADD.RM, FADD, FFMA.RM) [elements]", 32, 8);
    return 0;
}
