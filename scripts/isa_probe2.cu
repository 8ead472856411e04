// isa_probe2.cu -- per-SM throughput of the LB element under different SASS mixes.
// Inline PTX pins the instruction forms.  Each thread runs 8 independent element
// chains; all inputs come from registers that the loop rotates so nothing is
// loop-invariant.  Reports elements per SM clock (clock64 per CTA, 4 CTAs/SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o isa_probe2 isa_probe2.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 65536

__device__ __forceinline__ float fsub(float a, float b) { float d; asm volatile("sub.rn.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b)); return d; }
__device__ __forceinline__ float fmax3(float a, float b, float c) { float d; asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ __forceinline__ float fmax2(float a, float b) { float d; asm volatile("max.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b)); return d; }
__device__ __forceinline__ float fmin2(float a, float b) { float d; asm volatile("min.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b)); return d; }
__device__ __forceinline__ float ffma(float a, float b, float c) { float d; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ __forceinline__ float fadd(float a, float b) { float d; asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b)); return d; }

template <int V>
__global__ void probe(float *out, const float *in, long long *cycles) {
    float x[8], u[8], l[8], acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        x[j] = in[(threadIdx.x + j) & 63];
        u[j] = in[(threadIdx.x + 3 * j + 1) & 63] + 1.f;
        l[j] = in[(threadIdx.x + 5 * j + 2) & 63] - 1.f;
        acc[j] = 0.f;
    }
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float xv = x[j], uv = u[j], lv = l[(j + 3) & 7];
            if constexpr (V == 0) {  // FADD, FADD, FMNMX3, FFMA
                float d = fmax3(fsub(xv, uv), fsub(lv, xv), 0.f);
                acc[j] = ffma(d, d, acc[j]);
            } else if constexpr (V == 1) {  // clamp: FMNMX, FMNMX, FADD, FFMA
                float h = fmin2(fmax2(xv, lv), uv);
                float d = fsub(xv, h);
                acc[j] = ffma(d, d, acc[j]);
            } else if constexpr (V == 2) {  // mix: even j form 0, odd j form 1
                if (j & 1) {
                    float h = fmin2(fmax2(xv, lv), uv);
                    float d = fsub(xv, h);
                    acc[j] = ffma(d, d, acc[j]);
                } else {
                    float d = fmax3(fsub(xv, uv), fsub(lv, xv), 0.f);
                    acc[j] = ffma(d, d, acc[j]);
                }
            } else if constexpr (V == 3) {  // p=1 clamp: FMNMX, FMNMX, FADD, FADD(abs)
                float h = fmin2(fmax2(xv, lv), uv);
                acc[j] = fadd(acc[j], fabsf(fsub(xv, h)));
            } else if constexpr (V == 4) {  // p=1 form 0: FADD, FADD, FMNMX3, FADD
                acc[j] = fadd(acc[j], fmax3(fsub(xv, uv), fsub(lv, xv), 0.f));
            }
        }
        // rotate the envelope registers (static moves) so nothing is loop-invariant
        const float t = u[0];
#pragma unroll
        for (int j = 0; j < 7; ++j) u[j] = u[j + 1];
        u[7] = t;
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += acc[j] + x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int V>
void run(const char *name) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int ctas = sms * 4, nt = 256;
    float *out, *in;
    long long *cyc;
    cudaMalloc(&out, sizeof(float) * ctas * nt);
    cudaMalloc(&in, sizeof(float) * 64);
    cudaMemset(in, 0, sizeof(float) * 64);
    cudaMalloc(&cyc, sizeof(long long) * ctas);
    probe<V><<<ctas, nt>>>(out, in, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<V><<<ctas, nt>>>(out, in, cyc);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[4096];
    cudaMemcpy(h, cyc, sizeof(long long) * ctas, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < ctas; ++i) avg += h[i];
    avg /= ctas;
    const double elems = (double)ctas * nt * ITERS * 8;
    printf("%-44s %6.2f elem/clk/SM (clock64)   %8.3f Telem/s (events, %.3f ms)\n", name,
           4.0 * nt * ITERS * 8 / avg, elems / (ms * 1e-3) / 1e12, ms);
}

int main() {
    run<0>("FADD,FADD,FMNMX3,FFMA (p=2 current)");
    run<1>("FMNMX,FMNMX,FADD,FFMA (p=2 clamp)");
    run<2>("mix of both (p=2)");
    run<3>("FMNMX,FMNMX,FADD,FADD|abs| (p=1 clamp)");
    run<4>("FADD,FADD,FMNMX3,FADD (p=1 current)");
    return 0;
}
