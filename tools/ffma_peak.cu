// Microbenchmark: FP32 FFMA throughput on this GPU (register-operand form, as in k_hist's
// accumulation acc += h * q, and the FADD rate).  Used to derive the ALU roofline peak.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk2(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}

// FFMA2 (fma.rn.f32x2, sm_100a): acc2 += broadcast(x) * (y_lo, y_hi), the k_hist pattern
__global__ void k2(float *out, float x0, float y0, int iters) {
    unsigned long long a[16], y2[4];
    float x[4];
    for (int i = 0; i < 4; ++i) { x[i] = x0 + i * threadIdx.x; y2[i] = pk2(y0 - i, y0 + i); }
    for (int i = 0; i < 16; ++i) a[i] = pk2((float)i, (float)(i + 1));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
            asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a[i]) : "l"(pk2(x[i & 3], x[i & 3])), "l"(y2[i >> 2]));
#pragma unroll
        for (int i = 0; i < 4; ++i) { x[i] += 1e-7f; }
    }
    float s = 0;
    for (int i = 0; i < 16; ++i) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[i]));
        s += lo + hi;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
__global__ void k(float *out, float x0, float y0, int iters) {
    float a[16], x[4], y[4];
    for (int i = 0; i < 4; ++i) { x[i] = x0 + i * threadIdx.x; y[i] = y0 - i; }
    for (int i = 0; i < 16; ++i) a[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (MODE == 0) a[i] = fmaf(x[i & 3], y[i >> 2], a[i]);       // 3-register FFMA
            else if (MODE == 1) a[i] = fmaf(a[i], 1.0001f, 0.5f);         // immediate form
            else a[i] = a[i] + x[i & 3];                                  // FADD
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) { x[i] += 1e-7f; }
    }
    float s = 0;
    for (int i = 0; i < 16; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float *out; cudaMalloc(&out, sizeof(float) * sms * 8 * 512);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000, blocks = sms * 4, threads = 512;
    const char *names[3] = {"ffma_3reg", "ffma_imm", "fadd"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<blocks, threads>>>(out, 1.f, 2.f, iters);
            if (mode == 1) k<1><<<blocks, threads>>>(out, 1.f, 2.f, iters);
            if (mode == 2) k<2><<<blocks, threads>>>(out, 1.f, 2.f, iters);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double ops = (double)blocks * threads * iters * 16;
            if (rep) printf("{\"op\": \"%s\", \"Tops\": %.3f, \"ms\": %.3f, \"per_sm_per_cycle_at_max_clk\": %.2f, \"sms\": %d, \"max_clock_mhz\": %d}\n",
                            names[mode], ops / ms / 1e9, ms, ops / (ms * 1e-3) / sms / (clk * 1e3), sms, clk / 1000);
        }
    }
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k2<<<blocks, threads>>>(out, 1.f, 2.f, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)blocks * threads * iters * 16 * 2;   // two FMAs per FFMA2
        if (rep) printf("{\"op\": \"ffma2_bcast\", \"Tfma_per_s\": %.3f, \"ms\": %.3f, \"fma_per_sm_per_cycle_at_max_clk\": %.2f}\n",
                        ops / ms / 1e9, ms, ops / (ms * 1e-3) / sms / (clk * 1e3));
    }
    return 0;
}
