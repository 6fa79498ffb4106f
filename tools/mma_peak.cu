// Microbenchmark: warp-level mma.sync (legacy HMMA path) throughput on this GPU, to decide
// whether the leaf binned product sum_y h_k(y) Q'(y,a') can run on it.
// Each warp issues independent m16n8k8 tf32 / m16n8k16 bf16 MMAs into 8 accumulators.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float *out, unsigned seed, int iters) {
    float c[8][4];
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 4; ++j) c[i][j] = 0.f;
    unsigned a[4], b[2];
    for (int j = 0; j < 4; ++j) a[j] = seed * (threadIdx.x + j) | 0x3f800000u;
    for (int j = 0; j < 2; ++j) b[j] = seed * (threadIdx.x + 7 * j) | 0x3f000000u;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0)
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                             : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
            else if (MODE == 1)
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                             : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
            else
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                             : "r"(a[0]), "r"(a[1]), "r"(b[0]));
        }
    }
    float s = 0;
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 4; ++j) s += c[i][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float *out; cudaMalloc(&out, sizeof(float) * sms * 8 * 512);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4000, blocks = sms * 4, threads = 256;
    const char *names[3] = {"mma_m16n8k8_tf32", "mma_m16n8k16_bf16", "mma_m16n8k4_tf32"};
    const double macs[3] = {16 * 8 * 8, 16 * 8 * 16, 16 * 8 * 4};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<blocks, threads>>>(out, 12345u, iters);
            if (mode == 1) k<1><<<blocks, threads>>>(out, 12345u, iters);
            if (mode == 2) k<2><<<blocks, threads>>>(out, 12345u, iters);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            const double nmma = (double)blocks * (threads / 32) * iters * 8;
            const double per = nmma / (ms * 1e-3) / sms / (clk * 1e3);
            if (rep) printf("{\"op\": \"%s\", \"ms\": %.3f, \"mma_per_sm_per_cycle_at_max_clk\": %.3f, \"mac_per_sm_per_cycle\": %.1f, \"TFLOPs\": %.1f}\n",
                            names[mode], ms, per, per * macs[mode], 2 * nmma * macs[mode] / (ms * 1e-3) / 1e12);
        }
    }
    return 0;
}
