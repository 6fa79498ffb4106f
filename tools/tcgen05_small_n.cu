// Microbenchmark: tcgen05.mma throughput at the small N of the leaf contraction (VERDICT r01
// item 6: "first measure the tcgen05 rate at the small N this contraction has").  The leaf's
// binned product is F[s][(parent, field)][a'] = sum over the class's cells of h * Q' -- as an MMA
// D[M = (parent, field)] [N = a'] += A[M][K = cells] B[K][N], with N = |A| = 8 (or 9 padded to
// 16).  One CTA per SM, one elected thread issues R back-to-back MMAs (cta_group::1, operands in
// shared memory, K-major, no swizzle; the operand values are irrelevant to the rate) into one
// TMEM accumulator, commits them to an mbarrier and waits; CUDA events time the launch.
// Compile: nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/tcgen05_small_n.cu -o /tmp/tc
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// instruction descriptor (cute/arch/mma_sm100_desc.hpp UMMA::InstrDescriptor): D fp32 (bits 4-5 = 1),
// A/B format (bits 7-9 / 10-12: 0 f16, 2 tf32), K-major A and B, N >> 3 at bit 17, M >> 4 at bit 24
__host__ __device__ constexpr uint32_t idesc(int fmt, int M, int N) {
    return (1u << 4) | ((uint32_t)fmt << 7) | ((uint32_t)fmt << 10) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}
// shared-memory matrix descriptor (UMMA::SmemDescriptor): start >> 4, LBO >> 4 at bit 16,
// SBO >> 4 at bit 32, version 1 at bit 46, no swizzle
__device__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

template <int FMT, int M, int N>
__global__ void __launch_bounds__(128, 1) k_mma(int reps, unsigned long long *cycles) {
    __shared__ __align__(128) uint8_t sa[M * 64];       // A: M x (K = 32 bytes of one MMA)
    __shared__ __align__(128) uint8_t sb[256 * 64];     // B: N x 32 bytes (N <= 256)
    __shared__ __align__(8) unsigned long long bar;
    __shared__ uint32_t s_tmem;
    const int t = threadIdx.x, warp = t >> 5;
    for (int i = t; i < M * 64 / 4; i += 128) reinterpret_cast<uint32_t *>(sa)[i] = 0x3c003c00u;
    for (int i = t; i < 256 * 64 / 4; i += 128) reinterpret_cast<uint32_t *>(sb)[i] = 0x3c003c00u;
    const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(&bar);
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    unsigned long long c0 = 0, c1 = 0;
    if (t == 0) {
        const uint64_t da = sdesc((uint32_t)__cvta_generic_to_shared(sa), 128, 256);
        const uint64_t db = sdesc((uint32_t)__cvta_generic_to_shared(sb), 128, 256);
        const uint32_t id = idesc(FMT, M, N);
        c0 = clock64();
        for (int r = 0; r < reps; ++r) {
            const uint32_t acc = r > 0 ? 1u : 0u;
            if constexpr (FMT == 2)
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                    " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(da), "l"(db),
                    "r"(id), "r"(acc));
            else
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                    " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(da), "l"(db),
                    "r"(id), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar_s)
                     : "memory");
        asm volatile(
            "{\n .reg .pred P1;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
            " @!P1 bra WAIT_%=;\n}\n" ::"r"(bar_s) : "memory");
        c1 = clock64();
        cycles[blockIdx.x] = c1 - c0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int FMT, int M, int N>
static void run(const char *name, int sms, int per_sm = 1) {
    unsigned long long *cyc;
    cudaMalloc(&cyc, sizeof(unsigned long long) * sms * 2);
    const int reps = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_mma<FMT, M, N><<<sms * per_sm, 128>>>(100, cyc);
    cudaEventRecord(e0);
    k_mma<FMT, M, N><<<sms * per_sm, 128>>>(reps, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h = 0;
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const int K = FMT == 2 ? 8 : 16;
    const double macs = (double)M * N * K;
    const cudaError_t err = cudaGetLastError();
    printf("{\"op\": \"%s\", \"M\": %d, \"N\": %d, \"K\": %d, \"ctas_per_sm\": %d, \"ms\": %.3f, \"cycles_per_mma_cta0\": %.2f, "
           "\"mma_per_sm_per_us\": %.1f, \"TFLOPs\": %.2f, \"err\": \"%s\"}\n",
           name, M, N, K, per_sm, ms, (double)h / reps, (double)reps * per_sm / (ms * 1e3),
           2.0 * macs * reps * sms * per_sm / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
    cudaFree(cyc);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0, 128, 8>("f16 M128 N8", sms);
    run<0, 128, 16>("f16 M128 N16", sms);
    run<0, 128, 64>("f16 M128 N64", sms);
    run<0, 128, 256>("f16 M128 N256", sms);
    run<0, 64, 8>("f16 M64 N8", sms);
    run<2, 128, 8>("tf32 M128 N8", sms);
    run<2, 128, 16>("tf32 M128 N16", sms);
    run<2, 128, 256>("tf32 M128 N256", sms);
    run<0, 128, 8>("f16 M128 N8, 2 CTAs per SM", sms, 2);
    run<2, 128, 8>("tf32 M128 N8, 2 CTAs per SM", sms, 2);
    return 0;
}
