// Precision check of the fp16 hi/lo split product on the legacy tensor path (mma.sync m16n8k16,
// fp32 accumulate) against fp64, for the leaf binned product S[p][a'] = sum_y b_p(y) Q'(y,a'):
// 16 beliefs x 8 columns over K cells, beliefs scaled by 2^14 before the split.
//   mode 0: C accumulated in the MMA across all chunks
//   mode 1: per-chunk MMA from zero, fp32 FADD into running sums
//   mode 2: fp32 scalar FMA (the current k_hist arithmetic), sequential
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

constexpr int K = 4096;
constexpr float SC = 16384.f;

__device__ __forceinline__ void split(float x, __half &hi, __half &lo) {
    hi = __float2half_rn(x);
    lo = __float2half_rn(x - __half2float(hi));
}
__device__ __forceinline__ unsigned pack(__half a, __half b) {
    return (unsigned)__half_as_ushort(a) | ((unsigned)__half_as_ushort(b) << 16);
}
__device__ __forceinline__ void mma(float (&c)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__global__ void kern(const float *b, const float *q, float *out, int mode) {   // b [16][K], q [K][8]
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    float c[4] = {0, 0, 0, 0}, s[4] = {0, 0, 0, 0};
    for (int k0 = 0; k0 < K; k0 += 16) {
        unsigned ah[4], al[4], bh[2], bl[2];
        const int rows[4] = {g, g + 8, g, g + 8}, cols[4] = {2 * t, 2 * t, 2 * t + 8, 2 * t + 8};
        for (int r = 0; r < 4; ++r) {
            __half h0, l0, h1, l1;
            split(b[rows[r] * K + k0 + cols[r]] * SC, h0, l0);
            split(b[rows[r] * K + k0 + cols[r] + 1] * SC, h1, l1);
            ah[r] = pack(h0, h1);
            al[r] = pack(l0, l1);
        }
        for (int r = 0; r < 2; ++r) {
            __half h0, l0, h1, l1;
            split(q[(k0 + 2 * t + 8 * r) * 8 + g], h0, l0);
            split(q[(k0 + 2 * t + 8 * r + 1) * 8 + g], h1, l1);
            bh[r] = pack(h0, h1);
            bl[r] = pack(l0, l1);
        }
        if (mode == 0) {
            mma(c, ah, bh[0], bh[1]);
            mma(c, ah, bl[0], bl[1]);
            mma(c, al, bh[0], bh[1]);
        } else {
            float d[4] = {0, 0, 0, 0};
            mma(d, ah, bh[0], bh[1]);
            mma(d, ah, bl[0], bl[1]);
            mma(d, al, bh[0], bh[1]);
            for (int i = 0; i < 4; ++i) s[i] += d[i];
        }
    }
    const float *r = mode == 0 ? c : s;
    out[g * 8 + 2 * t] = r[0] / SC;
    out[g * 8 + 2 * t + 1] = r[1] / SC;
    out[(g + 8) * 8 + 2 * t] = r[2] / SC;
    out[(g + 8) * 8 + 2 * t + 1] = r[3] / SC;
}

int main() {
    static float hb[16 * K], hq[K * 8];
    srand(7);
    auto urand = [] { return (rand() + 0.5) / (RAND_MAX + 1.0); };
    for (int dist = 0; dist < 3; ++dist) {
        // 0: near-uniform belief (~1/K), 1: localised (exponential decay, 1e-30..1), 2: sparse mix
        for (int p = 0; p < 16; ++p) {
            double tot = 0;
            for (int y = 0; y < K; ++y) {
                double v = dist == 0 ? urand() : dist == 1 ? exp(-40.0 * urand() * urand() * (1 + p)) * (urand() < 0.02 ? 1 : 1e-6)
                                                  : (urand() < 0.1 ? urand() : 0.0);
                hb[p * K + y] = (float)v;
                tot += (float)v;
            }
            for (int y = 0; y < K; ++y) hb[p * K + y] = (float)(hb[p * K + y] / tot);
        }
        for (int i = 0; i < K * 8; ++i) hq[i] = (float)(20.0 * urand() - 10.0);
        float *db, *dq, *dout;
        cudaMalloc(&db, sizeof hb); cudaMalloc(&dq, sizeof hq); cudaMalloc(&dout, 128 * 4);
        cudaMemcpy(db, hb, sizeof hb, cudaMemcpyHostToDevice);
        cudaMemcpy(dq, hq, sizeof hq, cudaMemcpyHostToDevice);
        for (int mode = 0; mode < 3; ++mode) {
            float res[128];
            if (mode < 2) {
                kern<<<1, 32>>>(db, dq, dout, mode);
                cudaMemcpy(res, dout, sizeof res, cudaMemcpyDeviceToHost);
            } else {
                for (int p = 0; p < 16; ++p)
                    for (int a = 0; a < 8; ++a) {
                        float acc = 0.f;
                        for (int y = 0; y < K; ++y) acc = fmaf(hb[p * K + y], hq[y * 8 + a], acc);
                        res[p * 8 + a] = acc;
                    }
            }
            double worst_abs = 0, worst_rel = 0;
            for (int p = 0; p < 16; ++p)
                for (int a = 0; a < 8; ++a) {
                    double ref = 0, mag = 0;
                    for (int y = 0; y < K; ++y) {
                        ref += (double)hb[p * K + y] * hq[y * 8 + a];
                        mag += fabs((double)hb[p * K + y] * hq[y * 8 + a]);
                    }
                    const double e = fabs(res[p * 8 + a] - ref);
                    worst_abs = fmax(worst_abs, e);
                    worst_rel = fmax(worst_rel, e / mag);
                }
            printf("{\"dist\": %d, \"mode\": %d, \"K\": %d, \"max_abs_err\": %.3e, \"max_err_over_sum_abs\": %.3e}\n", dist, mode, K,
                   worst_abs, worst_rel);
        }
        cudaFree(db); cudaFree(dq); cudaFree(dout);
    }
    return 0;
}
