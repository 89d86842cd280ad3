// Microbenchmark: FP64 DMMA (mma.sync m8n8k4 f64) vs DFMA throughput on one B200, and mixed.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void k(double* out, int iters, double a, double b) {
    double acc[8][2];
    double f[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = threadIdx.x;
#pragma unroll
    for (int i = 0; i < 16; ++i) f[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0 || MODE == 2) {
#pragma unroll
            for (int i = 0; i < 8; ++i) dmma(acc[i], a, b);
        }
        if (MODE == 1 || MODE == 2) {
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = fma(f[i], a, b);
#pragma unroll
            for (int i = 0; i < 16; ++i) f[i] = fma(f[i], a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
#pragma unroll
    for (int i = 0; i < 16; ++i) s += f[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// Fragment-layout check for K1's tensor-core path: a0 = A[lane>>2][lane&3],
// b0 = B[lane&3][lane>>2], {d0, d1} = D[lane>>2][2 (lane&3) + {0, 1}].
__global__ void layout_check(double* out) {
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    const double a = g * 10.0 + t + 1.0, b = t * 7.0 - g + 3.0;
    double d[2] = {0.0, 0.0};
    dmma(d, a, b);
    out[g * 8 + 2 * t] = d[0];
    out[g * 8 + 2 * t + 1] = d[1];
}
int main() {
    {
        double* o;
        cudaMalloc(&o, 64 * 8);
        layout_check<<<1, 32>>>(o);
        double h[64];
        cudaMemcpy(h, o, 64 * 8, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int m = 0; m < 8; ++m)
            for (int n = 0; n < 8; ++n) {
                double ref = 0;
                for (int k = 0; k < 4; ++k) ref += (m * 10.0 + k + 1.0) * (k * 7.0 - n + 3.0);
                bad += h[m * 8 + n] != ref;
            }
        printf("dmma fragment layout check: %s (%d mismatches)\n", bad ? "FAIL" : "ok", bad);
    }
    double* out;
    cudaMalloc(&out, 148 * 8 * 1024 * 8);
    const int iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int warps : {4, 8, 16, 32}) {
        for (int mode = 0; mode < 3; ++mode) {
            auto run = [&] {
                if (mode == 0) k<0><<<148, 32 * warps>>>(out, iters, 1.0000001, 1e-9);
                if (mode == 1) k<1><<<148, 32 * warps>>>(out, iters, 1.0000001, 1e-9);
                if (mode == 2) k<2><<<148, 32 * warps>>>(out, iters, 1.0000001, 1e-9);
            };
            run();
            cudaEventRecord(e0);
            run();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double nw = 148.0 * warps * iters;
            const double dmma_fl = (mode != 1) ? nw * 8 * 512 : 0;       // 8 mma x 8x8x4x2 flops
            const double dfma_fl = (mode != 0) ? nw * 32 * 32 * 2 : 0;   // 32 fma x 32 lanes x 2
            printf("warps/SM %2d mode %s: %.3f ms  DMMA %.1f TF  DFMA %.1f TF  total %.1f TF\n", warps,
                   mode == 0 ? "dmma" : mode == 1 ? "dfma" : "mix ", ms, dmma_fl / ms / 1e9, dfma_fl / ms / 1e9,
                   (dmma_fl + dfma_fl) / ms / 1e9);
        }
    }
    return 0;
}
