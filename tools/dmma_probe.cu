// Does DMMA (mma.sync m8n8k4 f64) run on a pipe separate from DFMA on sm_100a?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int NF, int NM>
__global__ void k(double* out, int iters, double s) {
    double f[8], d0[4], d1[4];
    for (int i = 0; i < 8; ++i) f[i] = threadIdx.x * 1e-3 + i;
    for (int i = 0; i < 4; ++i) { d0[i] = i; d1[i] = i + 1; }
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < NF; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = fma(f[i], s, 1e-7);
#pragma unroll
        for (int r = 0; r < NM; ++r)
#pragma unroll
            for (int i = 0; i < 4; ++i) dmma(d0[i], d1[i], a, b);
    }
    double acc = 0;
    for (int i = 0; i < 8; ++i) acc += f[i];
    for (int i = 0; i < 4; ++i) acc += d0[i] + d1[i];
    if (acc == 12345.678) out[0] = acc;
}
template <int NF, int NM>
void run(const char* name, int threads) {
    double* o; cudaMalloc(&o, 8);
    int iters = 2000, blocks = 148 * 4;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<NF, NM><<<blocks, threads>>>(o, 10, 0.9999999);
    cudaEventRecord(e0);
    k<NF, NM><<<blocks, threads>>>(o, iters, 0.9999999);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double warps = (double)blocks * threads / 32;
    double dfma_warp_instr = warps * iters * NF * 8, dmma_instr = warps * iters * NM * 4;
    double tf_dfma = dfma_warp_instr * 32 * 2 / (ms * 1e-3) / 1e12;
    double tf_dmma = dmma_instr * 8 * 8 * 4 * 2 / (ms * 1e-3) / 1e12;
    printf("%-10s threads %4d: %.3f ms  DFMA %.1f TF  DMMA %.1f TF  total %.1f TF\n", name, threads, ms, tf_dfma, tf_dmma,
           tf_dfma + tf_dmma);
    cudaFree(o);
}
int main() {
    for (int t : {256, 512}) {
        run<4, 0>("dfma", t);
        run<0, 4>("dmma", t);
        run<4, 4>("both", t);
        run<4, 2>("both4:2", t);
        run<2, 4>("both2:4", t);
    }
    return 0;
}
