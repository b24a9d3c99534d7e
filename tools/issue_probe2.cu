// FP64 issue probe 2 (sm_100a): what keeps a pair kernel's FP64 pipe below the DFMA-only rate?
//   V0  f = fma(f, s, imm)            one register operand pair + reuse: the peak probe's shape
//   V1  f = fma(f, s, t)              s, t registers shared by all chains
//   V2  f = fma(g_i, h_i, f)          three distinct 64-bit register operands per DFMA
//   V3  V2 with g_i, h_i rewritten by DADD every trip (no operand stays in the reuse cache)
//   V4  chains of length NCH = 1, 2, 4 (dependent-issue latency)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o issue_probe2 tools/issue_probe2.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int V, int NCH>
__global__ void k(double* out, int iters, double s, double t) {
    double f[8], g[8], h[8];
    for (int i = 0; i < 8; ++i) {
        f[i] = threadIdx.x * 1e-3 + i;
        g[i] = 1.0 + 1e-9 * (threadIdx.x + i);
        h[i] = 1.0 - 1e-9 * (threadIdx.x + 2 * i);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
#pragma unroll
            for (int i = 0; i < NCH; ++i) {
                if (V == 0) f[i] = fma(f[i], s, 1e-7);
                if (V == 1) f[i] = fma(f[i], s, t);
                if (V == 2) f[i] = fma(g[i], h[i], f[i]);
                if (V == 3) {
                    f[i] = fma(g[i], h[i], f[i]);
                    g[i] = g[i] + t;
                }
            }
        }
    }
    double acc = 0;
    for (int i = 0; i < 8; ++i) acc += f[i] + g[i] + h[i];
    if (acc == 12345.678) out[0] = acc;
}

template <int V, int NCH>
void run(const char* name, int warps_per_sm) {
    double* o;
    cudaMalloc(&o, 8);
    const int threads = 64, iters = 2000, blocks = 148 * warps_per_sm / 2;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<V, NCH><<<blocks, threads>>>(o, 10, 0.9999999, 1e-7);
    cudaEventRecord(e0);
    k<V, NCH><<<blocks, threads>>>(o, iters, 0.9999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (double)blocks * threads / 32;
    const double d = warps * iters * 4 * NCH * (V == 3 ? 2 : 1);
    const double per_smsp_cycle = d / (148.0 * 4) / (ms * 1e-3 * 1.965e9);
    printf("%-28s chains %d, %2d warps/SM: %.3f ms  %.3f FP64 instr/clk/SMSP (0.5 = pipe full)\n", name, NCH, warps_per_sm,
           ms, per_smsp_cycle);
    cudaFree(o);
}

int main() {
    for (int w : {4, 12, 32}) {
        run<0, 8>("V0 fma(f,s,imm)", w);
        run<1, 8>("V1 fma(f,s,t)", w);
        run<2, 8>("V2 fma(g_i,h_i,f_i)", w);
        run<3, 8>("V3 V2 + dadd on g_i", w);
    }
    run<0, 1>("V4 latency", 4);
    run<0, 2>("V4 latency", 4);
    run<0, 4>("V4 latency", 4);
    run<2, 1>("V4 latency (3 regs)", 4);
    run<2, 2>("V4 latency (3 regs)", 4);
    run<2, 4>("V4 latency (3 regs)", 4);
    return 0;
}
