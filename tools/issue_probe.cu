// Does a DFMA block the warp scheduler's issue port for both of its FP64-pipe cycles on sm_100a?
// 8 independent DFMA chains per thread, with K other instructions (integer ALU, FP32 FMA, shuffle,
// shared-memory load) interleaved per 8 DFMA.  If the FP64 rate stays at the DFMA-only rate while
// K <= 8, the other pipes issue in the FP64 pipe's second cycle and a pair kernel with 31 FP64 of
// 48 instructions can in principle fill the FP64 pipe; if it drops as 16 / (16 + K), it cannot.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o issue_probe tools/issue_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

enum Kind { kInt = 0, kFp32 = 1, kShfl = 2, kLds = 3 };

template <int KIND, int K>
__global__ void k(double* out, int iters, double s) {
    __shared__ double sm[256];
    double f[8];
    for (int i = 0; i < 8; ++i) f[i] = threadIdx.x * 1e-3 + i;
    if (threadIdx.x < 256) sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    unsigned x[8];
    float g[8];
    for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x + i; g[i] = threadIdx.x + i; }
    const float gs = (float)s;
    unsigned addr = (unsigned)__cvta_generic_to_shared(&sm[threadIdx.x & 255]);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                f[i] = fma(f[i], s, 1e-7);
                if (i < K) {
                    if (KIND == kInt) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(x[(i + 1) & 7]), "r"(it));
                    if (KIND == kFp32) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(g[i]) : "f"(gs));
                    if (KIND == kShfl) asm volatile("shfl.sync.idx.b32 %0, %0, %1, 31, 0xffffffff;" : "+r"(x[i]) : "r"((threadIdx.x + 1) & 31));
                    if (KIND == kLds) asm volatile("ld.shared.b32 %0, [%1];" : "=r"(x[i]) : "r"(addr));
                }
            }
        }
    }
    double acc = 0;
    for (int i = 0; i < 8; ++i) acc += f[i] + x[i] + g[i];
    if (acc == 12345.678) out[0] = acc;
}

template <int KIND, int K>
void run(const char* name, int threads, int blocks_per_sm) {
    double* o;
    cudaMalloc(&o, 8);
    int iters = 2000, blocks = 148 * blocks_per_sm;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<KIND, K><<<blocks, threads>>>(o, 10, 0.9999999);
    cudaEventRecord(e0);
    k<KIND, K><<<blocks, threads>>>(o, iters, 0.9999999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double warps = (double)blocks * threads / 32;
    double dfma = warps * iters * 4 * 8;
    double tf = dfma * 32 * 2 / (ms * 1e-3) / 1e12;
    printf("%-5s K=%d per 8 DFMA, %2d warps/SM: %.3f ms  DFMA %.2f TF\n", name, K, threads / 32 * blocks_per_sm, ms, tf);
    cudaFree(o);
}

template <int KIND>
void sweep(const char* name) {
    for (int w : {12, 32}) {
        const int threads = 64, bps = w / 2;
        run<KIND, 0>(name, threads, bps);
        run<KIND, 2>(name, threads, bps);
        run<KIND, 4>(name, threads, bps);
        run<KIND, 6>(name, threads, bps);
        run<KIND, 8>(name, threads, bps);
    }
}

int main() {
    sweep<kInt>("int");
    sweep<kFp32>("fp32");
    sweep<kShfl>("shfl");
    sweep<kLds>("lds");
    return 0;
}
