// Microbenchmark: FP64 tensor (DMMA m8n8k4) and FP64 FMA (DFMA) peak on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmma(double* out, int iters) {
    double d[8][2];
    for (int c = 0; c < 8; ++c) d[c][0] = d[c][1] = 0.0;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1];
    if (s == 1234.5) out[0] = s;
}

__global__ void k_dfma(double* out, int iters) {
    double d[8];
    for (int c = 0; c < 8; ++c) d[c] = threadIdx.x;
    const double a = 1.0000001, b = 1e-7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) d[c] = fma(d[c], a, b);
    }
    double s = 0;
    for (int c = 0; c < 8; ++c) s += d[c];
    if (s == 1234.5) out[0] = s;
}

template <int C>
__global__ void k_dmma_chain(double* out, int iters) {
    double d[C][2];
    for (int c = 0; c < C; ++c) d[c][0] = d[c][1] = 0.0;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int c = 0; c < C; ++c) s += d[c][0] + d[c][1];
    if (s == 1234.5) out[0] = s;
}

template <int C>
void chain_test(double* out, int sms) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    k_dmma_chain<C><<<sms, 128>>>(out, 100);
    cudaEventRecord(e0);
    k_dmma_chain<C><<<sms, 128>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double cyc = ms * 1e-3 * 1.965e9 / iters;   // cycles per iteration (1 warp / SMSP)
    printf("DMMA 1 warp/SMSP, %d chains: %.1f cycles per chain step (%.1f cyc/DMMA/SMSP)\n", C, cyc, cyc / C);
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int sms = p.multiProcessorCount;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int warps : {4, 8, 16, 32}) {
        const int iters = 20000;
        k_dmma<<<sms, warps * 32>>>(out, 100);
        cudaEventRecord(e0);
        k_dmma<<<sms, warps * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = (double)sms * warps * iters * 8 * 512.0;
        printf("DMMA warps/SM %2d: %.2f TFLOP/s (%.2f cyc/DMMA/SM @1.965GHz)\n", warps, flops / ms / 1e9,
               ms * 1e-3 * 1.965e9 / ((double)warps * iters * 8));
        k_dfma<<<sms, warps * 32>>>(out, 100);
        cudaEventRecord(e0);
        k_dfma<<<sms, warps * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double f2 = (double)sms * warps * 32 * iters * 8 * 2.0;
        printf("DFMA warps/SM %2d: %.2f TFLOP/s\n", warps, f2 / ms / 1e9);
    }
    chain_test<1>(out, sms);
    chain_test<2>(out, sms);
    chain_test<4>(out, sms);
    chain_test<8>(out, sms);
    return 0;
}
