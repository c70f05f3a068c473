// Microbenchmark: DMMA issue rate of one tensor warp per SMSP while other warps
// of the same SM issue FP64 vector instructions (DADD/DFMA) at a given density.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_mix tools/fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

// warps 0..3: DMMA, 8 independent chains, `iters` rounds; clock of the loop -> cyc[]
// warps 4..15: mode 0 idle, 1 pure DFMA chains, 2 one DADD per `gap` integer ops
__global__ void k_mix(double* out, long long* cyc, int iters, int mode, int gap, int vit) {
    const int warp = threadIdx.x >> 5;
    if (warp < 4) {
        double d[8][2];
        for (int c = 0; c < 8; ++c) d[c][0] = d[c][1] = 0.0;
        double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
        __syncwarp();
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int c = 0; c < 8; ++c)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
        }
        long long t1 = clock64();
        double s = 0;
        for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1];
        if (s == 1234.5) out[0] = s;
        if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 4 + warp] = t1 - t0;
        return;
    }
    if (mode == 0) return;
    if (mode == 1) {
        double d[8];
        for (int c = 0; c < 8; ++c) d[c] = threadIdx.x;
        for (int i = 0; i < vit; ++i) {
#pragma unroll
            for (int c = 0; c < 8; ++c) d[c] = fma(d[c], 1.0000001, 1e-7);
        }
        double s = 0;
        for (int c = 0; c < 8; ++c) s += d[c];
        if (s == 1234.5) out[0] = s;
        return;
    }
    // mode 2: sparse FP64 among integer work
    double x = threadIdx.x, y = 1e-7;
    unsigned u = threadIdx.x;
    for (int i = 0; i < vit; ++i) {
        for (int k = 0; k < gap; ++k) u = u * 1664525u + 1013904223u;
        x = x + y;
        y = (double)(u & 1) * 1e-9 + y;
    }
    if (x == 1234.5 || u == 7) out[0] = x;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 148 * 4 * 8);
    long long h[148 * 4];
    const int iters = 4000;
    struct { int mode, gap, vit; const char* name; } cases[] = {
        {0, 0, 0, "vector warps idle"},
        {1, 0, 20000, "vector warps: DFMA chains (saturating)"},
        {2, 4, 40000, "vector warps: 2 DADD-ish per 4 int ops"},
        {2, 16, 8000, "vector warps: 2 FP64 per 16 int ops"},
        {2, 64, 3000, "vector warps: 2 FP64 per 64 int ops"},
    };
    for (auto& c : cases) {
        k_mix<<<148, 512>>>(out, cyc, 100, c.mode, c.gap, 100);
        k_mix<<<148, 512>>>(out, cyc, iters, c.mode, c.gap, c.vit);
        cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
        double s = 0;
        for (int i = 0; i < 148 * 4; ++i) s += (double)h[i];
        s /= 148 * 4;
        printf("%-45s DMMA warp: %.1f cyc/DMMA\n", c.name, s / (iters * 8.0));
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
