// Microbenchmark: DMMA issue rate of the k_smooth2 prolongation loop shapes
// (5 accumulator chains, A fragments from shared memory, E in registers).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_ws tools/dmma_ws.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

constexpr int T = 5, NKMAX = 16;

// mode 0: runtime nk, loads right before the DMMAs of a k-step (no prefetch)
// mode 1: runtime nk, loads PD = 2 k-steps ahead
// mode 2: compile-time nk = 10, loads 2 ahead (no uniform branches)
template <int MODE>
__global__ void k_loop(double* out, long long* cyc, int nk, int reps) {
    __shared__ double w[64 * 48];
    for (int i = threadIdx.x; i < 64 * 48; i += blockDim.x) w[i] = 1e-3 * (i % 7);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp >= 4) return;
    double ef[NKMAX];
#pragma unroll
    for (int k = 0; k < NKMAX; ++k) ef[k] = k < nk ? 1.0 + k * 1e-3 : 0.0;
    const double* wb = w + (lane >> 2) * 44 + (lane & 3);
    double d0[T], d1[T];
#pragma unroll
    for (int i = 0; i < T; ++i) d0[i] = d1[i] = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (MODE == 0) {
#pragma unroll 1
            for (int k = 0; k < nk; k += 2) {
                double wa[T], wc[T];
#pragma unroll
                for (int i = 0; i < T; ++i) {
                    wa[i] = wb[i * 8 * 44 + 4 * k];
                    wc[i] = wb[i * 8 * 44 + 4 * k + 4];
                }
                const double e0 = wb[k], e1 = wb[k + 1];
#pragma unroll
                for (int i = 0; i < T; ++i) dmma(d0[i], d1[i], wa[i], e0);
#pragma unroll
                for (int i = 0; i < T; ++i) dmma(d0[i], d1[i], wc[i], e1);
            }
        } else {
            constexpr int PD = 2;
            const int n = MODE == 2 ? 10 : nk;
            double wf[PD + 1][T];
#pragma unroll
            for (int k = 0; k < PD; ++k)
#pragma unroll
                for (int i = 0; i < T; ++i) wf[k][i] = wb[i * 8 * 44 + 4 * k];
#pragma unroll
            for (int k = 0; k < NKMAX; ++k) {
                if (k < n) {
                    if (k + PD < n)
#pragma unroll
                        for (int i = 0; i < T; ++i) wf[(k + PD) % (PD + 1)][i] = wb[i * 8 * 44 + 4 * (k + PD)];
#pragma unroll
                    for (int i = 0; i < T; ++i) dmma(d0[i], d1[i], wf[k % (PD + 1)][i], ef[k]);
                }
            }
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < T; ++i) s += d0[i] + d1[i];
    if (s == 1234.5) out[0] = s;
    if (lane == 0) cyc[blockIdx.x * 4 + warp] = t1 - t0;
}

template <int MODE>
void run(const char* name, double* out, long long* cyc, int nk) {
    const int reps = 2000;
    k_loop<MODE><<<148, 512>>>(out, cyc, nk, 10);
    k_loop<MODE><<<148, 512>>>(out, cyc, nk, reps);
    cudaDeviceSynchronize();
    long long h[148 * 4];
    cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < 148 * 4; ++i) s += (double)h[i];
    s /= 148 * 4;
    printf("%-40s %.1f cyc/DMMA (%.0f cyc per 50-DMMA step)\n", name, s / (reps * (double)nk * T),
           s / reps * 10.0 / nk);
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 148 * 4 * 8);
    run<0>("runtime nk, loads in-iteration", out, cyc, 10);
    run<1>("runtime nk, prefetch 2", out, cyc, 10);
    run<2>("compile-time nk, prefetch 2", out, cyc, 10);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
