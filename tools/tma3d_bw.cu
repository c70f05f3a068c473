// tma3d_bw.cu -- microbenchmark: how fast can a z-plane march stream haloed plane tiles of a
// node-major batch vector v[m][m][m][16] (fp64) into shared memory on sm_100a?
//   mode 0: one 4-D tensor-map copy per plane (box [16][TX+2][TY+2][1], the zmarch.cuh path)
//   mode 1: 1-D bulk copies, one per tile row (TY+2 copies of (TX+2)*128 B)
//   mode 2: plain grid-stride copy v -> w with 16-byte loads (streaming reference)
// Each CTA (512 threads, one per SM) marches its (x, y) tiles through all planes with a ring of
// NS slots, DI planes in flight, one barrier per plane, no compute.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma3d_bw tools/tma3d_bw.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                                  \
        }                                                                             \
    } while (0)

constexpr int BP = 16;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
    asm volatile(
        "{\n.reg .pred P1;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W%=;\n}\n" ::"r"(
            su32(b)),
        "r"(par)
        : "memory");
}
__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6];" ::"r"(su32(dst)),
        "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(su32(b))
        : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(b))
                 : "memory");
}

struct P {
    int m, TX, TY, ntx, nty, NS, DI, mode;
    const double* v;
};

__global__ void __launch_bounds__(512, 1) k_march(const __grid_constant__ CUtensorMap map, const P p, double* sink) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bar[8];
    const int HX = p.TX + 2, HY = p.TY + 2;
    const uint32_t plane = HX * HY * BP * 8;
    if (threadIdx.x == 0) {
        for (int k = 0; k < p.NS; ++k) mbar_init(&bar[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t G = 0;
    double acc = 0.0;
    const int tiles = p.ntx * p.nty;
    for (int u = blockIdx.x; u < tiles; u += gridDim.x) {
        const int ty = u / p.ntx, tx = u - ty * p.ntx;
        const int x0 = 1 + tx * p.TX, y0 = 1 + ty * p.TY;
        const int T = p.m;
        auto issue = [&](int t) {
            const uint32_t q = G + t;
            uint64_t* b = &bar[q % p.NS];
            double* dst = sm + (size_t)(q % p.NS) * (plane / 8);
            if (p.mode == 0) {
                expect_tx(b, plane);
                tma4(dst, &map, 0, x0 - 2, y0 - 2, t, b);
            } else {
                // rows y0-1 .. y0+TY, columns x0-1 .. x0+TX clamped to the grid
                const int xa = max(1, x0 - 1), xb = min(p.m, x0 + p.TX);
                const int ya = max(1, y0 - 1), yb = min(p.m, y0 + p.TY);
                const uint32_t rb = (uint32_t)(xb - xa + 1) * BP * 8;
                expect_tx(b, rb * (yb - ya + 1));
                for (int y = ya; y <= yb; ++y)
                    bulk(dst + ((y - (y0 - 1)) * HX + (xa - (x0 - 1))) * BP,
                         p.v + (((size_t)t * p.m + (y - 1)) * p.m + (xa - 1)) * BP, rb, b);
            }
        };
        __syncthreads();
        if (threadIdx.x == 0)
            for (int t = 0; t < p.DI && t < T; ++t) issue(t);
        for (int t = 0; t < T; ++t) {
            const uint32_t q = G + t;
            mbar_wait(&bar[q % p.NS], (q / p.NS) & 1);
            acc += sm[(size_t)(q % p.NS) * (plane / 8) + threadIdx.x];
            __syncthreads();
            if (threadIdx.x == 0 && t + p.DI < T) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(t + p.DI);
            }
        }
        G += T;
    }
    if (acc == 12345.678) sink[threadIdx.x] = acc;
}

__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

int main(int argc, char** argv) {
    const int m = argc > 1 ? atoi(argv[1]) : 255;
    const size_t N = (size_t)m * m * m * BP;
    double *v, *w, *sink;
    CK(cudaMalloc(&v, N * 8));
    CK(cudaMalloc(&w, N * 8));
    CK(cudaMalloc(&sink, 4096));
    CK(cudaMemset(v, 0, N * 8));
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult qr;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr));
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    // streaming reference
    for (int rep = 0; rep < 2; ++rep) {
        CK(cudaEventRecord(e0));
        k_copy<<<sms * 8, 512>>>((const double2*)v, (double2*)w, N / 2);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
    }
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("copy: %.3f ms, %.1f GB/s (read+write)\n", ms, 2.0 * N * 8 / ms / 1e6);
    struct Cfg { int TX, TY, NS, DI; };
    std::vector<Cfg> cfgs = {{16, 8, 6, 3}, {16, 8, 8, 5}, {32, 8, 5, 3}, {32, 4, 6, 4}, {64, 4, 4, 2}, {16, 16, 5, 3}};
    CK(cudaFuncSetAttribute(k_march, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    for (int mode = 0; mode < 2; ++mode)
        for (auto c : cfgs) {
            const int HX = c.TX + 2, HY = c.TY + 2;
            const size_t smem = (size_t)c.NS * HX * HY * BP * 8;
            if (smem > 220 * 1024) continue;
            CUtensorMap map;
            cuuint64_t dims[4] = {BP, (cuuint64_t)m, (cuuint64_t)m, (cuuint64_t)m};
            cuuint64_t str[3] = {BP * 8, (cuuint64_t)m * BP * 8, (cuuint64_t)m * m * BP * 8};
            cuuint32_t box[4] = {BP, (cuuint32_t)HX, (cuuint32_t)HY, 1}, es[4] = {1, 1, 1, 1};
            if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, v, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
                printf("encode failed\n");
                continue;
            }
            P p{m, c.TX, c.TY, (m + c.TX - 1) / c.TX, (m + c.TY - 1) / c.TY, c.NS, c.DI, mode, v};
            const int tiles = p.ntx * p.nty;
            for (int rep = 0; rep < 2; ++rep) {
                CK(cudaEventRecord(e0));
                k_march<<<sms, 512, smem>>>(map, p, sink);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
            }
            CK(cudaGetLastError());
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const double interior = (double)N * 8, haloed = (double)tiles * HX * HY * BP * 8 * m;
            printf("mode %d tile %dx%d ring %d DI %d: %.3f ms, interior %.1f GB/s, smem-fill %.1f GB/s (tiles %d, "
                   "waves %.2f)\n",
                   mode, c.TX, c.TY, c.NS, c.DI, ms, interior / ms / 1e6, haloed / ms / 1e6, tiles,
                   (double)tiles / sms);
        }
    return 0;
}
