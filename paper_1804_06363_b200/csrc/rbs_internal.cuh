// rbs_internal.cuh -- shared device helpers of the B200 RB online solver.
//
// Geometry, fast integer division, the matrix-free cell-averaged stencil
// (eq12 with DESIGN.md AMB-1..4) and the FP64 tensor-core
// (DMMA m8n8k4) primitive.  sm_100a only.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "this library targets sm_100a (B200) only"
#endif

namespace rbs {

constexpr int kThreads = 256;      // threads per CTA of every streaming pass
constexpr int kMaxBatch = 64;      // B_pad <= 64 (8 DMMA column tiles)
constexpr int kMaxN = 64;          // n_pad <= 64 (8 DMMA row tiles)

// ---- fast unsigned division (Granlund-Montgomery), n < 2^31 ---------------
struct FastDiv {
    uint32_t d, M, s;
};

inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f;
    f.d = d;
    uint32_t s = 0;
    while ((1ull << s) < d) ++s;
    f.s = s;
    f.M = (uint32_t)((((1ull << 32) * ((1ull << s) - d)) / d) + 1ull);
    if (d == 1) { f.M = 0; f.s = 0; }
    return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
    return (__umulhi(n, f.M) + n) >> f.s;
}

// ---- grid geometry ---------------------------------------------------------
struct Geo {
    int dim;          // 2 or 3
    int m;            // interior nodes per axis, h = 1/(m+1)
    int64_t N;        // m^dim
    int Q;            // affine terms = px*py*pz
    int px, py, pz;   // blocks per axis
    FastDiv fm;       // division by m
    FastDiv f2m1;     // division by 2(m+1) (cell -> block)
    double scale;     // (m+1)^2 = h^-2 (AMB-3)
    double h2;        // h^2
    // 3D mesh slab: the local node range holds planes
    // K = kofs+1 .. kofs+mz of the global grid; planes own_lo <= K-kofs-1 < own_hi
    // are owned (count in reductions).  Full grid: kofs = 0, mz = m, own = [0, m).
    int kofs, mz, own_lo, own_hi;
    // general affine operator (rbs_set_operator_faces, NEXT(4), AMB-23): face
    // coefficients faces[(q*dim + d)*nf + idx] (layout in include/rbs.h); nullptr
    // for the thermal-block operator
    const double* faces;
    int64_t nf;
};

// z-neighbour availability of a node at global plane K inside its slab
__device__ __forceinline__ bool has_zm(const Geo& g, int K) { return K > 1 && K - g.kofs > 1; }
__device__ __forceinline__ bool has_zp(const Geo& g, int K) { return K < g.m && K - g.kofs < g.mz; }
// owned-plane mask of the slab (1 for every node of a 2D / full grid)
__device__ __forceinline__ bool owned(const Geo& g, int K) {
    const int u = K - g.kofs - 1;
    return u >= g.own_lo && u < g.own_hi;
}

// interior coordinates I,J,K in 1..m of node i (x fastest)
__device__ __forceinline__ void node_coords(const Geo& g, uint32_t i, int& I, int& J, int& K) {
    uint32_t t = fdiv(i, g.fm);
    I = (int)(i - t * (uint32_t)g.m) + 1;
    if (g.dim == 2) {
        J = (int)t + 1;
        K = 1;
    } else {
        uint32_t u = fdiv(t, g.fm);
        J = (int)(t - u * (uint32_t)g.m) + 1;
        K = (int)u + 1 + g.kofs;
    }
}

// block of cell index a (0..m) along an axis with p blocks: the cell centre
// (a + 1/2) h lies in block floor((2a+1) p / (2(m+1)))  (AMB-2)
__device__ __forceinline__ int axis_block(const Geo& g, int a, int p) {
    return (int)fdiv((uint32_t)((2 * a + 1) * p), g.f2m1);
}

// Edge coefficients of node (I,J,K) in neighbour order -x,+x,-y,+y(,-z,+z):
// mean of the cells sharing the edge (AMB-1), summed in AMB-4 order.
// th: theta laid out [q][ldb] (ldb = batch stride), b = this lane's query.
// face-operator edge coefficients (rbs_set_operator_faces, AMB-23)
template <int DIM>
__device__ __forceinline__ void node_kappa_faces(const Geo& g, const double* th, int ldb, int b,
                                                 int I, int J, int K, double* k) {
    // face indices from the node index P (layout in include/rbs.h):
    // x: P + (J-1) + m(K-1) (+1), y: P + m(K-1) (+m), z: P (+m^2); kappa = sum_q theta_q F_q
    const uint32_t m = (uint32_t)g.m, nf = (uint32_t)g.nf;
    const uint32_t P = (uint32_t)(I - 1) + m * ((uint32_t)(J - 1) + (DIM == 3 ? m * (uint32_t)(K - 1) : 0u));
    const uint32_t kz = DIM == 3 ? m * (uint32_t)(K - 1) : 0u;
    const uint32_t ix = P + (uint32_t)(J - 1) + kz, iy = nf + P + kz, iz = 2u * nf + P;
#pragma unroll
    for (int e = 0; e < 2 * DIM; ++e) k[e] = 0.0;
#pragma unroll 2
    for (int q = 0; q < g.Q; ++q) {
        const double t = th[q * ldb + b];
        const double* F = g.faces + (size_t)q * DIM * nf;
        k[0] = fma(t, __ldg(F + ix), k[0]);
        k[1] = fma(t, __ldg(F + ix + 1), k[1]);
        k[2] = fma(t, __ldg(F + iy), k[2]);
        k[3] = fma(t, __ldg(F + iy + m), k[3]);
        if (DIM == 3) {
            k[4] = fma(t, __ldg(F + iz), k[4]);
            k[5] = fma(t, __ldg(F + iz + m * m), k[5]);
        }
    }
}

template <int DIM>
__device__ __forceinline__ void node_kappa(const Geo& g, const double* th, int ldb, int b,
                                           int I, int J, int K, double* k) {
    if (g.faces) {
        node_kappa_faces<DIM>(g, th, ldb, b, I, J, K, k);
        return;
    }
    const int bx0 = axis_block(g, I - 1, g.px), bx1 = axis_block(g, I, g.px);
    const int by0 = axis_block(g, J - 1, g.py) * g.px, by1 = axis_block(g, J, g.py) * g.px;
    int bz0 = 0, bz1 = 0;
    if (DIM == 3) {
        const int pxy = g.px * g.py;
        bz0 = axis_block(g, K - 1, g.pz) * pxy;
        bz1 = axis_block(g, K, g.pz) * pxy;
    }
    if (bx0 == bx1 && by0 == by1 && bz0 == bz1) {
        // all cells around the node in one block: 0.5*(c+c) = 0.25*((c+c)+(c+c)) = c
        // exactly, so this is bitwise the general formula with one load
        const double c = th[(bx0 + by0 + bz0) * ldb + b];
#pragma unroll
        for (int e = 0; e < 2 * DIM; ++e) k[e] = c;
        return;
    }
    if (DIM == 2) {
        const double c00 = th[(bx0 + by0) * ldb + b], c10 = th[(bx1 + by0) * ldb + b];
        const double c01 = th[(bx0 + by1) * ldb + b], c11 = th[(bx1 + by1) * ldb + b];
        k[0] = 0.5 * (c00 + c01);
        k[1] = 0.5 * (c10 + c11);
        k[2] = 0.5 * (c00 + c10);
        k[3] = 0.5 * (c01 + c11);
    } else {
        // c[dx][dy][dz] = theta of cell (I-1+dx, J-1+dy, K-1+dz)
        const double c000 = th[(bx0 + by0 + bz0) * ldb + b], c100 = th[(bx1 + by0 + bz0) * ldb + b];
        const double c010 = th[(bx0 + by1 + bz0) * ldb + b], c110 = th[(bx1 + by1 + bz0) * ldb + b];
        const double c001 = th[(bx0 + by0 + bz1) * ldb + b], c101 = th[(bx1 + by0 + bz1) * ldb + b];
        const double c011 = th[(bx0 + by1 + bz1) * ldb + b], c111 = th[(bx1 + by1 + bz1) * ldb + b];
        k[0] = 0.25 * ((c000 + c010) + (c001 + c011));
        k[1] = 0.25 * ((c100 + c110) + (c101 + c111));
        k[2] = 0.25 * ((c000 + c100) + (c001 + c101));
        k[3] = 0.25 * ((c010 + c110) + (c011 + c111));
        k[4] = 0.25 * ((c000 + c100) + (c010 + c110));
        k[5] = 0.25 * ((c001 + c101) + (c011 + c111));
    }
}

// the general edge coefficients (block interfaces, face operators) out of line: keeps the
// register footprint of the common uniform-block path small
__device__ __noinline__ void node_kappa3_call(const Geo& g, const double* th, int ldb, int b, int I, int J,
                                              int K, double* k) {
    node_kappa<3>(g, th, ldb, b, I, J, K, k);
}

// 2D edge coefficients from precomputed cell blocks (bx of cells I-1, I; by*px of
// cells J-1, J): bitwise the same values as node_kappa<2>.
__device__ __forceinline__ void kappa2_blocks(const double* th, int ldb, int b, int bx0, int bx1,
                                              int by0, int by1, double* k) {
    if (bx0 == bx1 && by0 == by1) {
        const double c = th[(bx0 + by0) * ldb + b];
        k[0] = k[1] = k[2] = k[3] = c;
        return;
    }
    const double c00 = th[(bx0 + by0) * ldb + b], c10 = th[(bx1 + by0) * ldb + b];
    const double c01 = th[(bx0 + by1) * ldb + b], c11 = th[(bx1 + by1) * ldb + b];
    k[0] = 0.5 * (c00 + c01);
    k[1] = 0.5 * (c10 + c11);
    k[2] = 0.5 * (c00 + c10);
    k[3] = 0.5 * (c01 + c11);
}

// neighbour values (order -x,+x,-y,+y(,-z,+z); 0 outside) of element (i,b)
// of a node-major batch vector v[N][ldb].
template <int DIM>
__device__ __forceinline__ void node_nbrs(const Geo& g, const double* __restrict__ v, int ldb,
                                          int64_t i, int b, int I, int J, int K, double* nb) {
    const double* p = v + i * ldb + b;
    const int64_t sy = (int64_t)g.m * ldb;
    nb[0] = I > 1 ? __ldg(p - ldb) : 0.0;
    nb[1] = I < g.m ? __ldg(p + ldb) : 0.0;
    nb[2] = J > 1 ? __ldg(p - sy) : 0.0;
    nb[3] = J < g.m ? __ldg(p + sy) : 0.0;
    if (DIM == 3) {
        const int64_t sz = sy * g.m;
        nb[4] = has_zm(g, K) ? __ldg(p - sz) : 0.0;
        nb[5] = has_zp(g, K) ? __ldg(p + sz) : 0.0;
    }
}

// (A(theta) v)_P = (m+1)^2 sum_e kappa_e (v_P - v_P')
template <int DIM>
__device__ __forceinline__ double stencil_apply(const Geo& g, const double* k, double vp,
                                                const double* nb) {
    double s = k[0] * (vp - nb[0]);
#pragma unroll
    for (int e = 1; e < 2 * DIM; ++e) s = fma(k[e], vp - nb[e], s);
    return g.scale * s;
}

// Gauss-Seidel value (direct form, AMB-6): (h^2 b_P + sum kappa y_P') / sum kappa
template <int DIM>
__device__ __forceinline__ double gs_value(const Geo& g, const double* k, double rhs,
                                           const double* nb) {
    double num = g.h2 * rhs, den = k[0];
    num = fma(k[0], nb[0], num);
#pragma unroll
    for (int e = 1; e < 2 * DIM; ++e) {
        num = fma(k[e], nb[e], num);
        den += k[e];
    }
    return num / den;
}

// ---- programmatic dependent launch (the 2D iteration passes) -----------------
// A pass launched with cudaLaunchAttributeProgrammaticStreamSerialization may start
// its prologue (shared-memory zeroing, constant tables, barrier init) while the
// previous pass drains; pdl_wait() blocks until that pass has completed and its
// writes are visible (a no-op for an ordinary launch).  Every pass calls
// pdl_trigger() only after its own pdl_wait(), so when pass k+1 starts its prologue
// pass k-1 has completed: a prologue may read only inputs that do not change during
// the solve (W, theta, A_n^{-1}).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- FP64 tensor core: D(8x8) += A(8x4, row) * B(4x8, col) ------------------
// lane l: a = A[l>>2][l&3], b = B[l&3][l>>2], d0,d1 = D[l>>2][2(l&3)+{0,1}]
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

}  // namespace rbs
