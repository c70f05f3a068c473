// zmarch.cuh -- z-plane marching passes for 3D grids (sm_100a), fed by TMA tensor maps.
//
// The 3D streaming passes of an RBCG iteration as 2.5D marches: a CTA owns an (x, y)
// tile of TX x TY nodes and a segment of z-planes and walks up the planes.  Each
// plane's tile arrives by ONE 4-D tensor-map copy (cp.async.bulk.tensor.4d, SASS
// UTMALDG) of the node-major batch vector v[K][J][I][Bp] -- box [Bp][TX+2][TY+2][1]
// for the operand the 7-point stencil reads (its x/y halo included; halo nodes outside
// the grid are zero-filled by the TMA unit, i.e. the homogeneous Dirichlet values), box
// [Bp][TX][TY][1] for the pointwise operands -- into shared-memory rings completing on
// mbarriers, several planes ahead of the compute.  Every z-neighbour is served from the
// ring (each plane is read from HBM once per pass; the x/y halo, ~1.4x the tile, from
// L2) and every pass has one CTA barrier per plane.
//
//   k_cgz   RBCG Step 11 + sigma of Step 5: p = y + beta p_old, sigma = p^T A p
//            -- one pass instead of k_pnew3 + k_sigma3r
//   k_gsz   one red-black Gauss-Seidel half-sweep (eq8, AMB-5/6),
//           LAST: y^T r, y^T y and RBCG Step 10
//   k_xrz   RBCG Steps 6-7: x += alpha p, r -= alpha A p
//
// Per node the stencil is that of the row-segment kernels (node_kappa, stencil_apply,
// neighbour order -x,+x,-y,+y,-z,+z; bitwise the same values); a Gauss-Seidel update of
// a node inside one block is the direct form y = h^2/(6 theta) b + (sum of the six
// neighbours)/6 with the h^2/(6 theta) table in shared memory (no division; within an ulp
// of gs_value, AMB-4), block-interface nodes keep gs_value.  The half-sweep maps the
// CTA's threads onto the sweep's colour only (every lane of a warp updates a node).
// FACES instantiations take the face-coefficient operator (AMB-23) with the coefficients
// of every node loaded inline.  Kernel arguments are __grid_constant__ (the out-of-line interface path takes their
// address without a local-memory copy).  Full grid only (mesh slabs keep the row-segment
// kernels).
#pragma once
#include <cuda.h>

#include "march2.cuh"

namespace rbs {

constexpr int kZT = 512;                // threads per CTA (== kFlat: the LAST epilogues are shared)
static_assert(kZT == kFlat, "z-march epilogues reuse the flat passes' reductions");

// tile shapes: 2048 interior node-queries per plane (4 per thread) for every batch width
template <int BP> struct ZShape;
template <> struct ZShape<8>  { static constexpr int TX = 32, TY = 8; };
template <> struct ZShape<16> { static constexpr int TX = 16, TY = 8; };
template <> struct ZShape<32> { static constexpr int TX = 16, TY = 4; };

template <int BP>
struct ZGeom {
    static constexpr int TX = ZShape<BP>::TX, TY = ZShape<BP>::TY;
    static constexpr int HX = TX + 2, HY = TY + 2;
    static constexpr int HP = HX * HY * BP;      // doubles of a haloed plane tile
    static constexpr int IP = TX * TY * BP;      // doubles of an interior plane tile
    static constexpr int NE = IP / kZT;          // interior elements per thread
    static constexpr int LGB = LgB<BP>::v;
    // TMA issue distance DI (planes ahead of the compute): the stencil operand's ring holds
    // the 3-plane window + DI slots (a slot is refilled only after the step that last reads
    // it has passed its barrier); 2 for the widest batch so every ring fits 227 KB
    static constexpr int DI = BP == 32 ? 2 : 3;
    static constexpr int NA = DI + 3;
    static_assert(IP % kZT == 0, "tile must hold a whole number of elements per thread");
};

// work partition: ntx x nty tiles x nz z-segments of zlen planes, units handed out
// round-robin to a persistent grid (unit u: tile u % tiles, segment u / tiles)
struct ZPart {
    int ntx, nty, nz, zlen, units;
};

template <int BP>
__host__ __device__ constexpr size_t zsmem_bytes(int kind, int Q) {
    // kind 0: k_cgz (y ring NA + p_old ring DI, haloed), 1: k_gsz (y ring NA haloed + r ring
    // DI+1 interior + the h^2/(6 theta) table), 2: k_xrz (p ring of 5 haloed + x, r rings of 3
    // interior); + theta table
    using Z = ZGeom<BP>;
    return (size_t)8 * (kind == 0 ? (Z::NA + Z::DI) * Z::HP
                        : kind == 1 ? Z::NA * Z::HP + (Z::DI + 1) * Z::IP + Q * BP
                                    : 5 * Z::HP + 6 * Z::IP) +
           (size_t)Q * BP * 8;
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void zunit(const ZPart& p, int m, int u, int TX, int TY, int& x0, int& y0, int& za,
                                      int& zb) {
    const int tiles = p.ntx * p.nty;
    const int zs = u / tiles, t = u - zs * tiles;
    const int ty = t / p.ntx, tx = t - ty * p.ntx;
    x0 = 1 + tx * TX;
    y0 = 1 + ty * TY;
    za = 1 + zs * p.zlen;
    zb = min(m + 1, za + p.zlen);
}

// the 7-point stencil with all six edge coefficients equal to c: the operations of
// stencil_apply<3> with k[e] = c in the same order (bitwise equal), no coefficient array
__device__ __forceinline__ double stencil_c(double scale, double c, double vp, const double* nb) {
    double s = c * (vp - nb[0]);
#pragma unroll
    for (int e = 1; e < 6; ++e) s = fma(c, vp - nb[e], s);
    return scale * s;
}
// general node (block interface): cell-averaged coefficients out of line
// (neighbour values by value: the caller's arrays stay in registers)
__device__ __noinline__ double stencil_general(const Geo& g, const double* s_th, int ldb, int b, int I, int J,
                                               int K, double vp, double n0, double n1, double n2, double n3,
                                               double n4, double n5) {
    double k[6];
    const double nb[6] = {n0, n1, n2, n3, n4, n5};
    node_kappa<3>(g, s_th, ldb, b, I, J, K, k);
    return stencil_apply<3>(g, k, vp, nb);
}
__device__ __noinline__ double gs_general(const Geo& g, const double* s_th, int ldb, int b, int I, int J, int K,
                                          double rhs, double n0, double n1, double n2, double n3, double n4,
                                          double n5) {
    double k[6];
    const double nb[6] = {n0, n1, n2, n3, n4, n5};
    node_kappa<3>(g, s_th, ldb, b, I, J, K, k);
    return gs_value<3>(g, k, rhs, nb);
}

// per-thread view of its NE interior elements of the current tile (loop invariant over z)
template <int BP>
struct ZElems {
    using Z = ZGeom<BP>;
    uint32_t h[Z::NE];       // byte offset of the element in a haloed plane
    int gxy[Z::NE];          // element offset within a global plane: ((J-1) m + I-1) Bp + b (< 2^31)
    int cxy[Z::NE];          // bx + by*px of the node's cells if they agree in x and y, -1 if not,
                             // -2: node outside the grid
    __device__ __forceinline__ bool in(int j) const { return cxy[j] != -2; }
    __device__ __forceinline__ void init(const Geo& g, int x0, int y0, int tid) {
        const int b = tid & (BP - 1);
#pragma unroll
        for (int j = 0; j < Z::NE; ++j) {
            const int n = (tid + j * kZT) >> Z::LGB;
            const int ix = n % Z::TX, iy = n / Z::TX;
            const int I = x0 + ix, J = y0 + iy;
            h[j] = 8u * (uint32_t)(((iy + 1) * Z::HX + ix + 1) * BP + b);
            gxy[j] = ((J - 1) * g.m + (I - 1)) * BP + b;
            const int bx0 = axis_block(g, I - 1, g.px), bx1 = axis_block(g, I, g.px);
            const int by0 = axis_block(g, J - 1, g.py), by1 = axis_block(g, J, g.py);
            cxy[j] = (I > g.m || J > g.m) ? -2 : (bx0 == bx1 && by0 == by1) ? bx0 + by0 * g.px : -1;
        }
    }
};

// colour-compact view for a half-sweep: the TX*TY/2 nodes of one red-black colour of a
// plane tile, NC = NE/2 per thread.  Colour node cn = slot + (kZT/BP) j sits in tile row
// iy = cn / (TX/2) at column ix = 2 (cn % (TX/2)) + ((P + iy) & 1), where P = 0 / 1 is the
// colour's column parity in row 0 of that plane; both parities are kept (they alternate
// with the plane) -- the other parity is the other colour of the same plane (LAST's dots)
template <int BP>
struct ZColour {
    using Z = ZGeom<BP>;
    static constexpr int NC = Z::NE / 2;
    uint32_t h[2][NC];       // haloed-plane byte offset
    uint32_t ri[2][NC];      // interior-plane byte offset (the r ring)
    int gxy[2][NC];          // < 2^31: element offset within a global plane
    int cxy[2][NC];          // uniform x/y block index, -1: interface, -2: outside the grid
    __device__ __forceinline__ void init(const Geo& g, int x0, int y0, int tid) {
        const int b = tid & (BP - 1);
#pragma unroll
        for (int P = 0; P < 2; ++P)
#pragma unroll
            for (int j = 0; j < NC; ++j) {
                const int cn = (tid >> Z::LGB) + j * (kZT / BP);
                const int iy = cn / (Z::TX / 2);
                const int ix = 2 * (cn % (Z::TX / 2)) + ((P + iy) & 1);
                const int I = x0 + ix, J = y0 + iy;
                h[P][j] = 8u * (uint32_t)(((iy + 1) * Z::HX + ix + 1) * BP + b);
                ri[P][j] = 8u * (uint32_t)((iy * Z::TX + ix) * BP + b);
                gxy[P][j] = ((J - 1) * g.m + (I - 1)) * BP + b;
                const int bx0 = axis_block(g, I - 1, g.px), bx1 = axis_block(g, I, g.px);
                const int by0 = axis_block(g, J - 1, g.py), by1 = axis_block(g, J, g.py);
                cxy[P][j] = (I > g.m || J > g.m) ? -2 : (bx0 == bx1 && by0 == by1) ? bx0 + by0 * g.px : -1;
            }
    }
    // grid coordinates of colour element j at parity P (the interface path)
    __device__ __forceinline__ void coords(int x0, int y0, int tid, int P, int j, int& I, int& J) const {
        const int cn = (tid >> Z::LGB) + j * (kZT / BP);
        const int iy = cn / (Z::TX / 2);
        I = x0 + 2 * (cn % (Z::TX / 2)) + ((P + iy) & 1);
        J = y0 + iy;
    }
};

// ===========================================================================
// k_cgz: RBCG Step 11 + Step 5 for 3D grids.
//   step t (plane K = za-1+t arrives: y and p_old tiles with halo):
//     p = y + beta p_old over the whole haloed tile, in place in the y slot;
//     the owned interior nodes are stored to Pnew
//   then sigma += p^T A p on plane K-1 (slots of K-2, K-1, K)
// ===========================================================================
template <int BP, bool FACES>
__global__ void __launch_bounds__(kZT, 1)
    k_cgz(const __grid_constant__ CUtensorMap mY, const __grid_constant__ CUtensorMap mP,
          const __grid_constant__ CGPArgs a, const ZPart zp) {
    using Z = ZGeom<BP>;
    constexpr int NA = Z::NA, NP = Z::DI, DI = Z::DI;
    extern __shared__ __align__(128) double smd[];
    __shared__ __align__(8) uint64_t barA[NA], barP[NP];
    if (a.done && ld_flag(a.done)) return;
    const Geo& g = a.g;
    const int m = g.m, tid = threadIdx.x, b = tid & (BP - 1);
    const double scale = g.scale;
    double* s_th = smd + (NA + NP) * Z::HP;
    for (int t = tid; t < g.Q * BP; t += kZT) s_th[t] = a.theta[t];
    const uint32_t sth = smem_u32(s_th) + 8u * b;      // this lane's column of the theta table
    if (tid == 0) {
        for (int k = 0; k < NA; ++k) mbar_init(&barA[k], 1);
        for (int k = 0; k < NP; ++k) mbar_init(&barP[k], 1);
        mbar_fence_init();
        tma_prefetch_desc(&mY);
        tma_prefetch_desc(&mP);
    }
    const bool act = a.active[b] != 0;
    const double bet = a.beta[b];
    double* const Pnew = a.Pnew;
    const uint32_t sA = smem_u32(smd), sP = sA + 8u * NA * Z::HP;
    const int64_t sz = (int64_t)m * m * BP;
    const int pxy = g.px * g.py;
    constexpr uint32_t HPB = 8u * Z::HP;
    uint32_t G = 0;      // planes loaded by this CTA before the current unit
    double sig = 0.0;
    for (int u = blockIdx.x; u < zp.units; u += gridDim.x) {
        int x0, y0, za, zb;
        zunit(zp, m, u, Z::TX, Z::TY, x0, y0, za, zb);
        const int T = zb - za + 2;                 // planes za-1 .. zb
        ZElems<BP> el;
        el.init(g, x0, y0, tid);
        __syncthreads();                           // previous unit's slots are no longer read
        auto issue = [&](int t) {
            const int K = za - 1 + t;
            const uint32_t q = G + (uint32_t)t;
            const bool in = K >= 1 && K <= m;
            fence_async_smem();
            mbar_expect_tx(&barA[q % NA], in ? HPB : 0u);
            mbar_expect_tx(&barP[q % NP], in ? HPB : 0u);
            if (in) {
                tma_load_4d(smd + (q % NA) * Z::HP, &mY, 0, x0 - 2, y0 - 2, K - 1, &barA[q % NA]);
                tma_load_4d(smd + NA * Z::HP + (q % NP) * Z::HP, &mP, 0, x0 - 2, y0 - 2, K - 1, &barP[q % NP]);
            }
        };
        if (tid == 0)
            for (int t = 0; t < DI && t < T; ++t) issue(t);
        for (int t = 0; t < T; ++t) {
            const int K = za - 1 + t;
            const uint32_t q = G + (uint32_t)t;
            mbar_wait(&barA[q % NA], (q / NA) & 1);
            mbar_wait(&barP[q % NP], (q / NP) & 1);
            const bool in = K >= 1 && K <= m;
            const uint32_t ya = sA + (q % NA) * HPB, pa = sP + (q % NP) * HPB;
            if (in) {
                // interior elements (stored when owned) ...
                const bool own = K >= za && K < zb && act;
                double* pout = Pnew + (int64_t)(K - 1) * sz;
#pragma unroll
                for (int j = 0; j < Z::NE; ++j) {
                    const double v = fma(bet, ldsd(pa + el.h[j]), ldsd(ya + el.h[j]));
                    stsd(ya + el.h[j], v);
                    if (own && el.in(j)) pout[el.gxy[j]] = v;
                }
                // ... and the halo ring (x = 0 or TX+1, or y = 0 or TY+1)
                constexpr int NHALO = (2 * Z::HX + 2 * Z::TY) * BP;
                for (int e = tid; e < NHALO; e += kZT) {
                    const int n = e >> Z::LGB;
                    int hx, hy;
                    if (n < Z::HX) { hx = n; hy = 0; }
                    else if (n < 2 * Z::HX) { hx = n - Z::HX; hy = Z::HY - 1; }
                    else { const int r = n - 2 * Z::HX; hx = (r & 1) ? Z::HX - 1 : 0; hy = 1 + (r >> 1); }
                    const uint32_t o = 8u * (uint32_t)((hy * Z::HX + hx) * BP + b);
                    stsd(ya + o, fma(bet, ldsd(pa + o), ldsd(ya + o)));
                }
            }
            __syncthreads();
            if (tid == 0 && t + DI < T) issue(t + DI);
            // sigma on plane Kc = K - 1 (owned planes za .. zb-1)
            if (t >= 2 && act) {
                const int Kc = K - 1;
                const uint32_t ym = sA + ((q - 2) % NA) * HPB, yc = sA + ((q - 1) % NA) * HPB;
                const bool zm = Kc > 1, zpl = Kc < m;
                const int bz0 = axis_block(g, Kc - 1, g.pz), bz1 = axis_block(g, Kc, g.pz);
                const int bzu = bz0 == bz1 ? bz0 * pxy : -1;
                // all shared-memory loads of the thread's elements first, then the arithmetic
                // (uniform-block nodes), then the rare block-interface nodes out of line
                // per chunk of two elements: the shared-memory loads first, then the arithmetic
                // (uniform-block nodes), then the rare block-interface nodes out of line
#pragma unroll
                for (int c = 0; c < Z::NE; c += 2) {
                    double pp[2], nb[2][6], qv[2];
                    bool slow = false;
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const int j = c + i;
                        const uint32_t o = el.h[j];
                        pp[i] = ldsd(yc + o);
                        nb[i][0] = ldsd(yc + o - 8 * BP);
                        nb[i][1] = ldsd(yc + o + 8 * BP);
                        nb[i][2] = ldsd(yc + o - 8 * Z::HX * BP);
                        nb[i][3] = ldsd(yc + o + 8 * Z::HX * BP);
                        const double zlo = ldsd(ym + o), zhi = ldsd(ya + o);
                        nb[i][4] = zm ? zlo : 0.0;
                        nb[i][5] = zpl ? zhi : 0.0;
                        const bool fast = !FACES && el.cxy[j] >= 0 && bzu >= 0;
                        qv[i] = ldsd(sth + 8u * (uint32_t)((fast ? el.cxy[j] + bzu : 0) * BP));
                        slow |= el.in(j) && !fast;
                    }
#pragma unroll
                    for (int i = 0; i < 2; ++i) qv[i] = stencil_c(scale, qv[i], pp[i], nb[i]);
                    if (slow) {
#pragma unroll
                        for (int i = 0; i < 2; ++i) {
                            const int j = c + i;
                            if (el.in(j) && (FACES || !(el.cxy[j] >= 0 && bzu >= 0))) {
                                const int n = (tid + j * kZT) >> Z::LGB;
                                if (FACES) {      // face coefficients (AMB-23), inline
                                    double k[6];
                                    node_kappa_faces<3>(g, s_th, BP, b, x0 + n % Z::TX, y0 + n / Z::TX, Kc, k);
                                    qv[i] = stencil_apply<3>(g, k, pp[i], nb[i]);
                                } else {
                                    qv[i] = stencil_general(g, s_th, BP, b, x0 + n % Z::TX, y0 + n / Z::TX, Kc,
                                                            pp[i], nb[i][0], nb[i][1], nb[i][2], nb[i][3], nb[i][4],
                                                            nb[i][5]);
                                }
                            }
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 2; ++i)
                        if (el.in(c + i)) sig = fma(pp[i], qv[i], sig);
                }
            }
        }
        G += (uint32_t)T;
    }
    cgp_step5(a, sig);
}

// ===========================================================================
// k_gsz: one red-black half-sweep of colour a.color (eq8, AMB-5/6).
//   step t (plane K = za-1+t arrives): the sweep's nodes of plane K-1 are updated from
//   their neighbours (all of the other colour, unchanged by this half-sweep) and stored.
//   The threads map onto the sweep's colour only (ZColour); LAST also runs the other
//   colour's y^T r, y^T y terms, then RBCG Step 10 in the last CTA.
//   ZERO: the half-sweep from y = 0 (the symmetric two-level preconditioner's pre-sweep,
//   y1 = S*(A, r, 0), first colour): no y tiles are loaded (all neighbours are 0), the
//   sweep's colour gets the same value the loaded zeros would give, the other colour and
//   the frozen lanes get 0 -- the k_fill_batch + half-sweep pair in one pass.
// ===========================================================================
template <int BP, bool LAST, bool FACES, bool ZERO = false>
__global__ void __launch_bounds__(kZT, 1)
    k_gsz(const __grid_constant__ CUtensorMap mY, const __grid_constant__ CUtensorMap mR,
          const __grid_constant__ GSArgs a, const ZPart zp) {
    using Z = ZGeom<BP>;
    using C = ZColour<BP>;
    constexpr int NA = Z::NA, NB = Z::DI + 1, DI = Z::DI, NC = C::NC;
    static_assert(!(ZERO && LAST), "the pre-sweep from zero is never the last half-sweep");
    extern __shared__ __align__(128) double smd[];
    __shared__ __align__(8) uint64_t barA[NA], barB[NB];
    if (a.done && ld_flag(a.done)) return;
    const Geo& g = a.g;
    const int m = g.m, tid = threadIdx.x, b = tid & (BP - 1);
    double* s_th = smd + NA * Z::HP + NB * Z::IP;
    double* s_t6 = s_th + g.Q * BP;            // h^2 / (6 theta): the uniform-block GS weight
    for (int t = tid; t < g.Q * BP; t += kZT) {
        const double v = a.theta[t];
        s_th[t] = v;
        s_t6[t] = g.h2 / (6.0 * v);
    }
    const uint32_t st6 = smem_u32(s_t6) + 8u * b;
    const bool hasr = a.Rhs != nullptr;
    if (tid == 0) {
        for (int k = 0; k < NA; ++k) mbar_init(&barA[k], 1);
        for (int k = 0; k < NB; ++k) mbar_init(&barB[k], 1);
        mbar_fence_init();
        if (!ZERO) tma_prefetch_desc(&mY);
        if (hasr) tma_prefetch_desc(&mR);
    }
    const bool act = a.active[b] != 0;
    const int color = a.color;
    double* const Y = a.Y;
    const uint32_t sA = smem_u32(smd), sB = sA + 8u * NA * Z::HP;
    const int64_t sz = (int64_t)m * m * BP;
    const int pxy = g.px * g.py;
    constexpr uint32_t HPB = 8u * Z::HP, IPB = 8u * Z::IP;
    constexpr double kSixth = 1.0 / 6.0;
    const double rconst = a.rconst;
    uint32_t G = 0;
    double yr = 0.0, yy = 0.0;
    for (int u = blockIdx.x; u < zp.units; u += gridDim.x) {
        int x0, y0, za, zb;
        zunit(zp, m, u, Z::TX, Z::TY, x0, y0, za, zb);
        const int T = zb - za + 2;
        C el;
        el.init(g, x0, y0, tid);
        __syncthreads();
        // plane t: y haloed into A[q % NA]; r interior (owned planes) into B[q % NB]
        auto issue = [&](int t) {
            const int K = za - 1 + t;
            const uint32_t q = G + (uint32_t)t;
            const bool in = !ZERO && K >= 1 && K <= m, own = hasr && K >= za && K < zb;
            fence_async_smem();
            mbar_expect_tx(&barA[q % NA], in ? HPB : 0u);
            mbar_expect_tx(&barB[q % NB], own ? IPB : 0u);
            if (in) tma_load_4d(smd + (q % NA) * Z::HP, &mY, 0, x0 - 2, y0 - 2, K - 1, &barA[q % NA]);
            if (own)
                tma_load_4d(smd + NA * Z::HP + (q % NB) * Z::IP, &mR, 0, x0 - 1, y0 - 1, K - 1, &barB[q % NB]);
        };
        if (tid == 0)
            for (int t = 0; t < DI && t < T; ++t) issue(t);
        for (int t = 0; t < T; ++t) {
            const int K = za - 1 + t;
            const uint32_t q = G + (uint32_t)t;
            mbar_wait(&barA[q % NA], (q / NA) & 1);
            if (t >= 1) mbar_wait(&barB[(q - 1) % NB], ((q - 1) / NB) & 1);   // r of plane K-1
            if (t >= 2 && (act || ZERO)) {
                const int Kc = K - 1;
                const uint32_t ym = sA + ((q - 2) % NA) * HPB, yc = sA + ((q - 1) % NA) * HPB,
                               yp = sA + (q % NA) * HPB;
                const uint32_t rb = sB + ((q - 1) % NB) * IPB;
                const bool zm = Kc > 1, zpl = Kc < m;
                const int bz0 = axis_block(g, Kc - 1, g.pz), bz1 = axis_block(g, Kc, g.pz);
                const int bzu = bz0 == bz1 ? bz0 * pxy : -1;
                double* yo = Y + (int64_t)(Kc - 1) * sz;
                // the sweep colour's column parity in row 0 of this plane tile
                const int P = (color - x0 - y0 - Kc) & 1;
                // loads of the thread's colour elements first, the arithmetic after, the rare
                // block-interface nodes out of line
                double nb[NC][6], rh[NC], v[NC];
                bool slow = false;
#pragma unroll
                for (int j = 0; j < NC; ++j) {
                    const uint32_t o = P ? el.h[1][j] : el.h[0][j];
                    const int cx = P ? el.cxy[1][j] : el.cxy[0][j];
                    rh[j] = hasr ? ldsd(rb + (P ? el.ri[1][j] : el.ri[0][j])) : rconst;
                    if (ZERO) {
#pragma unroll
                        for (int e = 0; e < 6; ++e) nb[j][e] = 0.0;
                    } else {
                        nb[j][0] = ldsd(yc + o - 8 * BP);
                        nb[j][1] = ldsd(yc + o + 8 * BP);
                        nb[j][2] = ldsd(yc + o - 8 * Z::HX * BP);
                        nb[j][3] = ldsd(yc + o + 8 * Z::HX * BP);
                        const double zlo = ldsd(ym + o), zhi = ldsd(yp + o);
                        nb[j][4] = zm ? zlo : 0.0;
                        nb[j][5] = zpl ? zhi : 0.0;
                    }
                    const bool fast = !FACES && cx >= 0 && bzu >= 0;
                    v[j] = ldsd(st6 + 8u * (uint32_t)((fast ? cx + bzu : 0) * BP));
                    slow |= cx != -2 && !fast;
                }
#pragma unroll
                for (int j = 0; j < NC; ++j) {
                    // direct form inside one block: (h^2 b + theta sum nb) / (6 theta)
                    const double sn = ((nb[j][0] + nb[j][1]) + (nb[j][2] + nb[j][3])) + (nb[j][4] + nb[j][5]);
                    v[j] = fma(v[j], rh[j], sn * kSixth);
                }
                if (slow) {
#pragma unroll
                    for (int j = 0; j < NC; ++j) {
                        const int cx = P ? el.cxy[1][j] : el.cxy[0][j];
                        if (cx != -2 && (FACES || !(cx >= 0 && bzu >= 0))) {
                            int I, J;
                            el.coords(x0, y0, tid, P, j, I, J);
                            if (FACES) {          // face coefficients (AMB-23), inline
                                double k[6];
                                node_kappa_faces<3>(g, s_th, BP, b, I, J, Kc, k);
                                v[j] = gs_value<3>(g, k, rh[j], nb[j]);
                            } else {
                                v[j] = gs_general(g, s_th, BP, b, I, J, Kc, rh[j], nb[j][0], nb[j][1], nb[j][2],
                                                  nb[j][3], nb[j][4], nb[j][5]);
                            }
                        }
                    }
                }
#pragma unroll
                for (int j = 0; j < NC; ++j) {
                    if ((P ? el.cxy[1][j] : el.cxy[0][j]) == -2) continue;
                    yo[P ? el.gxy[1][j] : el.gxy[0][j]] = (ZERO && !act) ? 0.0 : v[j];
                    if (LAST) {
                        yr = fma(v[j], rh[j], yr);
                        yy = fma(v[j], v[j], yy);
                    }
                }
                if (ZERO) {           // the other colour stays at the start value 0
#pragma unroll
                    for (int j = 0; j < NC; ++j) {
                        if ((P ? el.cxy[0][j] : el.cxy[1][j]) == -2) continue;
                        yo[P ? el.gxy[0][j] : el.gxy[1][j]] = 0.0;
                    }
                }
                if (LAST) {           // the other colour: unchanged values
#pragma unroll
                    for (int j = 0; j < NC; ++j) {
                        const double w = ldsd(yc + (P ? el.h[0][j] : el.h[1][j]));
                        const double r2 = hasr ? ldsd(rb + (P ? el.ri[0][j] : el.ri[1][j])) : rconst;
                        if ((P ? el.cxy[0][j] : el.cxy[1][j]) == -2) continue;
                        yr = fma(w, r2, yr);
                        yy = fma(w, w, yy);
                    }
                }
            }
            __syncthreads();
            if (tid == 0 && t + DI < T) issue(t + DI);
        }
        G += (uint32_t)T;
    }
    if (LAST) gs_step10(a, yr, yy);
}

// ===========================================================================
// k_xrz: RBCG Steps 6-7 for 3D grids: x += alpha p, r -= alpha A p.
//   step t (plane K = za-1+t of p arrives, with the x and r tiles of plane K-1): plane K-1
//   is updated and stored.  p: haloed ring of kXNA slots; x, r: interior rings of 3 slots;
//   all three are issued 2 planes ahead.
// RES = true: the residual v = b - A y of the symmetric two-level preconditioner's coarse
//   correction (PAPER.md:161 Step 2 form, NEXT(3)): mP maps y (haloed), mR the right-hand
//   side b (a.V == nullptr: the constant a.vconst, no r tiles); v is stored to a.X (a
//   scratch vector), no x tiles are loaded.  Same value as k_proj<MODE_RESID> (c1 - q, the
//   same stencil); W^T v then streams through k_wtr.  Also RBI Step 2 (v = f - A x).
// ===========================================================================
constexpr int kXDI = 2, kXNA = kXDI + 3, kXNR = 3;
template <int BP, bool FACES, bool RES = false>
__global__ void __launch_bounds__(kZT, 1)
    k_xrz(const __grid_constant__ CUtensorMap mP, const __grid_constant__ CUtensorMap mX,
          const __grid_constant__ CUtensorMap mR, const __grid_constant__ ProjArgs a, const ZPart zp) {
    using Z = ZGeom<BP>;
    constexpr int NA = kXNA, NR = kXNR, DI = kXDI;
    extern __shared__ __align__(128) double smd[];
    __shared__ __align__(8) uint64_t barA[NA], barX[NR];
    if (a.done && ld_flag(a.done)) return;
    const Geo& g = a.g;
    const int m = g.m, tid = threadIdx.x, b = tid & (BP - 1);
    const double scale = g.scale;
    double* s_th = smd + NA * Z::HP + 2 * NR * Z::IP;
    for (int t = tid; t < g.Q * BP; t += kZT) s_th[t] = a.theta[t];
    const uint32_t sth = smem_u32(s_th) + 8u * b;
    if (tid == 0) {
        for (int k = 0; k < NA; ++k) mbar_init(&barA[k], 1);
        for (int k = 0; k < NR; ++k) mbar_init(&barX[k], 1);
        mbar_fence_init();
        tma_prefetch_desc(&mP);
        tma_prefetch_desc(&mX);
        tma_prefetch_desc(&mR);
    }
    const bool act = a.active[b] != 0;
    const double al = RES ? 1.0 : a.alpha[b];
    const bool vc = RES && a.V == nullptr;     // constant right-hand side: no r tiles
    double* const X = a.X;
    double* const R = a.R;
    const uint32_t sA = smem_u32(smd), sX = sA + 8u * NA * Z::HP, sR = sX + 8u * NR * Z::IP;
    const int64_t sz = (int64_t)m * m * BP;
    const int pxy = g.px * g.py;
    constexpr uint32_t HPB = 8u * Z::HP, IPB = 8u * Z::IP;
    uint32_t G = 0;
    for (int u = blockIdx.x; u < zp.units; u += gridDim.x) {
        int x0, y0, za, zb;
        zunit(zp, m, u, Z::TX, Z::TY, x0, y0, za, zb);
        const int T = zb - za + 2;
        ZElems<BP> el;
        el.init(g, x0, y0, tid);
        __syncthreads();
        auto issue = [&](int t) {
            const int K = za - 1 + t;
            const uint32_t q = G + (uint32_t)t;
            const bool in = K >= 1 && K <= m, own = K >= za && K < zb;
            fence_async_smem();
            mbar_expect_tx(&barA[q % NA], in ? HPB : 0u);
            mbar_expect_tx(&barX[q % NR], own ? (RES ? (vc ? 0u : 1u) : 2u) * IPB : 0u);
            if (in) tma_load_4d(smd + (q % NA) * Z::HP, &mP, 0, x0 - 2, y0 - 2, K - 1, &barA[q % NA]);
            if (own) {
                if (!RES)
                    tma_load_4d(smd + NA * Z::HP + (q % NR) * Z::IP, &mX, 0, x0 - 1, y0 - 1, K - 1, &barX[q % NR]);
                if (!vc)
                    tma_load_4d(smd + NA * Z::HP + NR * Z::IP + (q % NR) * Z::IP, &mR, 0, x0 - 1, y0 - 1, K - 1,
                                &barX[q % NR]);
            }
        };
        if (tid == 0)
            for (int t = 0; t < DI && t < T; ++t) issue(t);
        for (int t = 0; t < T; ++t) {
            const int K = za - 1 + t;
            const uint32_t q = G + (uint32_t)t;
            mbar_wait(&barA[q % NA], (q / NA) & 1);
            if (t >= 1) mbar_wait(&barX[(q - 1) % NR], ((q - 1) / NR) & 1);   // x, r of plane K-1
            if (t >= 2 && act) {
                const int Kc = K - 1;
                const uint32_t ym = sA + ((q - 2) % NA) * HPB, yc = sA + ((q - 1) % NA) * HPB,
                               yp = sA + (q % NA) * HPB;
                const uint32_t xs = sX + ((q - 1) % NR) * IPB + 8u * tid, rs = sR + ((q - 1) % NR) * IPB + 8u * tid;
                const bool zm = Kc > 1, zpl = Kc < m;
                const int bz0 = axis_block(g, Kc - 1, g.pz), bz1 = axis_block(g, Kc, g.pz);
                const int bzu = bz0 == bz1 ? bz0 * pxy : -1;
                double* const Xc = X + (int64_t)(Kc - 1) * sz;
                double* const Rc = R + (int64_t)(Kc - 1) * sz;
#pragma unroll
                for (int c = 0; c < Z::NE; c += 2) {
                    double pp[2], nb[2][6], qv[2], xv[2], rv[2];
                    bool slow = false;
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const int j = c + i;
                        const uint32_t o = el.h[j];
                        pp[i] = ldsd(yc + o);
                        nb[i][0] = ldsd(yc + o - 8 * BP);
                        nb[i][1] = ldsd(yc + o + 8 * BP);
                        nb[i][2] = ldsd(yc + o - 8 * Z::HX * BP);
                        nb[i][3] = ldsd(yc + o + 8 * Z::HX * BP);
                        const double zlo = ldsd(ym + o), zhi = ldsd(yp + o);
                        nb[i][4] = zm ? zlo : 0.0;
                        nb[i][5] = zpl ? zhi : 0.0;
                        xv[i] = RES ? 0.0 : ldsd(xs + 8u * j * kZT);
                        rv[i] = vc ? a.vconst : ldsd(rs + 8u * j * kZT);
                        const bool fast = !FACES && el.cxy[j] >= 0 && bzu >= 0;
                        qv[i] = ldsd(sth + 8u * (uint32_t)((fast ? el.cxy[j] + bzu : 0) * BP));
                        slow |= el.in(j) && !fast;
                    }
#pragma unroll
                    for (int i = 0; i < 2; ++i) qv[i] = stencil_c(scale, qv[i], pp[i], nb[i]);
                    if (slow) {
#pragma unroll
                        for (int i = 0; i < 2; ++i) {
                            const int j = c + i;
                            if (el.in(j) && (FACES || !(el.cxy[j] >= 0 && bzu >= 0))) {
                                const int n = (tid + j * kZT) >> Z::LGB;
                                if (FACES) {      // face coefficients (AMB-23), inline
                                    double k[6];
                                    node_kappa_faces<3>(g, s_th, BP, b, x0 + n % Z::TX, y0 + n / Z::TX, Kc, k);
                                    qv[i] = stencil_apply<3>(g, k, pp[i], nb[i]);
                                } else {
                                    qv[i] = stencil_general(g, s_th, BP, b, x0 + n % Z::TX, y0 + n / Z::TX, Kc,
                                                            pp[i], nb[i][0], nb[i][1], nb[i][2], nb[i][3], nb[i][4],
                                                            nb[i][5]);
                                }
                            }
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const int j = c + i;
                        if (!el.in(j)) continue;
                        if (RES) {
                            Xc[el.gxy[j]] = rv[i] - qv[i];
                        } else {
                            Xc[el.gxy[j]] = fma(al, pp[i], xv[i]);
                            Rc[el.gxy[j]] = fma(-al, qv[i], rv[i]);
                        }
                    }
                }
            }
            __syncthreads();
            if (tid == 0 && t + DI < T) issue(t + DI);
        }
        G += (uint32_t)T;
    }
}

// ===========================================================================
// k_prolz: the prolongation y0 = W e (+ x_old when accumulating; eq7)
// of a 3D grid with an odd number m of nodes per axis, for the nodes outside the colour of
// the half-sweep that follows (those are overwritten unread, AMB-6).  With m odd the
// red-black colour alternates with the linear node index ((I+J+K) odd <=> i even), so the
// rows needed are every other row of W: a 3-D tensor map views W as [pairs][2][ldw] and
// one copy of box [ldw][1][CH] brings the CH needed rows of a chunk -- half the W bytes,
// dense in shared memory (row stride ldw = npad + 4: conflict-free A fragments).
// Warps own (8-node x 8-query) tiles of a chunk; E fragments stay in registers; two
// accumulator chains per tile (even / odd k-steps).  Persistent grid, NS-slot ring.
// ===========================================================================
struct ProlzArgs {
    int64_t npairs;          // ceil(N / 2)
    int64_t N;
    int Bp, npad, ldw, par;  // par: index parity of the rows prolongated (= skip colour)
    const double* E;         // [npad][Bp]
    const int* active;
    double* Y;               // [N8][Bp]
    int accumulate;
    const int* done;
};
constexpr int kPzNS = 4;
template <int BP>
struct PzShape {
    static constexpr int CH = 128 / (BP / 8);          // node rows per chunk: 16 warp tasks
};
inline size_t prolz_smem_bytes(int Bp, int ldw) {
    return (size_t)kPzNS * (128 / (Bp / 8)) * ldw * 8;
}
template <int BP>
__global__ void __launch_bounds__(kZT, 1) k_prolz(const __grid_constant__ CUtensorMap mW, const ProlzArgs a) {
    constexpr int NKC = kMaxN / 4;           // k-steps, predicated on npad / 4
    constexpr int CH = PzShape<BP>::CH, NBT = BP / 8, NS = kPzNS;
    extern __shared__ __align__(128) double smd[];
    __shared__ __align__(8) uint64_t bars[NS];
    if (a.done && ld_flag(a.done)) return;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ldw = a.ldw;
    const uint32_t slot = (uint32_t)CH * ldw * 8;
    if (tid == 0) {
        for (int k = 0; k < NS; ++k) mbar_init(&bars[k], 1);
        mbar_fence_init();
        tma_prefetch_desc(&mW);
    }
    // this warp's task in every chunk: node tile nt, query tile bt
    const int bt = warp % NBT, nt = warp / NBT;
    const int nk = a.npad >> 2;
    double ef[NKC];
    const double* ecol = a.E + (lane & 3) * BP + bt * 8 + (lane >> 2);
#pragma unroll
    for (int kk = 0; kk < NKC; ++kk) ef[kk] = kk < nk ? __ldg(ecol + (int64_t)kk * 4 * BP) : 0.0;
    const int b = bt * 8 + 2 * (lane & 3);
    const bool act0 = a.active[b] != 0, act1 = a.active[b + 1] != 0;
    __syncthreads();
    const int64_t nchunk = (a.npairs + CH - 1) / CH;
    const int64_t c0 = blockIdx.x, cs = gridDim.x;
    const int64_t mine = c0 < nchunk ? (nchunk - 1 - c0) / cs + 1 : 0;
    auto issue = [&](int64_t k) {            // this CTA's k-th chunk -> slot k % NS
        const int sl = (int)(k % NS);
        fence_async_smem();
        mbar_expect_tx(&bars[sl], slot);
        tma_load_3d(smd + (size_t)sl * CH * ldw, &mW, 0, a.par, (int)((c0 + k * cs) * CH), &bars[sl]);
    };
    if (tid == 0)
        for (int64_t k = 0; k < NS - 1 && k < mine; ++k) issue(k);
    const uint32_t sb = smem_u32(smd) + 8u * ((nt * 8 + (lane >> 2)) * ldw + (lane & 3));
    for (int64_t k = 0; k < mine; ++k) {
        if (tid == 0 && k + NS - 1 < mine) issue(k + NS - 1);
        const int sl = (int)(k % NS);
        mbar_wait(&bars[sl], (uint32_t)((k / NS) & 1));
        const uint32_t wb = sb + (uint32_t)sl * slot;
        double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < NKC; kk += 2) {
            if (kk < nk) dmma_8x8x4(d0, d1, ldsd(wb + 32u * kk), ef[kk]);
            if (kk + 1 < nk) dmma_8x8x4(e0, e1, ldsd(wb + 32u * (kk + 1)), ef[kk + 1]);
        }
        d0 += e0;
        d1 += e1;
        const int64_t pair = (c0 + k * cs) * CH + nt * 8 + (lane >> 2);
        const int64_t i = 2 * pair + a.par;
        if (pair < a.npairs && i < a.N) {
            double* y = a.Y + i * BP + b;
            double2 v = make_double2(d0, d1);
            if (a.accumulate) {
                const double2 o = *reinterpret_cast<const double2*>(y);
                v.x += o.x;
                v.y += o.y;
            }
            if (act0 && act1) *reinterpret_cast<double2*>(y) = v;
            else {
                if (act0) y[0] = v.x;
                if (act1) y[1] = v.y;
            }
        }
        __syncthreads();            // slot sl is reissued NS - 1 chunks later
    }
}

}  // namespace rbs
