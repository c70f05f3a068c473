// api.cu -- C ABI (include/rbs.h) of the B200 batched RB online solver.
//
// Host runtime: context + validation, basis packing and on-device offline
// blocks (eq12c), and the batched RBI / RBCG drivers
// (algorithm1, 260-279 algorithm2).  The iteration loop is
// captured once into a CUDA graph of `graph_chunk` iterations and replayed;
// per-query convergence is tracked on the device (masks + a done flag) and
// the host polls the flag one graph behind, so the loop never stalls on a
// host round trip.  The library allocates no device memory: all buffers are
// carved out of caller-owned storage / workspace.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cudaTypedefs.h>
#include <nccl.h>

#include "../../include/rbs.h"
#include "zmarch.cuh"

using namespace rbs;

struct rbs_ctx {
    int device = 0;
    int num_sms = 148;
    int v2off = 0;   // RBS_DISABLE_V2 debug bits (read once at rbs_create)
    std::string err;
    // operator
    bool has_op = false;
    Geo g{};
    int64_t N8 = 0;
    double fconst = 1.0;
    // basis
    bool has_basis = false;
    int n = 0, npad = 0, ldw = 4;   // ldw = npad + 4: row stride of the packed W
    double* Wi = nullptr;    // [N8][ldw]
    double* dANq = nullptr;  // [Q][npad][npad]
    double* scratch = nullptr;
    std::vector<double> hANq, hfn;  // Q*n*n, n (fn = W^T 1)
    // affine right-hand side f(phi) = sum_r phi_r f_r (rbs_set_rhs_terms; R = 0: constant):
    // borrowed term vectors, their packed copy T [N8][ldt] in the basis storage, and the
    // offline quantities f_{n,r} = W^T f_r (R x n) and the Gram matrix f_r^T f_s (R x R)
    int R = 0, ldt = 0;
    std::vector<const double*> fr;
    double* T = nullptr;
    std::vector<double> hfNr, hG;
    // parameter map (rbs_set_param_map): theta = Ta [1; mu], phi = Pa [1; mu]
    int P = 0;
    std::vector<double> Ta, Pa;      // Q x (P+1) / R x (P+1); empty = identity / all ones
    bool qcomm = false;              // communicator for query sharding (rbs_comm_init)
    // mesh slabs (virtual, one process): 1 = off
    int nslab = 1;
    // mesh slabs over ranks (rbs_dist_init): this rank's slab, NCCL communicator
    bool dist = false;
    int nranks = 1, rank = 0, dz0 = 0, dz1 = 0, dg0 = 0, dg1 = 0, dH = 0;
    ncclComm_t comm = nullptr;
    Geo gglob{};
    // instrumentation / polling
    int64_t launches = 0;
    std::vector<int> last_na;   // active RB dimension per query of the last solve
    int* h_flag = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    // graph cache
    cudaGraphExec_t gexec = nullptr;
    std::string gkey;
    int g_per_chunk = 0;
    // profiling (opts.profile): eager launches bracketed by events
    std::vector<cudaEvent_t> pev;
    double prof_ms[RBS_K_NCLASS] = {0};
    int64_t prof_cnt[RBS_K_NCLASS] = {0};
};

namespace {

rbs_status fail(rbs_ctx* c, rbs_status s, const std::string& msg) {
    if (c) c->err = msg;
    return s;
}

#define CK(call)                                                                            \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return fail(ctx, RBS_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define CKL()                                                                               \
    do {                                                                                    \
        cudaError_t e_ = cudaGetLastError();                                                \
        if (e_ != cudaSuccess)                                                              \
            return fail(ctx, RBS_E_CUDA, std::string("launch: ") + cudaGetErrorString(e_)); \
    } while (0)

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }
// packed W row stride: npad + 4 doubles = 2(npad+4) words = 8 or 24 mod 32, so the
// 4-row DMMA fragment reads of a half-warp hit distinct shared-memory banks
inline int w_ld(int npad) { return npad + 4; }
inline int pow2_batch(int B) {
    int p = 8;
    while (p < B) p <<= 1;
    return p;
}
inline int ilog2(int v) {
    int l = 0;
    while ((1 << l) < v) ++l;
    return l;
}

// number of CTAs of the projection pass: depends on N only (determinism)
inline int proj_ctas(const Geo& g) {
    int64_t groups = (g.N + 3) / 4;
    int64_t c = (groups + 31) / 32;
    return (int)std::max<int64_t>(1, std::min<int64_t>(c, 296));
}
inline int flat_ctas(const Geo& g) {
    int64_t c = (g.N + 63) / 64;
    return (int)std::max<int64_t>(1, std::min<int64_t>(c, 296));
}
// strip partition of the 2D row-marching passes (march.cuh): ~one CTA per SM
inline int march_tx(int Bp) { return Bp <= 32 ? 32 : 16; }
inline MarchPart march_part(const Geo& g, int TX, int sms) {
    MarchPart p;
    p.nsx = (g.m + TX - 1) / TX;
    int nsy = std::max(1, sms / p.nsx);
    p.rows_per_seg = std::max(8, (g.m + nsy - 1) / nsy);
    p.nsy = (g.m + p.rows_per_seg - 1) / p.rows_per_seg;
    return p;
}
// columns of the per-CTA partial buffers of the flat / march passes
inline int part_ctas(const Geo& g, int sms) {
    const MarchPart a = march_part(g, 32, sms), b = march_part(g, 16, sms), c = march_part(g, 24, sms);
    const MarchPart d = march_part(g, 32, 2 * sms);    // k_cgp2: 2 CTAs per SM
    return std::max(std::max(flat_ctas(g), c.nsx * c.nsy),
                    std::max(std::max(a.nsx * a.nsy, b.nsx * b.nsy), d.nsx * d.nsy));
}
inline int grid_for(int64_t work, int per, int cap) {
    int64_t c = (work + per - 1) / per;
    return (int)std::max<int64_t>(1, std::min<int64_t>(c, cap));
}

// bump allocator over a caller buffer
struct Carve {
    char* base;
    size_t off = 0;
    explicit Carve(void* b) : base((char*)b) {}
    template <class T>
    T* take(size_t count) {
        off = (off + 255) & ~size_t(255);
        T* p = base ? (T*)(base + off) : nullptr;
        off += count * sizeof(T);
        return p;
    }
};

size_t proj_smem(const Geo& g, int Bp, int npad) {
    const int nlc = 8 / (Bp / 8) > 0 ? 8 / (Bp / 8) : 1;
    return (size_t)(g.Q * Bp + Bp + nlc * (npad + 1) * Bp) * 8 + (size_t)Bp * 4 + 16;
}
size_t flat_smem(const Geo& g, int Bp) { return (size_t)g.Q * Bp * 8 + (size_t)Bp * 4 + 16; }

template <int MODE>
void launch_proj(const Geo& g, int grid, size_t smem, cudaStream_t st, const ProjArgs& a) {
    if (g.dim == 2) k_proj<MODE, 2><<<grid, kThreads, smem, st>>>(a);
    else k_proj<MODE, 3><<<grid, kThreads, smem, st>>>(a);
}

// launch with programmatic dependent launch (the 2D iteration passes, rbs_internal.cuh
// pdl_wait / pdl_trigger): the pass may start its prologue while the previous drains
template <typename... P, typename... A>
void launch_k(bool pdl, void (*k)(P...), unsigned grid, unsigned block, size_t smem, cudaStream_t st, A... args) {
    if (!pdl) {
        k<<<grid, block, smem, st>>>(args...);
        return;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, args...);
}

// k_smooth2 dynamic shared memory cap: 227 KB per CTA minus its static part
constexpr int kSmooth2MaxDyn = 225 * 1024;
template <int BP, bool R, int TX, int WR>
void set_attrs_smooth2() {
    const int mx = kSmooth2MaxDyn;
    cudaFuncSetAttribute(k_smooth2<BP, 0, R, TX, WR>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_smooth2<BP, 1, R, TX, WR>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_smooth2<BP, 2, R, TX, WR>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_smooth2<BP, 3, R, TX, WR>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
}
template <int BP>
void set_attrs_v2() {
    const int mx = 214 * 1024;
    if (BP == 32) {
        cudaFuncSetAttribute(k_smooth2<32, 3, true, 32, 3, 10>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmooth2MaxDyn);
        cudaFuncSetAttribute(k_smooth2<32, 3, true, 32, 2, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmooth2MaxDyn);
    }
    set_attrs_smooth2<BP, false, 32, 3>();
    set_attrs_smooth2<BP, true, 32, 3>();
    set_attrs_smooth2<BP, false, 32, 2>();
    set_attrs_smooth2<BP, true, 32, 2>();
    set_attrs_smooth2<BP, false, 24, 3>();
    set_attrs_smooth2<BP, true, 24, 3>();
    cudaFuncSetAttribute(k_cgp2<BP>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_cgp2<BP>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_resid2<BP, 0, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_resid2<BP, 1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_resid2<BP, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    cudaFuncSetAttribute(k_resid2<BP, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
}
template <int BP, bool R, int TX, int WR>
void launch_smooth2t(int S, int grid, size_t smem, cudaStream_t st, const SmoothMarchArgs& a, bool pdl) {
    switch (S) {
        case 0: launch_k(pdl, k_smooth2<BP, 0, R, TX, WR>, grid, kMT, smem, st, a); break;
        case 1: launch_k(pdl, k_smooth2<BP, 1, R, TX, WR>, grid, kMT, smem, st, a); break;
        case 2: launch_k(pdl, k_smooth2<BP, 2, R, TX, WR>, grid, kMT, smem, st, a); break;
        default: launch_k(pdl, k_smooth2<BP, 3, R, TX, WR>, grid, kMT, smem, st, a); break;
    }
}
// variant: 0 = strip 32 / W ring 3, 1 = strip 32 / W ring 2, 2 = strip 24 / W ring 3
template <int BP>
void launch_smooth2(int var, int S, int grid, size_t smem, cudaStream_t st, const SmoothMarchArgs& a, int v2off) {
    const bool pdl = !(v2off & 16384);
    if (BP == 32 && S == 3 && a.Rhs && a.npad == 40 && var == 0 && !(v2off & 1024)) {
        launch_k(pdl, k_smooth2<32, 3, true, 32, 3, 10>, grid, kMT, smem, st, a);     // n = 33..40 (c2)
        return;
    }
    if (BP == 32 && S == 3 && a.Rhs && a.npad == 64 && var == 1 && !(v2off & 1024)) {
        launch_k(pdl, k_smooth2<32, 3, true, 32, 2, 16>, grid, kMT, smem, st, a);     // n = 57..64 (c3)
        return;
    }
    if (var == 0) {
        if (a.Rhs) launch_smooth2t<BP, true, 32, 3>(S, grid, smem, st, a, pdl);
        else launch_smooth2t<BP, false, 32, 3>(S, grid, smem, st, a, pdl);
    } else if (var == 1) {
        if (a.Rhs) launch_smooth2t<BP, true, 32, 2>(S, grid, smem, st, a, pdl);
        else launch_smooth2t<BP, false, 32, 2>(S, grid, smem, st, a, pdl);
    } else {
        if (a.Rhs) launch_smooth2t<BP, true, 24, 3>(S, grid, smem, st, a, pdl);
        else launch_smooth2t<BP, false, 24, 3>(S, grid, smem, st, a, pdl);
    }
}
template <int BP, int PF>
void launch_resid2(int md, int grid, size_t smem, cudaStream_t st, const ResidMarchArgs& r, bool pdl) {
    if (md == 0) launch_k(pdl, k_resid2<BP, 0, PF>, grid, kMT, smem, st, r);
    else launch_k(pdl, k_resid2<BP, 1, PF>, grid, kMT, smem, st, r);
}

// ---- TMA tensor maps of the 3D z-plane marches (zmarch.cuh) -------------------
// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link);
// resolved once, immutable afterwards
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        else
            cudaGetLastError();
    });
    return fn;
}
// 4-D map of a node-major batch vector v[m][m][m][Bp] (dims innermost first: lane, I, J, K)
// with box [Bp][bx][by][1]; out-of-range elements of a box are zero-filled
bool zmap(CUtensorMap* map, const double* v, const Geo& g, int Bp, int bx, int by) {
    auto enc = tmap_encoder();
    if (!enc) return false;
    const cuuint64_t m = (cuuint64_t)g.m;
    cuuint64_t dims[4] = {(cuuint64_t)Bp, m, m, (cuuint64_t)g.mz};
    cuuint64_t strides[3] = {(cuuint64_t)Bp * 8, m * Bp * 8, m * m * Bp * 8};
    cuuint32_t box[4] = {(cuuint32_t)Bp, (cuuint32_t)bx, (cuuint32_t)by, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(v), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// z-march work partition: tiles x z-segments; the segment count minimises
// rounds x (planes per unit + 2 halo planes) over a persistent grid of `grid` CTAs
ZPart z_part(const Geo& g, int TX, int TY, int grid) {
    ZPart p{};
    p.ntx = (g.m + TX - 1) / TX;
    p.nty = (g.m + TY - 1) / TY;
    const int tiles = p.ntx * p.nty;
    int64_t best = -1;
    for (int nz = 1; nz <= std::min(g.m, 64); ++nz) {
        const int zlen = (g.m + nz - 1) / nz, nze = (g.m + zlen - 1) / zlen;
        const int64_t units = (int64_t)tiles * nze, rounds = (units + grid - 1) / grid;
        const int64_t cost = rounds * (zlen + 2);
        if (best < 0 || cost < best) {
            best = cost;
            p.nz = nze;
            p.zlen = zlen;
            p.units = (int)units;
        }
    }
    return p;
}
// dynamic shared memory of the z-march kernels: rings + theta table, capped so the
// kernels' static shared memory (barriers, LAST epilogue buffers, ~9 KB) still fits 227 KB
constexpr size_t kZMaxDyn = 217 * 1024;
template <int BP>
void set_attrs_z() {
    auto cap = [](size_t b) { return (int)std::min(b, kZMaxDyn); };
    const int c0 = cap(zsmem_bytes<BP>(0, RBS_MAX_Q)), c1 = cap(zsmem_bytes<BP>(1, RBS_MAX_Q)),
              c2 = cap(zsmem_bytes<BP>(2, RBS_MAX_Q));
    cudaFuncSetAttribute(k_cgz<BP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, c0);
    cudaFuncSetAttribute(k_cgz<BP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, c0);
    cudaFuncSetAttribute(k_gsz<BP, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, c1);
    cudaFuncSetAttribute(k_gsz<BP, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, c1);
    cudaFuncSetAttribute(k_gsz<BP, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, c1);
    cudaFuncSetAttribute(k_gsz<BP, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, c1);
    cudaFuncSetAttribute(k_gsz<BP, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, c1);
    cudaFuncSetAttribute(k_gsz<BP, false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, c1);
    cudaFuncSetAttribute(k_xrz<BP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, c2);
    cudaFuncSetAttribute(k_xrz<BP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, c2);
    cudaFuncSetAttribute(k_xrz<BP, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, c2);
    cudaFuncSetAttribute(k_xrz<BP, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, c2);
    cudaFuncSetAttribute(k_prolz<BP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kZMaxDyn);
}

// cudaFuncSetAttribute applies to the current device only: once per device
std::mutex g_attr_mu;
bool g_attr_done[64] = {false};
void set_attrs(int dev) {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    if (dev < 0 || dev >= 64 || g_attr_done[dev]) return;
    const int big = 200 * 1024;
    cudaFuncSetAttribute(k_proj<MODE_CG, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_proj<MODE_CG, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_proj<MODE_RESID, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_proj<MODE_RESID, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_proj<MODE_PLAIN, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_proj<MODE_PLAIN, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_gs<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_gs<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_gs<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_gs<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_cgp<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    // 227 KB per CTA in total: leave room for the kernels' static shared memory
    cudaFuncSetAttribute(k_smooth_march<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    cudaFuncSetAttribute(k_smooth_march<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    cudaFuncSetAttribute(k_resid_march<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    cudaFuncSetAttribute(k_resid_march<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    cudaFuncSetAttribute(k_cgp<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(k_wtr<8, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    cudaFuncSetAttribute(k_wtr<16, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    cudaFuncSetAttribute(k_wtr<32, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    cudaFuncSetAttribute(k_wtr<8, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    cudaFuncSetAttribute(k_wtr<16, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    cudaFuncSetAttribute(k_wtr<32, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    set_attrs_v2<8>();
    set_attrs_v2<16>();
    set_attrs_v2<32>();
    set_attrs_z<8>();
    set_attrs_z<16>();
    set_attrs_z<32>();
    g_attr_done[dev] = true;
}

// storage of a basis of dimension n
struct BasisLayout {
    double *Wi, *ANq, *Z, *part, *rows, *T;
    size_t bytes;
};
// terms: packed row stride (R rounded to 8, + 4 like W)
inline int terms_ld(int R) { return R > 0 ? (int)round_up(R, 8) + 4 : 0; }
BasisLayout basis_layout(const rbs_ctx* c, int n, void* base) {
    const int npad = (int)round_up(n, 8);
    const int rpad = (int)round_up(c->R, 8), mpad = std::max(npad, rpad);
    Carve cv(base);
    BasisLayout L;
    L.Wi = cv.take<double>((size_t)c->N8 * w_ld(npad));
    // offline blocks [Q][npad][npad], then f_n (npad): the region rbs_broadcast_basis sends
    L.ANq = cv.take<double>((size_t)c->g.Q * npad * npad + npad + 8);
    L.Z = cv.take<double>((size_t)c->N8 * 8);
    L.part = cv.take<double>((size_t)8 * (mpad + 1) * proj_ctas(c->g));
    L.rows = cv.take<double>((size_t)8 * (mpad + 1));
    L.T = c->R > 0 ? cv.take<double>((size_t)c->N8 * terms_ld(c->R)) : nullptr;
    L.bytes = cv.off + 256;
    return L;
}

// solve workspace
struct SolveLayout {
    double *X, *X2, *R, *P0, *P1, *Y, *F, *Xout, *T, *Rold;
    double *theta, *fproj, *L, *Ainv, *E, *a_n, *partP, *partF, *phi;
    double *alpha, *beta, *rho, *rr, *fnorm, *relres, *hist, *rho_prev;
    int *active, *status, *its, *pivot, *ints, *na;
    size_t bytes;
};
SolveLayout solve_layout(const rbs_ctx* c, int B, const rbs_solve_opts* o, bool rhs, void* base) {
    const int Bp = pow2_batch(B), npad = c->npad;
    const size_t vec = (size_t)c->N8 * Bp;
    const int nct = proj_ctas(c->g), nctf = part_ctas(c->g, c->num_sms);
    Carve cv(base);
    SolveLayout L{};
    const bool cg = o->method == RBS_RBCG;
    L.X = cv.take<double>(vec);
    L.X2 = (!cg && c->g.dim == 2 && o->smoother != RBS_SMOOTH_JACOBI) ? cv.take<double>(vec)
                                                                        : nullptr;   // RBI ping-pong (march)
    // Jacobi ping-pong; 3D z-march residual-projection (k_xrz<RES> + k_wtr) of the symmetric
    // two-level preconditioner (v = r - A y1) and of RBI (v = f - A x)
    L.T = (o->smoother == RBS_SMOOTH_JACOBI ||
           (c->g.dim == 3 && (!cg || o->precond == RBS_PRECOND_SYM)))
              ? cv.take<double>(vec) : nullptr;
    L.R = cg ? cv.take<double>(vec) : nullptr;
    L.P0 = cg ? cv.take<double>(vec) : nullptr;
    L.P1 = cg ? cv.take<double>(vec) : nullptr;
    L.Y = cg ? cv.take<double>(vec) : nullptr;
    L.F = rhs ? cv.take<double>(vec) : nullptr;
    L.Rold = (cg && o->beta_rule == RBS_BETA_PR) ? cv.take<double>(vec) : nullptr;   // r_k (PR beta)
    L.Xout = o->x_location == RBS_MEM_HOST ? cv.take<double>((size_t)B * c->g.N) : nullptr;
    L.theta = cv.take<double>((size_t)c->g.Q * Bp);
    L.phi = c->R > 0 ? cv.take<double>((size_t)Bp * c->R) : nullptr;
    L.fproj = cv.take<double>((size_t)Bp * (npad + 1));
    L.L = cv.take<double>((size_t)Bp * npad * npad + 8);
    L.Ainv = cv.take<double>((size_t)Bp * npad * npad + 8);
    L.E = cv.take<double>((size_t)std::max(npad, 8) * Bp);
    L.a_n = cv.take<double>((size_t)Bp * npad + 8);
    const MarchPart rp = march_part(c->g, kRmTX, c->num_sms);
    L.partP = cv.take<double>((size_t)Bp * (npad + 1) * std::max(nct, rp.nsx * rp.nsy));
    L.partF = cv.take<double>((size_t)Bp * 2 * nctf);
    L.alpha = cv.take<double>(Bp);
    L.beta = cv.take<double>(Bp);
    L.rho = cv.take<double>(Bp);
    L.rr = cv.take<double>(Bp);
    L.fnorm = cv.take<double>(Bp);
    L.relres = cv.take<double>(Bp);
    L.rho_prev = cv.take<double>(Bp);
    L.hist = o->record_history ? cv.take<double>((size_t)Bp * (o->max_iter + 1)) : nullptr;
    L.active = cv.take<int>(Bp);
    L.status = cv.take<int>(Bp);
    L.its = cv.take<int>(Bp);
    L.pivot = cv.take<int>(Bp);
    L.ints = cv.take<int>(8);
    L.na = cv.take<int>(Bp);
    L.bytes = cv.off + 256;
    return L;
}

// active RB dimension (opts.n_active, gamma rule): leading-block reduced solves (AMB-19)
void set_active_dim(SolveState& S, int* na, const rbs_solve_opts* o, int n) {
    S.na = na;
    S.na0 = (o->n_active > 0 && o->n_active < n) ? o->n_active : n;
    S.gamma = o->method == RBS_RBCG ? o->gamma : 0.0;
    S.tri = (S.na0 < n || S.gamma > 0.0) ? 1 : 0;
}

rbs_status check_opts(rbs_ctx* ctx, const rbs_solve_opts* o) {
    if (!o) return fail(ctx, RBS_E_ARG, "opts is NULL");
    if (o->method != RBS_RBI && o->method != RBS_RBCG) return fail(ctx, RBS_E_ARG, "bad method");
    if (o->smoother != RBS_SMOOTH_SYM_RBGS && o->smoother != RBS_SMOOTH_FWD_RBGS &&
        o->smoother != RBS_SMOOTH_JACOBI)
        return fail(ctx, RBS_E_UNSUPPORTED, "smoother must be SYM_RBGS, FWD_RBGS or JACOBI");
    if (o->smoother == RBS_SMOOTH_JACOBI && !(o->omega > 0.0 && o->omega < 2.0))
        return fail(ctx, RBS_E_ARG, "Jacobi damping omega must be in (0, 2)");
    if (o->sweeps < 0 || o->sweeps > 64) return fail(ctx, RBS_E_ARG, "sweeps out of range");
    if (o->max_iter < 0) return fail(ctx, RBS_E_ARG, "max_iter < 0");
    if (!(o->tol >= 0.0)) return fail(ctx, RBS_E_ARG, "tol must be >= 0");
    if (o->x_location != RBS_MEM_DEVICE && o->x_location != RBS_MEM_HOST)
        return fail(ctx, RBS_E_ARG, "bad x_location");
    if (o->graph_chunk < 2 || (o->graph_chunk & 1)) return fail(ctx, RBS_E_ARG, "graph_chunk must be even >= 2");
    if (o->n_active < 0 || o->n_active > ctx->n) return fail(ctx, RBS_E_ARG, "n_active out of range 0..n");
    if (!(o->gamma >= 0.0)) return fail(ctx, RBS_E_ARG, "gamma must be >= 0");
    if (o->gamma > 0.0 && o->method != RBS_RBCG) return fail(ctx, RBS_E_ARG, "gamma rule is RBCG only");
    if (o->precond != RBS_PRECOND_POST && o->precond != RBS_PRECOND_SYM) return fail(ctx, RBS_E_ARG, "bad precond");
    if (o->beta_rule != RBS_BETA_FR && o->beta_rule != RBS_BETA_PR) return fail(ctx, RBS_E_ARG, "bad beta_rule");
    if ((o->precond != RBS_PRECOND_POST || o->beta_rule != RBS_BETA_FR) && o->method != RBS_RBCG)
        return fail(ctx, RBS_E_ARG, "precond / beta_rule are RBCG options");
    if ((o->precond != RBS_PRECOND_POST || o->beta_rule != RBS_BETA_FR) && (ctx->dist || ctx->nslab > 1))
        return fail(ctx, RBS_E_UNSUPPORTED, "mesh slabs: precond / beta_rule variants not supported");
    return RBS_OK;
}

// half-sweep colour sequence: symmetric sweep = R,B,B,R; repeated half-sweeps
// of one colour are bitwise no-ops (AMB-6) and are dropped.
std::vector<int> color_seq(int smoother, int sweeps) {
    std::vector<int> s;
    for (int k = 0; k < sweeps; ++k) {
        const int sym[4] = {0, 1, 1, 0}, fwd[2] = {0, 1};
        const int* seq = smoother == RBS_SMOOTH_SYM_RBGS ? sym : fwd;
        const int len = smoother == RBS_SMOOTH_SYM_RBGS ? 4 : 2;
        for (int t = 0; t < len; ++t)
            if (s.empty() || s.back() != seq[t]) s.push_back(seq[t]);
    }
    return s;
}

}  // namespace

namespace {
// affine right-hand side terms (rbs_set_rhs_terms) of a loaded basis: packed copy T,
// f_{n,r} = W^T f_r and the Gram matrix (rbs_load_basis, rbs_broadcast_basis)
rbs_status terms_offline(rbs_ctx* ctx, const BasisLayout& L, cudaStream_t st) {
    // affine right-hand side terms (rbs_set_rhs_terms): packed copy T, f_{n,r} = W^T f_r
    // (eq12c) and the Gram matrix f_r^T f_s for ||f(mu)||^2 = phi^T G phi --
    // both by the projection pass, 8 terms at a time (a term chunk is the projected vector V;
    // for G, T itself plays W)
    const Geo& g = ctx->g;
    const int n = ctx->n, npad = ctx->npad;
    ctx->T = L.T;
    ctx->ldt = terms_ld(ctx->R);
    ctx->hfNr.assign((size_t)ctx->R * n, 0.0);
    ctx->hG.assign((size_t)ctx->R * ctx->R, 0.0);
    if (ctx->R > 0) {
        TermPtrs tp{};
        for (int r = 0; r < ctx->R; ++r) tp.p[r] = ctx->fr[r];
        k_pack_terms<<<grid_for(ctx->N8 * ctx->ldt, 256, 4 * ctx->num_sms * 8), 256, 0, st>>>(
            tp, ctx->R, g.N, ctx->N8, ctx->ldt, L.T);
        CKL();
        const int nct = proj_ctas(g), rpad = (int)round_up(ctx->R, 8);
        std::vector<double> rows((size_t)8 * (std::max(npad, rpad) + 1));
        for (int r0 = 0; r0 < ctx->R; r0 += 8) {
            k_take8<<<grid_for(ctx->N8 * 8, 256, 4 * ctx->num_sms * 8), 256, 0, st>>>(L.T, ctx->ldt, r0, ctx->R,
                                                                                   ctx->N8, L.Z);
            CKL();
            for (int pass = 0; pass < 2; ++pass) {     // 0: W^T f_r, 1: T^T f_r (Gram)
                const int np_ = pass == 0 ? npad : rpad;
                if (np_ == 0) continue;
                ProjArgs a{};
                a.g = g; a.Bp = 8; a.npad = np_; a.nct = nct; a.ngroups = (g.N + 3) / 4;
                a.ldw = pass == 0 ? ctx->ldw : ctx->ldt;
                a.W = pass == 0 ? L.Wi : L.T; a.V = L.Z; a.part = L.part;
                launch_proj<MODE_PLAIN>(g, nct, proj_smem(g, 8, np_), st, a);
                CKL();
                k_reduce_rows<<<8, 128, 0, st>>>(L.part, np_ + 1, nct, L.rows);
                CKL();
                CK(cudaMemcpyAsync(rows.data(), L.rows, (size_t)8 * (np_ + 1) * 8, cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                for (int k = 0; k < 8 && r0 + k < ctx->R; ++k) {
                    const int r = r0 + k;
                    if (pass == 0)
                        for (int j = 0; j < n; ++j) ctx->hfNr[(size_t)r * n + j] = rows[(size_t)k * (np_ + 1) + j];
                    else
                        for (int j = 0; j < ctx->R; ++j) ctx->hG[(size_t)j * ctx->R + r] = rows[(size_t)k * (np_ + 1) + j];
                }
            }
        }
        for (int i = 0; i < ctx->R; ++i)          // exactly symmetric (i <= j mirrored)
            for (int j = 0; j < i; ++j) ctx->hG[(size_t)i * ctx->R + j] = ctx->hG[(size_t)j * ctx->R + i];
    }
    return RBS_OK;
}

}  // namespace

#include "slab.inc.cu"

// ============================================================================
extern "C" {

int rbs_version(void) { return RBS_VERSION; }

const char* rbs_status_string(rbs_status s) {
    switch (s) {
        case RBS_OK: return "RBS_OK";
        case RBS_E_ARG: return "RBS_E_ARG";
        case RBS_E_DIM: return "RBS_E_DIM";
        case RBS_E_STATE: return "RBS_E_STATE";
        case RBS_E_NOT_SPD: return "RBS_E_NOT_SPD";
        case RBS_E_CUDA: return "RBS_E_CUDA";
        case RBS_E_NOMEM: return "RBS_E_NOMEM";
        case RBS_E_UNSUPPORTED: return "RBS_E_UNSUPPORTED";
    }
    return "RBS_E_UNKNOWN";
}

rbs_status rbs_create(int cuda_device, rbs_ctx** out) {
    rbs_ctx* ctx = nullptr;
    if (!out) return RBS_E_ARG;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || cuda_device < 0 || cuda_device >= count)
        return RBS_E_CUDA;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, cuda_device) != cudaSuccess) return RBS_E_CUDA;
    if (prop.major != 10) return RBS_E_UNSUPPORTED;
    if (cudaSetDevice(cuda_device) != cudaSuccess) return RBS_E_CUDA;
    ctx = new rbs_ctx();
    ctx->device = cuda_device;
    ctx->num_sms = prop.multiProcessorCount;
    if (cudaHostAlloc(&ctx->h_flag, 4 * sizeof(int), cudaHostAllocDefault) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev[1], cudaEventDisableTiming) != cudaSuccess) {
        delete ctx;
        return RBS_E_CUDA;
    }
    set_attrs(cuda_device);
    const char* dv2 = getenv("RBS_DISABLE_V2");   // debug / A-B bits, read once per context
    ctx->v2off = dv2 ? atoi(dv2) : 0;
    *out = ctx;
    return RBS_OK;
}

void rbs_destroy(rbs_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    if (ctx->h_flag) cudaFreeHost(ctx->h_flag);
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : ctx->pev) cudaEventDestroy(e);
    delete ctx;
}

const char* rbs_last_error(const rbs_ctx* ctx) { return ctx ? ctx->err.c_str() : "NULL context"; }

int64_t rbs_last_launch_count(const rbs_ctx* ctx) { return ctx ? ctx->launches : -1; }

#ifdef RBS_CLK
// instrumented builds: per-warp cycle accounting of k_smooth2 (march2.cuh), read and reset
int rbs_debug_s2clk(unsigned long long* host) {
    if (cudaMemcpyFromSymbol(host, g_s2clk, sizeof(g_s2clk)) != cudaSuccess) return 1;
    if (cudaMemcpyFromSymbol(host + 148 * 16 * 6, g_s2t, sizeof(g_s2t)) != cudaSuccess) return 1;
    static unsigned long long zero[148 * 16 * 6];
    return cudaMemcpyToSymbol(g_s2clk, zero, sizeof(zero)) != cudaSuccess;
}
#endif

rbs_status rbs_last_n_active(const rbs_ctx* ctx, int* out) {
    if (!ctx || !out) return RBS_E_ARG;
    for (size_t b = 0; b < ctx->last_na.size(); ++b) out[b] = ctx->last_na[b];
    return RBS_OK;
}

rbs_status rbs_last_profile(const rbs_ctx* ctx, double* ms_total, int64_t* launches) {
    if (!ctx || !ms_total || !launches) return RBS_E_ARG;
    for (int k = 0; k < RBS_K_NCLASS; ++k) {
        ms_total[k] = ctx->prof_ms[k];
        launches[k] = ctx->prof_cnt[k];
    }
    return RBS_OK;
}

const char* rbs_kernel_class_name(int k) {
    static const char* names[RBS_K_NCLASS] = {"k_cgp", "k_alpha", "k_proj", "k_reduce_solve",
                                              "k_prolong", "k_gs", "k_beta"};
    return (k >= 0 && k < RBS_K_NCLASS) ? names[k] : "";
}

rbs_status rbs_set_operator_blocks(rbs_ctx* ctx, int dim, const int64_t m[3], const int blocks[3]) {
    if (!ctx) return RBS_E_ARG;
    ctx->err.clear();
    if (!m || !blocks) return fail(ctx, RBS_E_ARG, "m/blocks is NULL");
    if (dim != 2 && dim != 3) return fail(ctx, RBS_E_DIM, "dim must be 2 or 3");
    for (int d = 0; d < dim; ++d) {
        if (m[d] != m[0]) return fail(ctx, RBS_E_UNSUPPORTED, "m must be equal on every axis");
        if (blocks[d] < 1 || blocks[d] > 16) return fail(ctx, RBS_E_DIM, "blocks must be in 1..16");
    }
    if (m[0] < 1 || m[0] > 65535) return fail(ctx, RBS_E_DIM, "m must be in 1..65535");
    const int64_t N = dim == 2 ? m[0] * m[0] : m[0] * m[0] * m[0];
    if (N >= (int64_t(1) << 31)) return fail(ctx, RBS_E_DIM, "N too large (>= 2^31)");
    Geo g{};
    g.dim = dim;
    g.m = (int)m[0];
    g.N = N;
    g.px = blocks[0];
    g.py = blocks[1];
    g.pz = dim == 3 ? blocks[2] : 1;
    g.Q = g.px * g.py * g.pz;
    if (g.Q > RBS_MAX_Q) return fail(ctx, RBS_E_DIM, "Q > RBS_MAX_Q");
    g.fm = make_fastdiv((uint32_t)g.m);
    g.f2m1 = make_fastdiv((uint32_t)(2 * (g.m + 1)));
    g.scale = (double)(g.m + 1) * (double)(g.m + 1);
    g.h2 = 1.0 / g.scale;
    g.kofs = 0;
    g.mz = g.m;
    g.own_lo = 0;
    g.own_hi = g.m;
    ctx->g = g;
    ctx->gglob = g;
    ctx->N8 = round_up(N, 8);
    ctx->has_op = true;
    ctx->has_basis = false;
    ctx->R = 0;                 // a new operator drops the affine rhs terms and the parameter map
    ctx->fr.clear();
    ctx->T = nullptr;
    ctx->P = 0;
    ctx->Ta.clear();
    ctx->Pa.clear();
    ctx->dist = false;
    ctx->nslab = 1;
    return RBS_OK;
}

rbs_status rbs_set_operator_faces(rbs_ctx* ctx, int dim, int64_t m, int Q, const double* faces_dev) {
    if (!ctx) return RBS_E_ARG;
    ctx->err.clear();
    if (!faces_dev) return fail(ctx, RBS_E_ARG, "faces_dev is NULL");
    if (Q < 1 || Q > RBS_MAX_Q) return fail(ctx, RBS_E_DIM, "Q must be in 1..RBS_MAX_Q");
    if ((int64_t)dim * (m + 1) * (dim == 3 ? m * m : m) >= (int64_t(1) << 32))
        return fail(ctx, RBS_E_DIM, "face arrays too large (dim * nf >= 2^32)");
    const int64_t mm[3] = {m, m, m};
    const int ones[3] = {1, 1, 1};
    const rbs_status st = rbs_set_operator_blocks(ctx, dim, mm, ones);
    if (st != RBS_OK) return st;
    ctx->g.Q = Q;
    ctx->g.faces = faces_dev;
    ctx->g.nf = (m + 1) * (dim == 3 ? m * m : m);
    ctx->gglob = ctx->g;
    return RBS_OK;
}

rbs_status rbs_affine_rhs(rbs_ctx* ctx, int B, int R, const double* phi_host, const double* terms_dev,
                          double* out_dev, void* stream) {
    if (!ctx) return RBS_E_ARG;
    ctx->err.clear();
    if (!ctx->has_op) return fail(ctx, RBS_E_STATE, "no operator");
    if (B < 1 || R < 1 || R > RBS_MAX_R) return fail(ctx, RBS_E_DIM, "B >= 1 and 1 <= R <= RBS_MAX_R");
    if (!phi_host || !terms_dev || !out_dev) return fail(ctx, RBS_E_ARG, "phi/terms/out is NULL");
    const cudaStream_t st = (cudaStream_t)stream;
    CK(cudaSetDevice(ctx->device));
    double* dphi = nullptr;
    CK(cudaMallocAsync((void**)&dphi, (size_t)B * R * 8, st));
    CK(cudaMemcpyAsync(dphi, phi_host, (size_t)B * R * 8, cudaMemcpyHostToDevice, st));
    const int64_t tot = (int64_t)B * ctx->g.N;
    k_affine_rhs<<<(unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 16), 256, 0, st>>>(
        dphi, R, terms_dev, ctx->g.N, B, out_dev);
    CKL();
    CK(cudaFreeAsync(dphi, st));
    CK(cudaStreamSynchronize(st));
    return RBS_OK;
}

rbs_status rbs_set_rhs_constant(rbs_ctx* ctx, double value) {
    if (!ctx) return RBS_E_ARG;
    ctx->err.clear();
    if (!std::isfinite(value)) return fail(ctx, RBS_E_ARG, "rhs constant must be finite");
    ctx->fconst = value;
    if (ctx->R > 0) {           // back to the constant right-hand side: the basis layout changes
        ctx->R = 0;
        ctx->fr.clear();
        ctx->T = nullptr;
        ctx->Pa.clear();
        ctx->has_basis = false;
    }
    return RBS_OK;
}

rbs_status rbs_set_rhs_terms(rbs_ctx* ctx, int R, const double* const* f_dev) {
    if (!ctx) return RBS_E_ARG;
    ctx->err.clear();
    if (!ctx->has_op) return fail(ctx, RBS_E_STATE, "set the operator first");
    if (ctx->dist || ctx->nslab > 1) return fail(ctx, RBS_E_UNSUPPORTED, "mesh slabs: affine rhs terms not supported");
    if (R < 0 || R > RBS_MAX_R) return fail(ctx, RBS_E_DIM, "R must be in 0..RBS_MAX_R");
    if (R > 0 && !f_dev) return fail(ctx, RBS_E_ARG, "f_dev is NULL");
    for (int r = 0; r < R; ++r)
        if (!f_dev[r]) return fail(ctx, RBS_E_ARG, "a term pointer is NULL");
    ctx->R = R;
    ctx->fr.assign(f_dev, f_dev + R);
    ctx->T = nullptr;
    ctx->Pa.clear();            // phi map (R rows) refers to the old terms
    ctx->has_basis = false;     // f_{n,r}, the Gram matrix and the storage layout are per basis
    if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; ctx->gkey.clear(); }
    return RBS_OK;
}

rbs_status rbs_set_param_map(rbs_ctx* ctx, int P, const double* theta_aff, const double* phi_aff) {
    if (!ctx) return RBS_E_ARG;
    ctx->err.clear();
    if (!ctx->has_op) return fail(ctx, RBS_E_STATE, "set the operator first");
    if (P < 1 || P > RBS_MAX_Q) return fail(ctx, RBS_E_DIM, "P must be in 1..RBS_MAX_Q");
    const int Q = ctx->g.Q, R = ctx->R;
    if (!theta_aff && P != Q) return fail(ctx, RBS_E_DIM, "identity theta map needs P == Q");
    if (phi_aff && R == 0) return fail(ctx, RBS_E_STATE, "phi map without rhs terms (rbs_set_rhs_terms)");
    ctx->P = P;
    ctx->Ta.clear();
    ctx->Pa.clear();
    if (theta_aff) ctx->Ta.assign(theta_aff, theta_aff + (size_t)Q * (P + 1));
    if (phi_aff) ctx->Pa.assign(phi_aff, phi_aff + (size_t)R * (P + 1));
    for (double v : ctx->Ta)
        if (!std::isfinite(v)) return fail(ctx, RBS_E_ARG, "theta map not finite");
    for (double v : ctx->Pa)
        if (!std::isfinite(v)) return fail(ctx, RBS_E_ARG, "phi map not finite");
    return RBS_OK;
}

rbs_status rbs_operator_labels_size(int dim, int64_t m, int Q, size_t* bytes) {
    if (!bytes || (dim != 2 && dim != 3) || m < 1 || Q < 1 || Q > RBS_MAX_Q) return RBS_E_ARG;
    *bytes = (size_t)Q * dim * (size_t)(m + 1) * (size_t)(dim == 3 ? m * m : m) * 8;
    return RBS_OK;
}

rbs_status rbs_set_operator_labels(rbs_ctx* ctx, int dim, int64_t m, int Q, const uint8_t* cell_label_dev,
                                   void* faces_storage_dev, size_t storage_bytes, void* stream) {
    if (!ctx) return RBS_E_ARG;
    ctx->err.clear();
    if (!cell_label_dev || !faces_storage_dev) return fail(ctx, RBS_E_ARG, "labels / storage is NULL");
    size_t need = 0;
    if (rbs_operator_labels_size(dim, m, Q, &need) != RBS_OK) return fail(ctx, RBS_E_DIM, "bad dim/m/Q");
    if (storage_bytes < need) return fail(ctx, RBS_E_NOMEM, "face storage too small");
    if (Q > 255) return fail(ctx, RBS_E_DIM, "labels are uint8: Q <= 255");
    CK(cudaSetDevice(ctx->device));
    const cudaStream_t st = (cudaStream_t)stream;
    const int64_t nfd = (int64_t)dim * (m + 1) * (dim == 3 ? m * m : m);
    k_labels_to_faces<<<grid_for(nfd, 256, ctx->num_sms * 8), 256, 0, st>>>(cell_label_dev, dim, (int)m, Q,
                                                                          (double*)faces_storage_dev);
    CKL();
    CK(cudaStreamSynchronize(st));
    return rbs_set_operator_faces(ctx, dim, m, Q, (const double*)faces_storage_dev);
}

rbs_status rbs_basis_storage_size(const rbs_ctx* c, int n, size_t* bytes) {
    rbs_ctx* ctx = const_cast<rbs_ctx*>(c);
    if (!ctx || !bytes) return RBS_E_ARG;
    if (!ctx->has_op) return fail(ctx, RBS_E_STATE, "set the operator first");
    if (n < 0 || n > RBS_MAX_N) return fail(ctx, RBS_E_DIM, "n out of range");
    *bytes = basis_layout(ctx, n, nullptr).bytes;
    return RBS_OK;
}

rbs_status rbs_load_basis(rbs_ctx* ctx, int n, const double* W_dev, int64_t ldw,
                          const double* ANq_host, const double* fn_host, void* storage_dev,
                          size_t storage_bytes, void* stream) {
    if (!ctx) return RBS_E_ARG;
    ctx->err.clear();
    if (!ctx->has_op) return fail(ctx, RBS_E_STATE, "set the operator first");
    if (n < 0 || n > RBS_MAX_N) return fail(ctx, RBS_E_DIM, "n out of range 0..64");
    if (n > 0 && (!W_dev || ldw < ctx->g.N)) return fail(ctx, RBS_E_DIM, "W_dev NULL or ldw < N");
    if (ctx->dist && n > 0 && (!ANq_host || !fn_host))
        return fail(ctx, RBS_E_ARG, "mesh slabs over ranks: pass the offline blocks (ANq_host, fn_host)");
    if (!storage_dev) return fail(ctx, RBS_E_ARG, "storage_dev is NULL");
    BasisLayout L = basis_layout(ctx, n, storage_dev);
    if (storage_bytes < L.bytes) return fail(ctx, RBS_E_NOMEM, "storage too small");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    const Geo& g = ctx->g;
    const int npad = (int)round_up(n, 8);
    ctx->has_basis = false;
    ctx->n = n;
    ctx->npad = npad;
    ctx->ldw = w_ld(npad);
    ctx->Wi = L.Wi;
    ctx->dANq = L.ANq;
    ctx->scratch = L.Z;
    if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; ctx->gkey.clear(); }
    const int Q = g.Q;
    if (n > 0) {
        k_pack_W<<<grid_for(ctx->N8 * ctx->ldw, 256, 4 * ctx->num_sms * 8), 256, 0, st>>>(
            W_dev, ldw, g.N, ctx->N8, n, ctx->ldw, L.Wi);
        CKL();
    }
    ctx->hANq.assign((size_t)Q * n * n, 0.0);
    ctx->hfn.assign(n, 0.0);
    if (n > 0 && ANq_host) {
        std::memcpy(ctx->hANq.data(), ANq_host, sizeof(double) * Q * n * n);
    } else if (n > 0) {
        // A_{n,q} = W^T A_q W, 8 columns at a time: Z = A_q W[:, j0:j0+8], then
        // the DMMA projection W^T Z; entries (i <= j) mirrored (oracle O-3).
        const int nct = proj_ctas(g);
        std::vector<double> rows((size_t)8 * (npad + 1));
        for (int q = 0; q < Q; ++q)
            for (int j0 = 0; j0 < npad; j0 += 8) {
                const int grid = grid_for(g.N * 8, kThreads, ctx->num_sms * 8);
                if (g.dim == 2) k_apply_Aq<2><<<grid, kThreads, 0, st>>>(g, q, L.Wi, ctx->ldw, j0, L.Z);
                else k_apply_Aq<3><<<grid, kThreads, 0, st>>>(g, q, L.Wi, ctx->ldw, j0, L.Z);
                CKL();
                ProjArgs a{};
                a.g = g; a.Bp = 8; a.npad = npad; a.nct = nct; a.ngroups = (g.N + 3) / 4; a.ldw = ctx->ldw;
                a.W = L.Wi; a.V = L.Z; a.part = L.part;
                launch_proj<MODE_PLAIN>(g, nct, proj_smem(g, 8, npad), st, a);
                CKL();
                k_reduce_rows<<<8, 128, 0, st>>>(L.part, npad + 1, nct, L.rows);
                CKL();
                CK(cudaMemcpyAsync(rows.data(), L.rows, rows.size() * 8, cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                for (int jj = 0; jj < 8 && j0 + jj < n; ++jj) {
                    const int j = j0 + jj;
                    for (int i = 0; i <= j; ++i) {
                        const double v = rows[(size_t)jj * (npad + 1) + i];
                        ctx->hANq[((size_t)q * n + i) * n + j] = v;
                        ctx->hANq[((size_t)q * n + j) * n + i] = v;
                    }
                }
            }
    }
    if (n > 0 && fn_host) {
        std::memcpy(ctx->hfn.data(), fn_host, sizeof(double) * n);
    } else if (n > 0) {
        const int nct = proj_ctas(g);
        ProjArgs a{};
        a.g = g; a.Bp = 8; a.npad = npad; a.nct = nct; a.ngroups = (g.N + 3) / 4; a.ldw = ctx->ldw;
        a.W = L.Wi; a.V = nullptr; a.vconst = 1.0; a.part = L.part;
        launch_proj<MODE_PLAIN>(g, nct, proj_smem(g, 8, npad), st, a);
        CKL();
        k_reduce_rows<<<8, 128, 0, st>>>(L.part, npad + 1, nct, L.rows);
        CKL();
        std::vector<double> rows((size_t)8 * (npad + 1));
        CK(cudaMemcpyAsync(rows.data(), L.rows, rows.size() * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int j = 0; j < n; ++j) ctx->hfn[j] = rows[j];
    }
    if (rbs_status ts = terms_offline(ctx, L, st); ts != RBS_OK) return ts;
    // padded device copy of the blocks, then f_n (the broadcast region)
    std::vector<double> pad((size_t)Q * npad * npad + npad + 8, 0.0);
    for (int q = 0; q < Q; ++q)
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                pad[((size_t)q * npad + i) * npad + j] = ctx->hANq[((size_t)q * n + i) * n + j];
    for (int j = 0; j < n; ++j) pad[(size_t)Q * npad * npad + j] = ctx->hfn[j];
    CK(cudaMemcpyAsync(L.ANq, pad.data(), pad.size() * 8, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    ctx->has_basis = true;
    return RBS_OK;
}

rbs_status rbs_get_offline_blocks(const rbs_ctx* c, double* ANq_host, double* fn_host) {
    rbs_ctx* ctx = const_cast<rbs_ctx*>(c);
    if (!ctx) return RBS_E_ARG;
    if (!ctx->has_basis) return fail(ctx, RBS_E_STATE, "no basis loaded");
    if (ANq_host) std::memcpy(ANq_host, ctx->hANq.data(), ctx->hANq.size() * 8);
    if (fn_host) std::memcpy(fn_host, ctx->hfn.data(), ctx->hfn.size() * 8);
    return RBS_OK;
}

void rbs_default_opts(rbs_solve_opts* o) {
    if (!o) return;
    o->method = RBS_RBCG;
    o->tol = 1e-10;
    o->max_iter = 20000;
    o->smoother = RBS_SMOOTH_SYM_RBGS;
    o->sweeps = 1;
    o->delta = 1e-12;
    o->record_history = 0;
    o->x_location = RBS_MEM_DEVICE;
    o->graph_chunk = 16;
    o->profile = 0;
    o->n_active = 0;
    o->gamma = 0.0;
    o->omega = 1.0;
    o->precond = RBS_PRECOND_POST;
    o->beta_rule = RBS_BETA_FR;
}

rbs_status rbs_solve_workspace_size(const rbs_ctx* c, int B, const rbs_solve_opts* o, size_t* bytes) {
    rbs_ctx* ctx = const_cast<rbs_ctx*>(c);
    if (!ctx || !bytes) return RBS_E_ARG;
    if (!ctx->has_basis) return fail(ctx, RBS_E_STATE, "no basis loaded");
    if (B < 1 || B > RBS_MAX_BATCH) return fail(ctx, RBS_E_DIM, "B out of range 1..64");
    rbs_status s = check_opts(ctx, o);
    if (s != RBS_OK) return s;
    *bytes = solve_layout(ctx, B, o, true, nullptr).bytes;
    if (ctx->nslab > 1 || ctx->dist) *bytes = std::max(*bytes, slab_plan(ctx, B, o, nullptr).bytes);
    return RBS_OK;
}

// mu_host here is theta (B x Q, the parameter map already applied); phi_host (B x R)
// the right-hand-side coefficients when affine terms are set
static rbs_status solve_batch_impl(rbs_ctx* ctx, int B, const double* mu_host, const double* phi_host,
                                   const rbs_solve_opts* o,
                                   const double* rhs_dev, double* X, int* iters, int* qstatus,
                                   double* relres, double* true_relres, double* a_n, double* history,
                                   void* workspace_dev, size_t workspace_bytes, void* stream) {
    if (!ctx) return RBS_E_ARG;
    ctx->err.clear();
    ctx->launches = 0;
    if (!ctx->has_basis) return fail(ctx, RBS_E_STATE, "no basis loaded");
    if (B < 1 || B > RBS_MAX_BATCH) return fail(ctx, RBS_E_DIM, "B out of range 1..64");
    if (!mu_host || !X || !workspace_dev) return fail(ctx, RBS_E_ARG, "mu_host/X/workspace is NULL");
    rbs_status s0 = check_opts(ctx, o);
    if (s0 != RBS_OK) return s0;
    const bool terms = ctx->R > 0 && rhs_dev == nullptr;   // f(mu) = sum_r phi_r f_r online
    if (ctx->nslab > 1 || ctx->dist) {
        if (rhs_dev) return fail(ctx, RBS_E_UNSUPPORTED, "mesh slabs: rhs override not supported");
        if (ctx->R > 0) return fail(ctx, RBS_E_UNSUPPORTED, "mesh slabs: affine rhs terms not supported");
        if (o->smoother == RBS_SMOOTH_JACOBI)
            return fail(ctx, RBS_E_UNSUPPORTED, "mesh slabs: Jacobi smoother not supported");
        CK(cudaSetDevice(ctx->device));
        return solve_slabs(ctx, B, mu_host, o, X, iters, qstatus, relres, true_relres, a_n, history,
                           workspace_dev, workspace_bytes, (cudaStream_t)stream);
    }
    SolveLayout L = solve_layout(ctx, B, o, rhs_dev != nullptr || terms, workspace_dev);
    if (workspace_bytes < solve_layout(ctx, B, o, rhs_dev != nullptr || terms, nullptr).bytes)
        return fail(ctx, RBS_E_NOMEM, "workspace too small");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    const Geo& g = ctx->g;
    const int Bp = pow2_batch(B), lgB = ilog2(Bp), n = ctx->n, npad = ctx->npad, Q = g.Q;
    // RBS_DISABLE_V2 (debug / A-B, read at rbs_create): bit 0 smoother, bit 1 p-update, bit 2 projection,
    // bit 14 programmatic dependent launch of the 2D iteration passes
    const int v2off = ctx->v2off;
    const bool pdl = !(v2off & 16384);
    const bool cg = o->method == RBS_RBCG;
    // 2D, B_pad <= 32: the projection pass is the row march (k_resid_march)
    const bool use_rmarch = g.dim == 2 && Bp <= 32 && !g.faces;   // row marches: block tables
    const MarchPart rpart = march_part(g, kRmTX, ctx->num_sms);
    const int nct = use_rmarch ? rpart.nsx * rpart.nsy : proj_ctas(g), nctf = part_ctas(g, ctx->num_sms);
    const int nct_plain = proj_ctas(g);
    const int64_t vecN = ctx->N8 * Bp;
    const size_t psm = proj_smem(g, Bp, npad), fsm = flat_smem(g, Bp);
    int64_t launches = 0;

    // ---- parameters: theta_q = mu_q (Q = P), padded lanes get 1 -------------
    std::vector<double> th((size_t)Q * Bp, 1.0);
    for (int b = 0; b < B; ++b)
        for (int q = 0; q < Q; ++q) {
            const double v = mu_host[(size_t)b * Q + q];
            th[(size_t)q * Bp + b] = v;
        }
    CK(cudaMemcpyAsync(L.theta, th.data(), th.size() * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(L.ints, 0, 8 * sizeof(int), st));
    int* kcount = L.ints;
    int* done = L.ints + 1;
    unsigned* ticket = (unsigned*)(L.ints + 2);
    CK(cudaMemsetAsync(L.E, 0, (size_t)std::max(npad, 8) * Bp * 8, st));
    CK(cudaMemsetAsync(L.a_n, 0, ((size_t)Bp * npad + 8) * 8, st));
    if (L.hist) {
        // NaN-fill history: 0xFF bytes are a NaN pattern
        CK(cudaMemsetAsync(L.hist, 0xFF, (size_t)Bp * (o->max_iter + 1) * 8, st));
    }
    const int fgrid = grid_for(vecN, 256, ctx->num_sms * 8);

    // ---- right-hand side, f_n and ||f|| per query ---------------------------
    const double* Fv = nullptr;
    if (rhs_dev) {
        k_fill_batch<<<fgrid, 256, 0, st>>>(L.F, g.N, ctx->N8, Bp, B, rhs_dev, 0.0);
        CKL();
        ++launches;
        Fv = L.F;
        ProjArgs a{};
        a.g = g; a.Bp = Bp; a.npad = npad; a.nct = nct_plain; a.ngroups = (g.N + 3) / 4; a.ldw = ctx->ldw;
        a.W = ctx->Wi; a.theta = L.theta; a.V = L.F; a.part = L.partP;
        launch_proj<MODE_PLAIN>(g, nct_plain, psm, st, a);
        CKL();
        k_reduce_rows<<<Bp, 128, 0, st>>>(L.partP, npad + 1, nct_plain, L.fproj);
        CKL();
        launches += 2;
    } else if (terms) {
        // affine right-hand side, online (eq12b): F = sum_r phi_r f_r on the
        // device (one pass over the packed terms), f_n(mu) = sum_r phi_r f_{n,r} and
        // ||f(mu)||^2 = phi^T G phi from the offline quantities -- no projection pass
        const int R = ctx->R;
        std::vector<double> ph((size_t)Bp * R, 0.0), fp((size_t)Bp * (npad + 1), 0.0);
        for (int b = 0; b < B; ++b) {
            const double* pb = phi_host + (size_t)b * R;
            for (int r = 0; r < R; ++r) ph[(size_t)b * R + r] = pb[r];
            for (int j = 0; j < n; ++j) {
                double v = 0.0;
                for (int r = 0; r < R; ++r) v += pb[r] * ctx->hfNr[(size_t)r * n + j];
                fp[(size_t)b * (npad + 1) + j] = v;
            }
            double ff = 0.0;
            for (int r = 0; r < R; ++r) {
                double gr = 0.0;
                for (int t2 = 0; t2 < R; ++t2) gr += ctx->hG[(size_t)r * R + t2] * pb[t2];
                ff += pb[r] * gr;
            }
            fp[(size_t)b * (npad + 1) + npad] = ff;
        }
        CK(cudaMemcpyAsync(L.phi, ph.data(), ph.size() * 8, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(L.fproj, fp.data(), fp.size() * 8, cudaMemcpyHostToDevice, st));
        k_fill_terms<<<fgrid, 256, 0, st>>>(L.F, g.N, ctx->N8, Bp, B, ctx->T, ctx->ldt, R, L.phi);
        CKL();
        ++launches;
        Fv = L.F;
    } else {
        std::vector<double> fp((size_t)Bp * (npad + 1), 0.0);
        for (int b = 0; b < Bp; ++b) {
            for (int j = 0; j < n; ++j) fp[(size_t)b * (npad + 1) + j] = ctx->fconst * ctx->hfn[j];
            fp[(size_t)b * (npad + 1) + npad] = ctx->fconst * ctx->fconst * (double)g.N;
        }
        CK(cudaMemcpyAsync(L.fproj, fp.data(), fp.size() * 8, cudaMemcpyHostToDevice, st));
    }
    CK(cudaMemsetAsync(L.X, 0, vecN * 8, st));
    if (L.X2) CK(cudaMemsetAsync(L.X2, 0, vecN * 8, st));
    if (cg) {
        CK(cudaMemsetAsync(L.P0, 0, vecN * 8, st));
        CK(cudaMemsetAsync(L.P1, 0, vecN * 8, st));
        if (terms) {
            CK(cudaMemcpyAsync(L.R, L.F, vecN * 8, cudaMemcpyDeviceToDevice, st));   // r_0 = f
        } else {
            k_fill_batch<<<fgrid, 256, 0, st>>>(L.R, g.N, ctx->N8, Bp, B, rhs_dev, ctx->fconst);
            CKL();
            ++launches;
        }
    }

    SolveState S{};
    S.B = B; S.Bp = Bp; S.n = n; S.npad = npad; S.nct = nct; S.nctf = nctf;
    S.maxit = o->max_iter; S.method = cg ? 1 : 0; S.tol = o->tol; S.delta = o->delta;
    S.ANq = ctx->dANq; S.Q = Q; S.theta = L.theta; S.fproj = L.fproj; S.L = L.L; S.Ainv = L.Ainv; S.E = L.E;
    S.a_n = L.a_n; S.partP = L.partP; S.partF = L.partF; S.alpha = L.alpha; S.beta = L.beta;
    S.rho = L.rho; S.rr = L.rr; S.fnorm = L.fnorm; S.relres = L.relres; S.active = L.active;
    S.status = L.status; S.its = L.its; S.pivot = L.pivot; S.kcount = kcount; S.done = done;
    S.ticket = ticket; S.hist = L.hist;
    set_active_dim(S, L.na, o, n);

    k_setup_reduced<<<Bp, 128, 0, st>>>(S, cg ? 0 : 1);
    CKL();
    ++launches;

    const std::vector<int> seq = color_seq(o->smoother, o->sweeps);
    const int pgrid = grid_for(((g.N + 7) / 8) * (Bp / 8), 8, ctx->num_sms * 16);

    // 3D z-plane marches fed by TMA tensor maps (zmarch.cuh): full grid, B_pad 8 / 16 / 32, thermal
    // blocks or face coefficients (RBS_DISABLE_V2 bit 16 keeps the row-segment kernels, bit 17 for faces)
    const bool zm3 = g.dim == 3 && g.kofs == 0 && g.mz == g.m && (Bp == 8 || Bp == 16 || Bp == 32) &&
                     !(v2off & 65536) && !(g.faces && (v2off & 131072)) && tmap_encoder() != nullptr;
    const bool zf = g.faces != nullptr;   // face-coefficient instantiations (AMB-23)
    const int ztx = Bp == 8 ? ZShape<8>::TX : Bp == 16 ? ZShape<16>::TX : ZShape<32>::TX;
    const int zty = Bp == 8 ? ZShape<8>::TY : Bp == 16 ? ZShape<16>::TY : ZShape<32>::TY;
    ZPart zpt{};
    int zgrid = 0;
    if (zm3) {
        zpt = z_part(g, ztx, zty, std::min(ctx->num_sms, nctf));
        zgrid = std::min(std::min(ctx->num_sms, nctf), zpt.units);
    }
    auto zsm = [&](int kind) {
        const size_t b = Bp == 8 ? zsmem_bytes<8>(kind, Q) : Bp == 16 ? zsmem_bytes<16>(kind, Q) : zsmem_bytes<32>(kind, Q);
        return b <= kZMaxDyn ? b : (size_t)0;
    };
    // 3D prolongation by TMA (k_prolz): odd m (colour = index parity), full grid, rows of at most
    // kMaxN + 4 doubles, ring within the shared-memory budget (RBS_DISABLE_V2 bit 18 keeps k_prolong)
    const bool zprol = g.dim == 3 && (g.m & 1) && g.kofs == 0 && g.mz == g.m && (Bp == 8 || Bp == 16 || Bp == 32) &&
                       !(v2off & 262144) && tmap_encoder() != nullptr && ctx->ldw <= kMaxN + 4 &&
                       prolz_smem_bytes(Bp, ctx->ldw) <= kZMaxDyn;
    // W viewed as [pairs][2][ldw]: box [ldw][1][CH] = CH rows of one index parity
    auto zmap_w = [&](CUtensorMap* mp) {
        auto enc = tmap_encoder();
        if (!enc) return false;
        const int ch = 128 / (Bp / 8);
        cuuint64_t dims[3] = {(cuuint64_t)ctx->ldw, 2, (cuuint64_t)((g.N + 1) / 2)};
        cuuint64_t strides[2] = {(cuuint64_t)ctx->ldw * 8, (cuuint64_t)ctx->ldw * 16};
        cuuint32_t box[3] = {(cuuint32_t)ctx->ldw, 1, (cuuint32_t)ch};
        cuuint32_t es[3] = {1, 1, 1};
        return enc(mp, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, ctx->Wi, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    // haloed (stencil operand) / interior (pointwise operand) plane-tile maps of a batch vector
    auto zmap_h = [&](CUtensorMap* mp, const double* v) { return zmap(mp, v, g, Bp, ztx + 2, zty + 2); };
    auto zmap_i = [&](CUtensorMap* mp, const double* v) { return zmap(mp, v, g, Bp, ztx, zty); };

    // ---- profiling hooks (no-ops unless opts.profile) -------------------------
    const bool prof = o->profile != 0;
    int pne = 0;
    std::vector<int> pcls;
    if (prof && ctx->pev.empty()) {
        ctx->pev.resize(2 * 256);
        for (auto& e : ctx->pev) CK(cudaEventCreate(&e));
    }
    for (int k = 0; k < RBS_K_NCLASS; ++k) { ctx->prof_ms[k] = 0.0; ctx->prof_cnt[k] = 0; }
    auto pb = [&](int cls) {
        if (prof && pne < 256) { cudaEventRecord(ctx->pev[2 * pne], st); pcls.push_back(cls); }
    };
    auto pe = [&]() {
        if (prof && pne < 256) { cudaEventRecord(ctx->pev[2 * pne + 1], st); ++pne; }
    };

    // ---- pass builders -------------------------------------------------------
    // skip: the colour of the half-sweep that follows (its nodes are overwritten unread)
    auto prolong = [&](double* Yv, int acc, int skip = -1) {
        ProlongArgs a{};
        a.N = g.N; a.Bp = Bp; a.npad = npad; a.ldw = ctx->ldw; a.W = ctx->Wi; a.E = L.E; a.active = L.active;
        a.Y = Yv; a.accumulate = acc; a.done = done;
        a.skip_color = skip; a.dim = g.dim; a.m = g.m; a.kofs = g.kofs; a.fm = g.fm;
        pb(RBS_K_PROLONG);
        CUtensorMap mw;
        if (npad > 0 && zprol && skip >= 0 && zmap_w(&mw)) {
            // odd m: the rows outside the skipped colour are the rows of index parity `skip`
            ProlzArgs z{};
            z.N = g.N; z.npairs = (g.N + 1) / 2; z.Bp = Bp; z.npad = npad; z.ldw = ctx->ldw; z.par = skip;
            z.E = L.E; z.active = L.active; z.Y = Yv; z.accumulate = acc; z.done = done;
            const size_t sm = prolz_smem_bytes(Bp, ctx->ldw);
            const int64_t nch = (z.npairs + (128 / (Bp / 8)) - 1) / (128 / (Bp / 8));
            const int grid = (int)std::min<int64_t>(ctx->num_sms, nch);
            if (Bp == 8) k_prolz<8><<<grid, kZT, sm, st>>>(mw, z);
            else if (Bp == 16) k_prolz<16><<<grid, kZT, sm, st>>>(mw, z);
            else k_prolz<32><<<grid, kZT, sm, st>>>(mw, z);
        } else if (npad > 0) {
            k_prolong<<<pgrid, kThreads, 0, st>>>(a);
        } else if (!acc) {  // empty basis: y0 = 0
            k_fill_batch<<<fgrid, 256, 0, st>>>(Yv, g.N, ctx->N8, Bp, 0, nullptr, 0.0);
        } else {
            pe();
            return 0;
        }
        pe();
        return 1;
    };
    const bool jac = o->smoother == RBS_SMOOTH_JACOBI;
    // Jacobi: sweeps alternate between Ys and the other buffer (T, or Yf when Ys == T);
    // the result must end in Yf (a device copy when the parity leaves it elsewhere)
    auto smooth_jac = [&](double* Ys, double* Yf, const double* rhs, double rconst, bool last, int init) {
        GSArgs a{};
        a.g = g; a.Bp = Bp; a.lgB = lgB; a.NB = g.N * Bp; a.theta = L.theta; a.active = L.active;
        a.Rhs = rhs; a.rconst = rconst; a.init = init; a.s = S; a.done = done; a.omega = o->omega;
        double* buf[2] = {Ys, Ys == L.T ? Yf : L.T};
        const int nu = o->sweeps;
        int cnt = 0;
        for (int t = 0; t < nu; ++t) {
            a.Yin = buf[t & 1];
            a.Y = buf[(t + 1) & 1];
            const bool l = last && t + 1 == nu;
            pb(RBS_K_GS);
            if (g.dim == 2) {
                if (l) k_jac<2, true><<<nctf, kFlat, fsm, st>>>(a);
                else k_jac<2, false><<<nctf, kFlat, fsm, st>>>(a);
            } else {
                if (l) k_jac<3, true><<<nctf, kFlat, fsm, st>>>(a);
                else k_jac<3, false><<<nctf, kFlat, fsm, st>>>(a);
            }
            pe();
            ++cnt;
        }
        if (buf[nu & 1] != Yf) {
            k_copy_unless_done<<<fgrid, 256, 0, st>>>(Yf, buf[nu & 1], (int64_t)ctx->N8 * Bp, done);  // CKL after
        }
        if (nu == 0 && last) {   // no sweep: y = y0, Step 10 partials by an empty GS pass
            a.Y = Yf;
            a.color = -1;
            pb(RBS_K_GS);
            if (g.dim == 2) k_gs<2, true><<<nctf, kFlat, fsm, st>>>(a);
            else k_gs<3, true><<<nctf, kFlat, fsm, st>>>(a);
            pe();
            ++cnt;
        }
        return cnt;
    };
    // sq: the colour sequence (default: the smoother's; the adjoint sweep of the symmetric
    // preconditioner passes it reversed)
    // zero0: the sweep starts from Yv = 0 (the symmetric preconditioner's pre-sweep).  On the
    // 3D z-plane march the first half-sweep then runs as k_gsz<ZERO> (no fill, no y tiles;
    // RBS_DISABLE_V2 bit 20 keeps the k_fill_batch + half-sweep pair, as does init: the
    // solve's first call also zeroes the padding rows); every other path fills Yv first
    auto smooth = [&](double* Yv, const double* rhs, double rconst, bool last, int init,
                      const std::vector<int>* sq = nullptr, bool zero0 = false) {
        int cnt = 0;
        std::vector<int> cs = sq ? *sq : seq;
        bool z0 = zero0 && !jac && zm3 && !init && !last && !cs.empty() && cs[0] >= 0 && zsm(1) &&
                  !(v2off & 1048576);
        if (z0) {
            CUtensorMap probe;
            z0 = zmap_h(&probe, Yv) && zmap_i(&probe, rhs ? rhs : Yv);
        }
        if (zero0 && !z0) {
            k_fill_batch<<<fgrid, 256, 0, st>>>(Yv, g.N, ctx->N8, Bp, 0, nullptr, 0.0);
            ++cnt;
        }
        if (jac) return cnt + smooth_jac(Yv, Yv, rhs, rconst, last, init);
        GSArgs a{};
        a.g = g; a.Bp = Bp; a.lgB = lgB; a.NB = g.N * Bp; a.theta = L.theta; a.active = L.active;
        a.Y = Yv; a.Rhs = rhs; a.rconst = rconst; a.init = init; a.s = S; a.done = done;
        if (cs.empty() && last) cs.push_back(-1);
        for (size_t t = 0; t < cs.size(); ++t) {
            a.color = cs[t];
            const bool l = last && t + 1 == cs.size();
            CUtensorMap my, mr;
            pb(RBS_K_GS);
            if (g.dim == 2) {
                if (l) k_gs<2, true><<<nctf, kFlat, fsm, st>>>(a);
                else k_gs<2, false><<<nctf, kFlat, fsm, st>>>(a);
            } else if (zm3 && a.color >= 0 && zsm(1) && zmap_h(&my, Yv) && zmap_i(&mr, rhs ? rhs : Yv)) {
                // z-plane march: y tile with halo + r tile per plane by tensor-map copies
#define RBS_GSZ(BPV, L, F) k_gsz<BPV, L, F><<<zgrid, kZT, zsm(1), st>>>(my, mr, a, zpt)
#define RBS_GSZ0(BPV, F) k_gsz<BPV, false, F, true><<<zgrid, kZT, zsm(1), st>>>(my, mr, a, zpt)
#define RBS_GSZ2(BPV) \
    if (z0 && t == 0) { if (zf) RBS_GSZ0(BPV, true); else RBS_GSZ0(BPV, false); } \
    else if (zf) { if (l) RBS_GSZ(BPV, true, true); else RBS_GSZ(BPV, false, true); } \
    else { if (l) RBS_GSZ(BPV, true, false); else RBS_GSZ(BPV, false, false); }
                if (Bp == 8) { RBS_GSZ2(8) }
                else if (Bp == 16) { RBS_GSZ2(16) }
                else { RBS_GSZ2(32) }
#undef RBS_GSZ2
#undef RBS_GSZ0
#undef RBS_GSZ
            } else if (Bp <= 32 && !(v2off & 8) && a.color >= 0) {   // row pencils (x in registers)
                // 4-node row segments, all loads of a segment in flight (128 registers,
                // one CTA per SM: measured 2.2x the element-per-thread k_gs at 127^3, B = 16)
                if (g.faces) {
                    if (l) k_gs3r<true, 4, true><<<nctf, kFlat, fsm, st>>>(a);
                    else k_gs3r<false, 4, true><<<nctf, kFlat, fsm, st>>>(a);
                } else {
                    if (l) k_gs3r<true, 4, false><<<nctf, kFlat, fsm, st>>>(a);
                    else k_gs3r<false, 4, false><<<nctf, kFlat, fsm, st>>>(a);
                }
            } else {
                if (l) k_gs<3, true><<<nctf, kFlat, fsm, st>>>(a);
                else k_gs<3, false><<<nctf, kFlat, fsm, st>>>(a);
            }
            pe();
            ++cnt;
        }
        return cnt;
    };
    auto proj = [&](int mode, const double* P, bool use_active, double* Xv = nullptr, const double* Vv = nullptr) {
        if (use_rmarch && use_active) {
            ResidMarchArgs r{};
            r.g = g; r.Bp = Bp; r.npad = npad; r.ldw = ctx->ldw; r.mp = rpart; r.W = ctx->Wi;
            r.theta = L.theta; r.active = L.active; r.alpha = L.alpha; r.P = P;
            r.X = Xv ? Xv : L.X; r.R = L.R; r.V = Vv ? Vv : Fv; r.vconst = ctx->fconst;
            r.part = L.partP; r.nct = nct; r.done = done;
            const int PF = resid2_smem_bytes(2, Bp, ctx->ldw, Q) <= (size_t)214 * 1024 ? 2 : 1;
            const size_t rsm = resid2_smem_bytes(PF, Bp, ctx->ldw, Q);
            pb(RBS_K_PROJ);
            const int md = mode == MODE_CG ? 0 : 1;
            if (v2off & 4) {
                const ResidSmem rs1(Bp, ctx->ldw, Q, md, r.V != nullptr);
                if (md == 0) k_resid_march<0><<<nct, kMarchThreads, rs1.total, st>>>(r);
                else k_resid_march<1><<<nct, kMarchThreads, rs1.total, st>>>(r);
            } else if (Bp == 8) {
                if (PF == 2) launch_resid2<8, 2>(md, nct, rsm, st, r, pdl);
                else launch_resid2<8, 1>(md, nct, rsm, st, r, pdl);
            } else if (Bp == 16) {
                if (PF == 2) launch_resid2<16, 2>(md, nct, rsm, st, r, pdl);
                else launch_resid2<16, 1>(md, nct, rsm, st, r, pdl);
            } else {
                if (PF == 2) launch_resid2<32, 2>(md, nct, rsm, st, r, pdl);
                else launch_resid2<32, 1>(md, nct, rsm, st, r, pdl);
            }
            pe();
            return 1;
        }
        ProjArgs a{};
        a.g = g; a.Bp = Bp; a.npad = npad; a.nct = nct; a.ngroups = (g.N + 3) / 4; a.ldw = ctx->ldw;
        a.W = ctx->Wi; a.theta = L.theta; a.active = use_active ? L.active : nullptr;
        a.alpha = L.alpha; a.P = P; a.X = Xv ? Xv : L.X; a.R = L.R; a.V = Vv ? Vv : Fv; a.vconst = ctx->fconst;
        a.part = L.partP; a.done = use_active ? done : nullptr;
        a.nct = use_active ? nct : nct_plain;
        pb(RBS_K_PROJ);
        int nl = 1;
        if (mode == MODE_CG && g.dim == 3 && use_active && Bp <= 32 && !(v2off & 8)) {
            // two passes: x, r update in row segments, then W^T r, ||r||^2 on the new r
            CUtensorMap mpz, mxz, mrz;
            if (zm3 && zsm(2) && zmap_h(&mpz, P) && zmap_i(&mxz, a.X) && zmap_i(&mrz, a.R)) {
                // z-plane march: p tile with halo, x and r tiles by tensor maps
                if (Bp == 8) {
                    if (zf) k_xrz<8, true><<<zgrid, kZT, zsm(2), st>>>(mpz, mxz, mrz, a, zpt);
                    else k_xrz<8, false><<<zgrid, kZT, zsm(2), st>>>(mpz, mxz, mrz, a, zpt);
                } else if (Bp == 16) {
                    if (zf) k_xrz<16, true><<<zgrid, kZT, zsm(2), st>>>(mpz, mxz, mrz, a, zpt);
                    else k_xrz<16, false><<<zgrid, kZT, zsm(2), st>>>(mpz, mxz, mrz, a, zpt);
                } else {
                    if (zf) k_xrz<32, true><<<zgrid, kZT, zsm(2), st>>>(mpz, mxz, mrz, a, zpt);
                    else k_xrz<32, false><<<zgrid, kZT, zsm(2), st>>>(mpz, mxz, mrz, a, zpt);
                }
            } else if (g.faces) k_xr3r<4, true><<<nctf, kFlat, fsm, st>>>(a, lgB);
            else k_xr3r<4, false><<<nctf, kFlat, fsm, st>>>(a, lgB);
            ProjArgs b2 = a;
            b2.V = L.R;
            // streamed W^T r with two CTAs per SM: 64-node chunks, 32 when W rows are long
            const int ch = wtr_smem_bytes(Bp, ctx->ldw, 64) <= (size_t)110 * 1024 ? 64 : 32;
            const size_t wsm = wtr_smem_bytes(Bp, ctx->ldw, ch);
            if (!(v2off & 32) && wsm <= (size_t)110 * 1024 && npad <= 64) {
                if (ch == 64) {
                    if (Bp == 8) k_wtr<8, 64><<<a.nct, kMT, wsm, st>>>(b2);
                    else if (Bp == 16) k_wtr<16, 64><<<a.nct, kMT, wsm, st>>>(b2);
                    else k_wtr<32, 64><<<a.nct, kMT, wsm, st>>>(b2);
                } else {
                    if (Bp == 8) k_wtr<8, 32><<<a.nct, kMT, wsm, st>>>(b2);
                    else if (Bp == 16) k_wtr<16, 32><<<a.nct, kMT, wsm, st>>>(b2);
                    else k_wtr<32, 32><<<a.nct, kMT, wsm, st>>>(b2);
                }
            } else {
                launch_proj<MODE_PLAIN>(g, a.nct, psm, st, b2);
            }
            nl = 2;
        } else if (mode == MODE_RESID && (!cg || o->precond == RBS_PRECOND_SYM) && g.dim == 3 && use_active && L.T &&
                   !(v2off & 524288) && !jac &&   // Jacobi: T is the sweeps' ping-pong buffer, whose copy-back
                                                  // (smooth_jac, not guarded by `done`) must not find v in it
                   zm3 && zsm(2) && npad <= 64 && wtr_smem_bytes(Bp, ctx->ldw, 32) <= (size_t)110 * 1024) {
            // symmetric preconditioner's W^T (r - A y1) / RBI's W^T (f - A x), 3D full grid
            // (RBS_DISABLE_V2 bit 19 keeps the flat k_proj<MODE_RESID>): v by the z-plane march
            // into the scratch vector T, then the streamed W^T v, ||v||^2 (two passes, as K2)
            CUtensorMap myz, mrz;
            if (zmap_h(&myz, a.X) && zmap_i(&mrz, a.V ? a.V : a.X)) {
                ProjArgs ar = a;
                ar.X = L.T;
                if (Bp == 8) {
                    if (zf) k_xrz<8, true, true><<<zgrid, kZT, zsm(2), st>>>(myz, mrz, mrz, ar, zpt);
                    else k_xrz<8, false, true><<<zgrid, kZT, zsm(2), st>>>(myz, mrz, mrz, ar, zpt);
                } else if (Bp == 16) {
                    if (zf) k_xrz<16, true, true><<<zgrid, kZT, zsm(2), st>>>(myz, mrz, mrz, ar, zpt);
                    else k_xrz<16, false, true><<<zgrid, kZT, zsm(2), st>>>(myz, mrz, mrz, ar, zpt);
                } else {
                    if (zf) k_xrz<32, true, true><<<zgrid, kZT, zsm(2), st>>>(myz, mrz, mrz, ar, zpt);
                    else k_xrz<32, false, true><<<zgrid, kZT, zsm(2), st>>>(myz, mrz, mrz, ar, zpt);
                }
                ProjArgs b2 = a;
                b2.V = L.T;
                // 64-node chunks, 32 when W rows are long (as K2)
                const int ch = wtr_smem_bytes(Bp, ctx->ldw, 64) <= (size_t)110 * 1024 ? 64 : 32;
                const size_t wsm = wtr_smem_bytes(Bp, ctx->ldw, ch);
                if (ch == 64) {
                    if (Bp == 8) k_wtr<8, 64><<<a.nct, kMT, wsm, st>>>(b2);
                    else if (Bp == 16) k_wtr<16, 64><<<a.nct, kMT, wsm, st>>>(b2);
                    else k_wtr<32, 64><<<a.nct, kMT, wsm, st>>>(b2);
                } else {
                    if (Bp == 8) k_wtr<8, 32><<<a.nct, kMT, wsm, st>>>(b2);
                    else if (Bp == 16) k_wtr<16, 32><<<a.nct, kMT, wsm, st>>>(b2);
                    else k_wtr<32, 32><<<a.nct, kMT, wsm, st>>>(b2);
                }
                nl = 2;
            } else {
                launch_proj<MODE_RESID>(g, a.nct, psm, st, a);
            }
        } else if (mode == MODE_CG) launch_proj<MODE_CG>(g, a.nct, psm, st, a);
        else launch_proj<MODE_RESID>(g, a.nct, psm, st, a);
        pe();
        return nl;
    };
    auto cgp = [&](const double* Pold, double* Pnew) {
        CGPArgs a{};
        a.g = g; a.Bp = Bp; a.lgB = lgB; a.NB = g.N * Bp; a.theta = L.theta; a.active = L.active;
        a.beta = L.beta; a.Y = L.Y; a.Pold = Pold; a.Pnew = Pnew; a.s = S; a.done = done;
        int nl = 1;
        CUtensorMap zmy, zmp;
        pb(RBS_K_CGP);
        if (!(v2off & 2) && g.dim == 2 && Bp <= 32 && !g.faces) {
            CGP2Args c2{};
            c2.g = g; c2.Bp = Bp; c2.theta = L.theta;
            c2.part = march_part(g, kC2TX, 2 * ctx->num_sms);   // 2 CTAs per SM
            c2.active = L.active; c2.beta = L.beta; c2.Y = L.Y; c2.Pold = Pold; c2.Pnew = Pnew;
            c2.s = S; c2.done = done;
            const size_t csm = cgp2_smem_bytes(Bp, Q);
            const int gr = c2.part.nsx * c2.part.nsy;
            if (Bp == 8) launch_k(pdl, k_cgp2<8>, gr, kMT, csm, st, c2);
            else if (Bp == 16) launch_k(pdl, k_cgp2<16>, gr, kMT, csm, st, c2);
            else launch_k(pdl, k_cgp2<32>, gr, kMT, csm, st, c2);
        } else if (g.dim == 2) k_cgp<2><<<nctf, kFlat, fsm, st>>>(a);
        else if (zm3 && zsm(0) && zmap_h(&zmy, L.Y) && zmap_h(&zmp, Pold)) {
            // one z-plane march: p = y + beta p_old on the haloed tiles, sigma = p^T A p
            if (Bp == 8) {
                if (zf) k_cgz<8, true><<<zgrid, kZT, zsm(0), st>>>(zmy, zmp, a, zpt);
                else k_cgz<8, false><<<zgrid, kZT, zsm(0), st>>>(zmy, zmp, a, zpt);
            } else if (Bp == 16) {
                if (zf) k_cgz<16, true><<<zgrid, kZT, zsm(0), st>>>(zmy, zmp, a, zpt);
                else k_cgz<16, false><<<zgrid, kZT, zsm(0), st>>>(zmy, zmp, a, zpt);
            } else {
                if (zf) k_cgz<32, true><<<zgrid, kZT, zsm(0), st>>>(zmy, zmp, a, zpt);
                else k_cgz<32, false><<<zgrid, kZT, zsm(0), st>>>(zmy, zmp, a, zpt);
            }
        } else if (Bp <= 32 && !(v2off & 8)) {      // two passes: stream p_new, then sigma in row segments
            const int64_t nb2 = (int64_t)g.N * Bp / 2;
            k_pnew3<<<(unsigned)std::min<int64_t>((nb2 + 255) / 256, (int64_t)ctx->num_sms * 16), 256, 0, st>>>(
                a.Y, a.Pold, a.Pnew, a.beta, a.active, nb2, Bp, a.done);
            if (g.faces) k_sigma3r<4, true><<<nctf, kFlat, fsm, st>>>(a);
            else k_sigma3r<4, false><<<nctf, kFlat, fsm, st>>>(a);
            nl = 2;
        } else k_cgp<3><<<nctf, kFlat, fsm, st>>>(a);
        pe();
        return nl;
    };

    // 2D: prolongation + all half-sweeps (+ y^T r) in one row-marching pass
    // NEXT(3) variants run the flat kernels: the symmetric two-level preconditioner
    // (RBS_PRECOND_SYM) and the Polak-Ribiere beta (RBS_BETA_PR)
    const bool sym = cg && o->precond == RBS_PRECOND_SYM, pr = cg && o->beta_rule == RBS_BETA_PR;
    const std::vector<int> rseq(seq.rbegin(), seq.rend());     // adjoint sweep: colours reversed
    // the red-black half-sweep that follows every prolongation (none: Jacobi / no sweeps)
    const int first_col = (!jac && !seq.empty() && !(v2off & 32768)) ? seq[0] : -1;
    const bool use_march = g.dim == 2 && seq.size() <= (size_t)kMaxSweeps && !jac && !g.faces && !sym && !pr;
    // use_e = false: no prolongation in the pass (y0 = Xold, prolongated beforehand by k_prolong):
    // no W ring, no E tiles, the tensor warps only copy the x_old rows
    auto march = [&](const double* Xold, double* Yv, const double* rhs, double rconst, bool last,
                     int init, bool use_e = true) {
        SmoothMarchArgs a{};
        const int TX = march_tx(Bp);
        a.g = g; a.Bp = Bp; a.npad = use_e ? npad : 0; a.ldw = use_e ? ctx->ldw : 0;
        a.part = march_part(g, TX, ctx->num_sms);
        a.W = ctx->Wi; a.E = L.E; a.Xold = Xold; a.Rhs = rhs; a.rconst = rconst; a.Y = Yv;
        a.theta = L.theta; a.active = L.active; a.S = (int)seq.size();
        for (size_t t = 0; t < seq.size(); ++t) a.seq[t] = seq[t];
        a.has_e = use_e && npad > 0; a.last = last; a.init = init; a.s = S; a.done = done;
        pb(RBS_K_GS);
        const size_t kMaxDyn = (size_t)kSmooth2MaxDyn;
        // strip 32 with the 3-row W ring; else strip 32 with a 2-row ring (prefetch distance
        // 1; keeps ~all SMs busy at large m, e.g. 2047: 64 strips x 2 segments against 86 x 1
        // at strip 24); else strip 24
        int var = 0, TX2 = 32;
        const bool hr = rhs != nullptr, ax = Xold != nullptr;
        size_t sm2 = Smooth2Smem(32, a.S, Bp, a.ldw, Q, hr, ax, a.npad, 3).total;
        if (sm2 > kMaxDyn) {
            var = 1;
            sm2 = Smooth2Smem(32, a.S, Bp, a.ldw, Q, hr, ax, a.npad, 2).total;
        }
        if (sm2 > kMaxDyn || (v2off & 128)) {
            var = 2;
            TX2 = 24;
            sm2 = Smooth2Smem(24, a.S, Bp, a.ldw, Q, hr, ax, a.npad, 3).total;
        }
        if (!(v2off & 1) && Bp <= 32 && a.S <= 3 && sm2 <= kMaxDyn) {
            // v2: lagged one-barrier-per-row pipeline (march2.cuh)
            a.part = march_part(g, TX2, ctx->num_sms);
            const int grid2 = a.part.nsx * a.part.nsy;
            if (Bp == 8) launch_smooth2<8>(var, a.S, grid2, sm2, st, a, v2off);
            else if (Bp == 16) launch_smooth2<16>(var, a.S, grid2, sm2, st, a, v2off);
            else launch_smooth2<32>(var, a.S, grid2, sm2, st, a, v2off);
            pe();
            return 1;
        }
        const int grid = a.part.nsx * a.part.nsy;
        if (TX == 32) {
            SmoothSmem<32> sl(Bp, npad, ctx->ldw, Q, a.S, rhs != nullptr, Xold != nullptr);
            k_smooth_march<32><<<grid, kMarchThreads, sl.total, st>>>(a);
        } else {
            SmoothSmem<16> sl(Bp, npad, ctx->ldw, Q, a.S, rhs != nullptr, Xold != nullptr);
            k_smooth_march<16><<<grid, kMarchThreads, sl.total, st>>>(a);
        }
        pe();
        return 1;
    };

    // symmetric two-level preconditioner y = M^{-1} r (RBS_PRECOND_SYM, NEXT(3)):
    // y1 = S*(A, r, 0), y2 = y1 + W A_n^{-1} W^T (r - A y1), y = S(A, r, y2) (+ Step 10)
    auto precond_sym = [&](int init) {
        int c = 0;
        c += smooth(L.Y, L.R, 0.0, false, init, &rseq, true);     // pre: the adjoint sweep from 0
        if (npad > 0) {
            c += proj(MODE_RESID, nullptr, true, L.Y, L.R);        // W^T (r - A y1)
            pb(RBS_K_REDUCE_SOLVE);
            k_reduce_solve<<<Bp, kRsThreads, 0, st>>>(S, init ? 2 : 1);   // e (no stop test)
            pe();
            ++c;
            c += prolong(L.Y, 1, first_col);                       // y2 = y1 + W e
        }
        c += smooth(L.Y, L.R, 0.0, true, init);                    // post; Step 10 in the last CTA
        return c;
    };
    // Polak-Ribiere beta (RBS_BETA_PR): r_k kept before Step 7, rho_k before Step 10;
    // after it beta = (rho_{k+1} - y_{k+1}^T r_k) / rho_k
    auto pr_fix = [&]() {
        k_dot_pr<<<nctf, 256, 0, st>>>(L.Y, L.Rold, g.N, Bp, S);
        k_beta_pr<<<1, 256, 0, st>>>(S, L.rho_prev, nctf);
        return 2;
    };

    // ---- RBCG Step 2-3: y_0 = RBI(A, r_0, W, 1), rho_0 = r_0^T y_0 ------------
    if (cg) {
        if (sym) launches += precond_sym(1);
        else if (use_march) launches += march(nullptr, L.Y, L.R, 0.0, true, 1);   // + rho_0, PRECOND
        else if (jac) {
            double* y0b = (o->sweeps & 1) ? L.T : L.Y;
            launches += prolong(y0b, 0);
            launches += smooth_jac(y0b, L.Y, L.R, 0.0, true, 1);
        } else {
            launches += prolong(L.Y, 0, first_col);
            launches += smooth(L.Y, L.R, 0.0, true, 1);
        }
        CKL();
    } else {
        k_update_done<<<1, 1, 0, st>>>(L.active, Bp, done);
        ++launches;
        CKL();
    }

    // ---- iteration body, captured once per configuration --------------------
    int per_iter = 0;
    auto body = [&](int it) {
        int c = 0;
        if (cg) {
            double* Pold = (it & 1) ? L.P1 : L.P0;
            double* Pnew = (it & 1) ? L.P0 : L.P1;
            c += cgp(Pold, Pnew);             // Step 11 (prev) + A p, Step 5 (alpha) in last CTA
            if (pr) cudaMemcpyAsync(L.Rold, L.R, (size_t)vecN * 8, cudaMemcpyDeviceToDevice, st);   // r_k
            c += proj(MODE_CG, Pnew, true);   // Steps 6-7, ||r||, W^T r
            pb(RBS_K_REDUCE_SOLVE);
            launch_k(pdl && use_march, k_reduce_solve, Bp, kRsThreads, 0, st, S, 0);   // Step 8
            pe();
            ++c;
            if (pr) cudaMemcpyAsync(L.rho_prev, L.rho, (size_t)Bp * 8, cudaMemcpyDeviceToDevice, st);  // rho_k
            if (sym) {
                c += precond_sym(0);                           // Step 9 (two-level) + Step 10
            } else if (use_march) {
                c += march(nullptr, L.Y, L.R, 0.0, true, 0);   // Step 9 + Step 10 (last CTA)
            } else if (jac) {
                double* y0b = (o->sweeps & 1) ? L.T : L.Y;
                c += prolong(y0b, 0);                          // Step 9: y0 = W e
                c += smooth_jac(y0b, L.Y, L.R, 0.0, true, 0);  // Jacobi sweeps; Step 10
            } else {
                c += prolong(L.Y, 0, first_col);  // Step 9: y0 = W e
                c += smooth(L.Y, L.R, 0.0, true, 0);  // y = S(A, r, y0); Step 10 in last CTA
            }
            if (pr) c += pr_fix();
        } else if (use_march) {
            double* Xi = (it & 1) ? L.X2 : L.X;     // ping-pong: the march reads halos of x_old
            double* Xo = (it & 1) ? L.X : L.X2;
            c += march(Xi, Xo, Fv, ctx->fconst, false, 0);      // Steps 6-7
            c += proj(MODE_RESID, nullptr, true, Xo);           // Steps 2, 4
            pb(RBS_K_REDUCE_SOLVE); k_reduce_solve<<<Bp, kRsThreads, 0, st>>>(S); pe(); ++c;  // Steps 3, 5
        } else {
            c += prolong(L.X, 1, first_col);                    // Step 6
            c += smooth(L.X, Fv, ctx->fconst, false, 0);        // Step 7
            c += proj(MODE_RESID, nullptr, true);               // Steps 2, 4
            pb(RBS_K_REDUCE_SOLVE); k_reduce_solve<<<Bp, kRsThreads, 0, st>>>(S); pe(); ++c;  // Steps 3, 5
        }
        return c;
    };
    const int chunk = o->graph_chunk;
    char keybuf[512];
    // the key names every carved pointer the graph holds (the layout moves with
    // x_location / rhs / history), so a reused workspace never replays stale pointers
    snprintf(keybuf, sizeof keybuf, "%p|%p|%d|%d|%d|%d|%d|%d|%d|%.17g|%.17g|%d|%p|%p|%p|%d|%d|%d|%.17g|%d|%.17g|%.17g"
             "|%d|%p|%p|%p|%p|%p",
             workspace_dev, (void*)Fv, B, Bp, o->method, o->smoother, o->sweeps, o->max_iter, chunk,
             o->tol, o->delta, o->record_history, (void*)ctx->Wi, (void*)st, (void*)L.hist,
             rhs_dev ? 1 : 0, n, npad, ctx->fconst, o->n_active, o->gamma, o->omega,
             o->x_location, (void*)L.theta, (void*)L.partP, (void*)L.partF, (void*)L.ints, (void*)L.X);
    const std::string key = std::string(keybuf) + "|" + std::to_string(o->precond) + "|" +
                            std::to_string(o->beta_rule) + "|" + std::to_string((uintptr_t)L.Rold);
    if (prof) {
        // eager launches, one iteration at a time, events on the launching stream
        volatile int* hf = ctx->h_flag;
        for (int64_t it = 0; it <= (int64_t)o->max_iter + 1; ++it) {
            pne = 0;
            pcls.clear();
            launches += body((int)(it & 1));
            CKL();
            CK(cudaMemcpyAsync((void*)ctx->h_flag, done, sizeof(int), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            const bool fin = hf[0] != 0;
            if (!fin)  // only complete iterations (no early-exit launches) are accumulated
                for (int e = 0; e < pne; ++e) {
                    float ms = 0.f;
                    CK(cudaEventElapsedTime(&ms, ctx->pev[2 * e], ctx->pev[2 * e + 1]));
                    ctx->prof_ms[pcls[e]] += ms;
                    ctx->prof_cnt[pcls[e]] += 1;
                }
            if (fin) break;
        }
    } else if (!ctx->gexec || ctx->gkey != key) {
        if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; }
        cudaStream_t cap;
        CK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
        cudaGraph_t graph;
        CK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
        cudaStream_t keep = st;
        st = cap;
        per_iter = 0;
        for (int it = 0; it < chunk; ++it) per_iter += body(it);
        st = keep;
        CK(cudaStreamEndCapture(cap, &graph));
        CK(cudaGraphInstantiate(&ctx->gexec, graph, 0));
        cudaGraphDestroy(graph);
        cudaStreamDestroy(cap);
        ctx->gkey = key;
        ctx->g_per_chunk = per_iter;
    } else {
        per_iter = ctx->g_per_chunk;
    }
    CKL();

    // ---- replay until every query is frozen ---------------------------------
    const int64_t max_launch = (int64_t)o->max_iter / chunk + 3;
    volatile int* hf = ctx->h_flag;
    hf[0] = hf[1] = 0;
    for (int64_t l = 0; !prof; ++l) {
        CK(cudaGraphLaunch(ctx->gexec, st));
        launches += per_iter;
        CK(cudaMemcpyAsync((void*)(ctx->h_flag + (l & 1)), done, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(ctx->ev[l & 1], st));
        if (l >= 1) {
            CK(cudaEventSynchronize(ctx->ev[(l - 1) & 1]));
            if (hf[(l - 1) & 1]) break;
        }
        if (l > max_launch) break;
    }
    CK(cudaStreamSynchronize(st));

    // ---- outputs --------------------------------------------------------------
    std::vector<int> hs(Bp), hi(Bp), hp(Bp);
    std::vector<double> hrel(Bp), hfn(Bp), tr(Bp, NAN);
    CK(cudaMemcpyAsync(hs.data(), L.status, Bp * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hi.data(), L.its, Bp * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hp.data(), L.pivot, Bp * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hrel.data(), L.relres, Bp * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hfn.data(), L.fnorm, Bp * 8, cudaMemcpyDeviceToHost, st));
    ctx->last_na.assign(Bp, n);
    CK(cudaMemcpyAsync(ctx->last_na.data(), L.na, Bp * 4, cudaMemcpyDeviceToHost, st));
    if (cg) {
        // true residual ||f - A x|| / ||f|| (not used for stopping)
        proj(MODE_RESID, nullptr, false);
        ++launches;
        // reuse npad rows: the rr row of the partials is row npad
        k_reduce_rows<<<Bp, 128, 0, st>>>(L.partP, npad + 1, nct_plain, L.fproj);
        ++launches;
        CKL();
        std::vector<double> rows((size_t)Bp * (npad + 1));
        CK(cudaMemcpyAsync(rows.data(), L.fproj, rows.size() * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int b = 0; b < Bp; ++b) tr[b] = std::sqrt(rows[(size_t)b * (npad + 1) + npad]) / hfn[b];
    } else {
        CK(cudaStreamSynchronize(st));
        for (int b = 0; b < Bp; ++b) tr[b] = hrel[b];
    }
    // X: [N8][Bp] -> [B][N]
    double* xdst = o->x_location == RBS_MEM_HOST ? L.Xout : X;
    const double* Xfin = L.X;
    if (L.X2 && use_march) {  // RBI ping-pong: corrections applied so far decide the buffer
        int kc = 0;
        CK(cudaMemcpyAsync(&kc, kcount, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        Xfin = (kc & 1) ? L.X2 : L.X;
    }
    k_transpose_out<<<(unsigned)((g.N + 31) / 32), 256, 0, st>>>(Xfin, g.N, Bp, B, xdst, g.N);
    ++launches;
    CKL();
    if (o->x_location == RBS_MEM_HOST)
        CK(cudaMemcpyAsync(X, L.Xout, (size_t)B * g.N * 8, cudaMemcpyDeviceToHost, st));
    if (a_n && n > 0) {
        std::vector<double> ha((size_t)Bp * npad);
        CK(cudaMemcpyAsync(ha.data(), L.a_n, ha.size() * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int b = 0; b < B; ++b)
            for (int j = 0; j < n; ++j) a_n[(size_t)b * n + j] = ha[(size_t)b * npad + j];
    }
    if (history && L.hist)
        CK(cudaMemcpyAsync(history, L.hist, (size_t)B * (o->max_iter + 1) * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ctx->last_na.resize(B);
    for (int b = 0; b < B; ++b) {
        if (iters) iters[b] = hi[b];
        if (qstatus) qstatus[b] = hs[b];
        if (relres) relres[b] = hrel[b];
        if (true_relres) true_relres[b] = tr[b];
    }
    for (int b = 0; b < B; ++b)
        if (hs[b] == Q_NOT_SPD) {
            char buf[128];
            snprintf(buf, sizeof buf, "reduced matrix not SPD: query %d, pivot %d", b, hp[b]);
            ctx->err = buf;
            break;
        }
    ctx->launches = launches;
    return RBS_OK;
}


// Public entry.  2D grids run the row-march kernels with at most 32 queries per
// pass (their shared-memory rings hold 32-query rows); a larger batch is solved
// as independent sub-batches of 32 -- every query's iteration is independent of
// the others (per-query alpha, beta, stop test), so the results are the same.
rbs_status rbs_solve_batch(rbs_ctx* ctx, int B, const double* mu_host, const rbs_solve_opts* o,
                           const double* rhs_dev, double* X, int* iters, int* qstatus,
                           double* relres, double* true_relres, double* a_n, double* history,
                           void* workspace_dev, size_t workspace_bytes, void* stream) {
    if (!ctx) return RBS_E_ARG;
    // parameter map: theta_q(mu) and phi_r(mu) per query, on the host
    std::vector<double> th, ph;
    const double* thp = mu_host;
    const double* php = nullptr;
    if (ctx->has_op && mu_host && B >= 1 && B <= RBS_MAX_BATCH) {
        const int Q = ctx->g.Q, R = ctx->R, P = ctx->P > 0 ? ctx->P : Q;
        if (!ctx->Ta.empty()) {
            th.assign((size_t)B * Q, 0.0);
            for (int b = 0; b < B; ++b)
                for (int q = 0; q < Q; ++q) {
                    const double* row = ctx->Ta.data() + (size_t)q * (P + 1);
                    double v = row[0];
                    for (int k = 0; k < P; ++k) v += row[k + 1] * mu_host[(size_t)b * P + k];
                    th[(size_t)b * Q + q] = v;
                }
            thp = th.data();
        }
        if (R > 0) {
            ph.assign((size_t)B * R, 1.0);
            if (!ctx->Pa.empty())
                for (int b = 0; b < B; ++b)
                    for (int r = 0; r < R; ++r) {
                        const double* row = ctx->Pa.data() + (size_t)r * (P + 1);
                        double v = row[0];
                        for (int k = 0; k < P; ++k) v += row[k + 1] * mu_host[(size_t)b * P + k];
                        ph[(size_t)b * R + r] = v;
                    }
            php = ph.data();
        }
    }
    if (!ctx->has_op || ctx->g.dim != 2 || B <= 32 || B > RBS_MAX_BATCH || !mu_host || !X || !o)
        return solve_batch_impl(ctx, B, thp, php, o, rhs_dev, X, iters, qstatus, relres, true_relres, a_n,
                                history, workspace_dev, workspace_bytes, stream);
    const int64_t N = ctx->g.N;
    const int P = ctx->g.Q, nb = ctx->n, hl = o->max_iter + 1, Rr = ctx->R;
    int64_t total = 0;
    std::vector<int> na_all;
    for (int c0 = 0; c0 < B; c0 += 32) {
        const int b = std::min(32, B - c0);
        rbs_status s = solve_batch_impl(
            ctx, b, thp + (size_t)c0 * P, php ? php + (size_t)c0 * Rr : nullptr, o,
            rhs_dev ? rhs_dev + (size_t)c0 * N : nullptr,
            X + (size_t)c0 * N, iters ? iters + c0 : nullptr, qstatus ? qstatus + c0 : nullptr,
            relres ? relres + c0 : nullptr, true_relres ? true_relres + c0 : nullptr,
            a_n ? a_n + (size_t)c0 * nb : nullptr, history ? history + (size_t)c0 * hl : nullptr,
            workspace_dev, workspace_bytes, stream);
        total += ctx->launches;
        if (s != RBS_OK) return s;
        na_all.insert(na_all.end(), ctx->last_na.begin(), ctx->last_na.begin() + b);
    }
    ctx->launches = total;
    ctx->last_na = na_all;
    return RBS_OK;
}

}  // extern "C"

#include "greedy.inc.cu"
