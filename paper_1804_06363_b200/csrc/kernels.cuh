// kernels.cuh -- sm_100a kernels of the batched RB online solver.
//
// Every streaming pass works on node-major batch vectors v[N8][Bp] (lane =
// query, 8*Bp bytes per node contiguous) so that a warp's loads are fully
// coalesced.  The W-contractions (projection W^T r, eq5;
// prolongation W e, eq7) run on the FP64 tensor cores
// (mma.sync m8n8k4 f64 -> SASS DMMA): tcgen05 has no f64 kind on sm_100a.
// Reductions are deterministic two-stage sums (fixed CTA partition, fixed
// in-CTA order, fixed stage-2 order): bitwise reproducible run to run.
// Streaming passes are latency-bound unless each thread keeps several
// independent loads in flight: loops are unrolled with every load of the
// unrolled group issued before any arithmetic that consumes it.
// The tiny scalar steps (alpha, beta, stop tests) are folded into the
// last CTA of the producing pass (atomic ticket), not separate launches.
#pragma once
#include "rbs_internal.cuh"

namespace rbs {

enum { MODE_CG = 0, MODE_RESID = 1, MODE_PLAIN = 2 };
enum { Q_CONVERGED = 0, Q_MAXIT = 1, Q_NOT_SPD = 2, Q_CURVATURE = 3, Q_PRECOND = 4,
       Q_NONFINITE = 5 };

constexpr int kFlat = 512;     // threads per CTA of the flat (thread-per-element) passes

// ---------------------------------------------------------------------------
// Per-solve state shared by the bookkeeping steps.
// ---------------------------------------------------------------------------
struct SolveState {
    int B, Bp, n, npad, nct, nctf, maxit, method;
    double tol, delta;
    const double* ANq;        // [Q][npad][npad]
    int Q;
    double* theta;            // [Q][Bp]
    double* fproj;            // [Bp][npad+1]: f_n and ||f||^2
    double* L;                // [Bp][npad][npad]
    double* Ainv;             // [Bp][npad][npad]: A_n(mu)^{-1} ("invert the RB matrix")
    double* E;                // [npad][Bp]
    double* a_n;              // [Bp][npad]
    double* partP;            // [Bp][npad+1][nct]
    double* partF;            // [Bp][2][nctf]
    double *alpha, *beta, *rho, *rr, *fnorm, *relres;
    int *active, *status, *its, *pivot;
    int* kcount;
    int* done;
    unsigned* ticket;
    double* hist;             // [Bp][maxit+1] or nullptr
    int* na;                  // [Bp] active RB dimension per query
    int na0;                  // its start value (n_active, or n)
    int tri;                  // 1: reduced solves by the leading block of L (n_active < n or gamma)
    double gamma;             // RBCG adaptive-n rule, 0 = off
};

__device__ __forceinline__ int ld_flag(const int* p) { return *(volatile const int*)p; }

// deterministic warp sum of p[0..cnt) (4 independent loads in flight per lane)
__device__ __forceinline__ double warp_sum_row(const double* p, int cnt, int lane) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int c = lane;
    for (; c + 96 < cnt; c += 128) {
        s0 += __ldcg(p + c);
        s1 += __ldcg(p + c + 32);
        s2 += __ldcg(p + c + 64);
        s3 += __ldcg(p + c + 96);
    }
    for (; c < cnt; c += 32) s0 += __ldcg(p + c);
    double s = (s0 + s1) + (s2 + s3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// triangular solves L L^T e = rhs by one warp; lane owns rows lane, lane+32.
__device__ void warp_chol_solve(const double* L, int ld, int n, double* z0, double* z1, int lane) {
    for (int i = 0; i < n; ++i) {
        const int own = i & 31, slot = i >> 5;
        const double mine = slot ? *z1 : *z0;
        const double zi = __shfl_sync(0xffffffffu, mine, own) / L[i * ld + i];
        if (lane == own) { if (slot) *z1 = zi; else *z0 = zi; }
        if (lane > i && lane < n) *z0 -= L[lane * ld + i] * zi;
        if (lane + 32 > i && lane + 32 < n) *z1 -= L[(lane + 32) * ld + i] * zi;
    }
    for (int i = n - 1; i >= 0; --i) {
        const int own = i & 31, slot = i >> 5;
        const double mine = slot ? *z1 : *z0;
        const double ei = __shfl_sync(0xffffffffu, mine, own) / L[i * ld + i];
        if (lane == own) { if (slot) *z1 = ei; else *z0 = ei; }
        if (lane < i) *z0 -= L[i * ld + lane] * ei;
        if (lane + 32 < i) *z1 -= L[i * ld + lane + 32] * ei;
    }
}

// Atomic ticket: returns true in exactly one thread (threadIdx.x == 0) of the
// CTA that finishes last; all earlier CTAs' global writes are then visible.
__device__ __forceinline__ bool cta_is_last(unsigned* ticket, int* s_last) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned t = atomicAdd(ticket, 1u);
        *s_last = (t == gridDim.x - 1);
        if (*s_last) __threadfence();
    }
    __syncthreads();
    return *s_last != 0;
}

__device__ __forceinline__ void release_ticket(unsigned* ticket) {
    if (threadIdx.x == 0) {
        *(volatile unsigned*)ticket = 0u;
        __threadfence();
    }
}

// any query still active?  (whole CTA; one load per thread, no serial chain)
__device__ __forceinline__ int cta_any_active(const SolveState& s) {
    const int v = (int)threadIdx.x < s.Bp ? __ldcg(s.active + threadIdx.x) : 0;
    return __syncthreads_or(v);
}

__device__ __forceinline__ void update_done(const SolveState& s) {
    const int any = cta_any_active(s);
    if (threadIdx.x == 0) *(volatile int*)s.done = any ? 0 : 1;
}

// sum over the CTAs' partials part[(b*2+slot)*nctf + c] for every query b;
// result in s_out[b].  Whole CTA participates (blockDim.x multiple of Bp).
// (the producing kernel's own CTAs: gridDim.x columns, row stride s.nctf)
__device__ void cta_sum_slot(const SolveState& s, int slot, double* s_buf, double* s_out, int cnt = -1) {
    const int gsz = blockDim.x / s.Bp;
    const int b = threadIdx.x / gsz, t = threadIdx.x - b * gsz;
    if (cnt < 0) cnt = gridDim.x;
    double v0 = 0.0, v1 = 0.0;
    const double* p = s.partF + ((int64_t)b * 2 + slot) * s.nctf;
    int c = t;
    for (; c + gsz < cnt; c += 2 * gsz) {
        v0 += __ldcg(p + c);
        v1 += __ldcg(p + c + gsz);
    }
    if (c < cnt) v0 += __ldcg(p + c);
    s_buf[threadIdx.x] = v0 + v1;
    __syncthreads();
    if (t == 0) {
        double a = 0.0;
        for (int u = 0; u < gsz; ++u) a += s_buf[b * gsz + u];
        s_out[b] = a;
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Projection family: per node-query value v (mode-dependent), then
//   part[b][j][cta] = sum_{nodes of cta} W[i][j] v[i][b]   (j < npad)
//   part[b][npad][cta] = sum v[i][b]^2
// MODE_CG   (RBCG Steps 6-8): q = A p (recomputed from the
//           p halo), x += alpha p, r -= alpha q, v = r (stored).
// MODE_RESID (RBI Step 2): v = b - A x (not stored).
// MODE_PLAIN: v = V (or the constant vconst).
// Warp layout = DMMA B-fragment: lane l owns node 4g + (l&3), query 8bt + (l>>2).
// Two node groups per warp iteration, all loads of both issued first.
// ---------------------------------------------------------------------------
struct ProjArgs {
    Geo g;
    int Bp, npad, nct;
    int ldw;                  // row stride of W (npad + 4: conflict-free DMMA fragments)
    int64_t ngroups;          // ceil(N/4)
    const double* W;          // [N8][npad]
    const double* theta;      // [Q][Bp]
    const int* active;        // [Bp] or nullptr (all active)
    const double* alpha;      // [Bp] (MODE_CG)
    const double* P;          // MODE_CG
    double* X;                // MODE_CG (rw), MODE_RESID (r)
    double* R;                // MODE_CG (rw)
    const double* V;          // MODE_RESID rhs / MODE_PLAIN input, or nullptr
    double vconst;
    double* part;             // [Bp][npad+1][nct]
    const int* done;
    int col0;                 // first partial column of this launch (mesh slabs)
};

template <int MODE, int DIM>
__device__ __forceinline__ void proj_load(const ProjArgs& a, const double* s_th, int b, int64_t i,
                                          bool ok, double* nb, double& c0, double& c1, double& c2,
                                          int& I, int& J, int& K) {
    if (!ok) return;
    const int64_t e = i * a.Bp + b;
    if (MODE == MODE_PLAIN) {
        c0 = a.V ? __ldg(a.V + e) : a.vconst;
        return;
    }
    node_coords(a.g, (uint32_t)i, I, J, K);
    if (MODE == MODE_CG) {
        c0 = __ldg(a.P + e);
        node_nbrs<DIM>(a.g, a.P, a.Bp, i, b, I, J, K, nb);
        c1 = a.X[e];
        c2 = a.R[e];
    } else {
        c0 = a.X[e];
        node_nbrs<DIM>(a.g, a.X, a.Bp, i, b, I, J, K, nb);
        c1 = a.V ? __ldg(a.V + e) : a.vconst;
    }
}

template <int MODE, int DIM>
__device__ __forceinline__ double proj_value(const ProjArgs& a, const double* s_th, double al,
                                             int b, int64_t i, bool ok, const double* nb,
                                             double c0, double c1, double c2, int I, int J, int K) {
    if (!ok) return 0.0;
    if (MODE == MODE_PLAIN) return c0;
    double k[2 * DIM];
    node_kappa<DIM>(a.g, s_th, a.Bp, b, I, J, K, k);
    const double q = stencil_apply<DIM>(a.g, k, c0, nb);
    const int64_t e = i * a.Bp + b;
    if (MODE == MODE_CG) {
        const double xv = fma(al, c0, c1);
        const double rv = fma(-al, q, c2);
        a.X[e] = xv;
        a.R[e] = rv;
        return DIM == 3 && !owned(a.g, K) ? 0.0 : rv;     // slab ghost planes: not reduced
    }
    return DIM == 3 && !owned(a.g, K) ? 0.0 : c1 - q;
}

template <int MODE, int DIM>
__global__ void __launch_bounds__(kThreads, 2) k_proj(ProjArgs a) {
    if (a.done && ld_flag(a.done)) return;
    extern __shared__ double smem[];
    const int Bp = a.Bp, npad = a.npad, nbt = Bp >> 3, ntile = npad >> 3;
    const int nlc = 8 / nbt;  // node lanes per CTA
    double* s_th = smem;
    double* s_alpha = s_th + a.g.Q * Bp;
    double* s_red = s_alpha + Bp;
    int* s_act = (int*)(s_red + nlc * (npad + 1) * Bp);
    const int tid = threadIdx.x;
    if (MODE != MODE_PLAIN)
        for (int t = tid; t < a.g.Q * Bp; t += kThreads) s_th[t] = a.theta[t];
    for (int t = tid; t < Bp; t += kThreads) {
        s_alpha[t] = (MODE == MODE_CG) ? a.alpha[t] : 0.0;
        s_act[t] = a.active ? a.active[t] : 1;
    }
    __syncthreads();

    const int warp = tid >> 5, lane = tid & 31;
    const int bt = warp % nbt, nl = warp / nbt;
    const int b = bt * 8 + (lane >> 2);
    const bool wact = nl < nlc;
    const bool qact = s_act[b] != 0;
    const double al = s_alpha[b];
    const int64_t g0 = (a.ngroups * blockIdx.x) / gridDim.x;
    const int64_t g1 = (a.ngroups * (blockIdx.x + 1)) / gridDim.x;

    double acc[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) acc[t] = 0.0;
    double rr = 0.0;
    if (wact) {
        for (int64_t gi = g0 + nl; gi < g1; gi += 2 * nlc) {
            const int64_t gB = gi + nlc;
            const int64_t iA = gi * 4 + (lane & 3), iB = gB * 4 + (lane & 3);
            const bool okA = iA < a.g.N && qact, okB = gB < g1 && iB < a.g.N && qact;
            double nbA[2 * DIM], nbB[2 * DIM];
            double a0 = 0, a1 = 0, a2 = 0, b0 = 0, b1 = 0, b2 = 0;
            int IA = 1, JA = 1, KA = 1, IB = 1, JB = 1, KB = 1;
            proj_load<MODE, DIM>(a, s_th, b, iA, okA, nbA, a0, a1, a2, IA, JA, KA);
            proj_load<MODE, DIM>(a, s_th, b, iB, okB, nbB, b0, b1, b2, IB, JB, KB);
            double wA[8], wB[8];
            const double* wrowA = a.W + iA * a.ldw + (lane >> 2);
            const double* wrowB = a.W + (gB < g1 ? iB : iA) * a.ldw + (lane >> 2);
#pragma unroll
            for (int jt = 0; jt < 8; ++jt)
                if (jt < ntile) {
                    wA[jt] = __ldg(wrowA + jt * 8);
                    wB[jt] = __ldg(wrowB + jt * 8);
                }
            const double vA = proj_value<MODE, DIM>(a, s_th, al, b, iA, okA, nbA, a0, a1, a2, IA, JA, KA);
            const double vB = proj_value<MODE, DIM>(a, s_th, al, b, iB, okB, nbB, b0, b1, b2, IB, JB, KB);
            rr = fma(vA, vA, rr);
            rr = fma(vB, vB, rr);
#pragma unroll
            for (int jt = 0; jt < 8; ++jt)
                if (jt < ntile) {
                    dmma_8x8x4(acc[2 * jt], acc[2 * jt + 1], wA[jt], vA);
                    dmma_8x8x4(acc[2 * jt], acc[2 * jt + 1], wB[jt], vB);
                }
        }
    }
    // rr of query b: lanes sharing l>>2 (fixed order)
    rr += __shfl_xor_sync(0xffffffffu, rr, 1);
    rr += __shfl_xor_sync(0xffffffffu, rr, 2);
    if (wact) {
        const int rowbase = nl * (npad + 1);
#pragma unroll
        for (int jt = 0; jt < 8; ++jt)
            if (jt < ntile) {
                const int j = jt * 8 + (lane >> 2);
                const int bb = bt * 8 + 2 * (lane & 3);
                s_red[(rowbase + j) * Bp + bb] = acc[2 * jt];
                s_red[(rowbase + j) * Bp + bb + 1] = acc[2 * jt + 1];
            }
        if ((lane & 3) == 0) s_red[(rowbase + npad) * Bp + b] = rr;
    }
    __syncthreads();
    const int rows = npad + 1;
    for (int t = tid; t < rows * Bp; t += kThreads) {
        const int j = t / Bp, bb = t - j * Bp;
        double s = s_red[j * Bp + bb];
        for (int l = 1; l < nlc; ++l) s += s_red[(l * rows + j) * Bp + bb];
        a.part[((int64_t)bb * rows + j) * a.nct + a.col0 + blockIdx.x] = s;
    }
}

// ---------------------------------------------------------------------------
// RBCG Steps 6-7 for 3D grids in row segments (the first half of K2 in two passes):
// x += alpha p, r -= alpha A p with the p window and the y/z
// neighbours of a segment loaded together; the projection W^T r and ||r||^2 follow
// in k_proj<MODE_PLAIN> on the updated r.  Per node the same arithmetic as
// k_proj<MODE_CG, 3>.  Requires Bp <= 32; no mesh slabs (all planes owned).
// ---------------------------------------------------------------------------
template <int SEG, bool FACES>
__global__ void __launch_bounds__(kFlat, SEG <= 2 ? 2 : 1) k_xr3r(ProjArgs a, int lgB) {
    if (a.done && ld_flag(a.done)) return;
    extern __shared__ double smem[];
    double* s_th = smem;
    int* s_act = (int*)(s_th + a.g.Q * a.Bp);
    for (int t = threadIdx.x; t < a.g.Q * a.Bp; t += kFlat) s_th[t] = a.theta[t];
    for (int t = threadIdx.x; t < a.Bp; t += kFlat) s_act[t] = a.active[t];
    __syncthreads();
    const Geo& g = a.g;
    const int Bp = a.Bp, m = g.m;
    const int lane = threadIdx.x & 31, rpw = 32 >> lgB;
    const int sub = lane >> lgB, b = lane & (Bp - 1);
    const int nseg = (m + SEG - 1) / SEG;
    const int64_t items = (int64_t)m * g.mz * nseg;
    const int64_t nw = ((int64_t)gridDim.x * kFlat) >> 5;
    const int64_t w0 = (blockIdx.x * (int64_t)kFlat + threadIdx.x) >> 5;
    const int64_t sy = (int64_t)m * Bp, sz = sy * m;
    if (!s_act[b]) return;
    const double al = a.alpha[b];
    for (int64_t it = w0 * rpw + sub; it < items; it += nw * rpw) {
        const int64_t row = it / nseg;
        const int x0 = 1 + (int)(it - row * nseg) * SEG;
        const int J = (int)(row % m) + 1, Kl = (int)(row / m), K = Kl + 1 + g.kofs;
        const int64_t rb = ((int64_t)Kl * m * m + (int64_t)(J - 1) * m) * Bp + b;
        const bool hym = J > 1, hyp = J < m, hzm = has_zm(g, K), hzp = has_zp(g, K);
        double pw[SEG + 2], q[SEG][4], xv[SEG], rv[SEG];
#pragma unroll
        for (int j = 0; j < SEG + 2; ++j) {
            const int x = x0 - 1 + j;
            pw[j] = (x >= 1 && x <= m) ? __ldg(a.P + rb + (int64_t)(x - 1) * Bp) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < SEG; ++j) {
            const int x = x0 + j;
            const int64_t e = rb + (int64_t)(x - 1) * Bp;
            const bool in = x <= m;
            q[j][0] = in && hym ? __ldg(a.P + e - sy) : 0.0;
            q[j][1] = in && hyp ? __ldg(a.P + e + sy) : 0.0;
            q[j][2] = in && hzm ? __ldg(a.P + e - sz) : 0.0;
            q[j][3] = in && hzp ? __ldg(a.P + e + sz) : 0.0;
            xv[j] = in ? a.X[e] : 0.0;
            rv[j] = in ? a.R[e] : 0.0;
        }
        const int by0 = axis_block(g, J - 1, g.py) * g.px, by1 = axis_block(g, J, g.py) * g.px;
        const int pxy = g.px * g.py;
        const int bz0 = axis_block(g, K - 1, g.pz) * pxy, bz1 = axis_block(g, K, g.pz) * pxy;
        const bool rowu = !g.faces && by0 == by1 && bz0 == bz1;
#pragma unroll
        for (int j = 0; j < SEG; ++j) {
            const int x = x0 + j;
            if (x > m) break;
            double k[6];
            const int bxl = axis_block(g, x - 1, g.px), bxr = axis_block(g, x, g.px);
            if (FACES) {
                node_kappa_faces<3>(g, s_th, Bp, b, x, J, K, k);
            } else if (rowu && bxl == bxr) {
                const double c = s_th[(bxr + by0 + bz0) * Bp + b];
#pragma unroll
                for (int e = 0; e < 6; ++e) k[e] = c;
            } else {
                node_kappa3_call(g, s_th, Bp, b, x, J, K, k);
            }
            const double nb[6] = {pw[j], pw[j + 2], q[j][0], q[j][1], q[j][2], q[j][3]};
            const double qv = stencil_apply<3>(g, k, pw[j + 1], nb);
            const int64_t e = rb + (int64_t)(x - 1) * Bp;
            a.X[e] = fma(al, pw[j + 1], xv[j]);
            a.R[e] = fma(-al, qv, rv[j]);
        }
    }
}

// ---------------------------------------------------------------------------
// Prolongation  Y = W E  (or Y += W E), PAPER.md:144-147 (eq7) / 165.
// DMMA with M = 8 nodes, N = 8 queries, K = 4 basis vectors.  Each warp owns
// one query tile (its E fragments stay in registers) and runs two node tiles
// as independent accumulator chains.
// ---------------------------------------------------------------------------
struct ProlongArgs {
    int64_t N;
    int Bp, npad, ldw;
    const double* W;      // [N8][npad]
    const double* E;      // [npad][Bp]
    const int* active;    // [Bp]
    double* Y;            // [N8][Bp]
    int accumulate;
    const int* done;
    // skip_color >= 0: nodes of that red-black colour are not prolongated -- the
    // smoother's first half-sweep (that colour) overwrites them without reading them
    // (direct form, AMB-6), so their W rows are not loaded and y is not written there
    int skip_color, dim, m, kofs;
    FastDiv fm;
};

__device__ __forceinline__ void prolong_store(const ProlongArgs& a, int64_t i, int b, double d0,
                                              double d1, bool act0, bool act1) {
    if (i >= a.N) return;
    double* y = a.Y + i * a.Bp + b;
    if (act0 && act1) {
        double2 v = make_double2(d0, d1);
        if (a.accumulate) {
            const double2 o = *reinterpret_cast<const double2*>(y);
            v.x += o.x;
            v.y += o.y;
        }
        *reinterpret_cast<double2*>(y) = v;
    } else {
        if (act0) y[0] = a.accumulate ? y[0] + d0 : d0;
        if (act1) y[1] = a.accumulate ? y[1] + d1 : d1;
    }
}

__global__ void __launch_bounds__(kThreads) k_prolong(ProlongArgs a) {
    if (a.done && ld_flag(a.done)) return;
    const int lane = threadIdx.x & 31;
    const int nbt = a.Bp >> 3, nk = a.npad >> 2;
    const int64_t gw = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
    const int64_t tw = (int64_t)gridDim.x * (kThreads / 32);   // multiple of nbt (nbt | 8)
    const int bt = (int)(gw % nbt);
    const int64_t ts = tw / nbt;
    const int64_t ntile = (a.N + 7) >> 3;
    double ef[16];
    const double* ecol = a.E + (lane & 3) * a.Bp + bt * 8 + (lane >> 2);
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) ef[kk] = kk < nk ? __ldg(ecol + (int64_t)kk * 4 * a.Bp) : 0.0;
    const int b = bt * 8 + 2 * (lane & 3);
    const bool act0 = a.active[b] != 0, act1 = a.active[b + 1] != 0;
    for (int64_t nt = gw / nbt; nt < ntile; nt += 2 * ts) {
        const int64_t nt2 = nt + ts;
        const bool two = nt2 < ntile;
        const int64_t iA = nt * 8 + (lane >> 2), iB = (two ? nt2 : nt) * 8 + (lane >> 2);
        const double* wA = a.W + iA * a.ldw + (lane & 3);
        const double* wB = a.W + iB * a.ldw + (lane & 3);
        bool ldA = true, ldB = true;
        if (a.skip_color >= 0) {            // red-black colour of the fragment's node rows
            auto col = [&](int64_t i) {
                const uint32_t t = fdiv((uint32_t)i, a.fm);
                const int I = (int)((uint32_t)i - t * (uint32_t)a.m) + 1;
                int par;
                if (a.dim == 2) {
                    par = (I + (int)t + 1) & 1;
                } else {
                    const uint32_t u = fdiv(t, a.fm);
                    par = (I + (int)(t - u * (uint32_t)a.m) + 1 + (int)u + 1 + a.kofs) & 1;
                }
                return par;
            };
            ldA = iA >= a.N || col(iA) != a.skip_color;
            ldB = iB >= a.N || col(iB) != a.skip_color;
        }
        double xa[16], xb[16];
#pragma unroll
        for (int kk = 0; kk < 16; ++kk)
            if (kk < nk) {
                xa[kk] = ldA ? __ldg(wA + kk * 4) : 0.0;
                xb[kk] = ldB ? __ldg(wB + kk * 4) : 0.0;
            }
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < 16; ++kk)
            if (kk < nk) {
                dmma_8x8x4(a0, a1, xa[kk], ef[kk]);
                dmma_8x8x4(b0, b1, xb[kk], ef[kk]);
            }
        if (ldA) prolong_store(a, iA, b, a0, a1, act0, act1);
        if (two && ldB) prolong_store(a, iB, b, b0, b1, act0, act1);
    }
}

// ---------------------------------------------------------------------------
// Red-black Gauss-Seidel half-sweep of `color` (AMB-5; eq8)
// on A y = rhs, in place.  color < 0: no update.  LAST: also y^T rhs and
// y^T y per query; the last CTA then does RBCG Step 10:
// rho' = y^T r, PRECOND check (AMB-11), beta = rho'/rho (init: rho_0, beta 0).
// Flat thread-per-element mapping (e = i*Bp + b), Bp a power of two.
// ---------------------------------------------------------------------------
struct GSArgs {
    Geo g;
    int Bp, lgB;
    int64_t NB;               // N*Bp
    const double* theta;      // [Q][Bp]
    const int* active;
    double* Y;
    const double* Rhs;        // or nullptr -> rconst
    double rconst;
    int color;
    int init;                 // LAST: 1 = rho_0 (RBCG Step 2-3)
    SolveState s;             // LAST: partials + bookkeeping
    const int* done;
    int col0;                 // LAST: first partial column (mesh slabs)
    int ext;                  // LAST: 1 = partials only, Step 10 by k_slab_beta
    const double* Yin;        // k_jac: sweep input (Y is its output)
    double omega;             // k_jac: damping
};

constexpr int kGsUnroll = 4;

// f(mu_b) = sum_r phi_r(mu_b) f_r (affine right-hand side, eq12 with R
// terms; NEXT(4)): out[b][i] = sum_r phi[b][r] terms[r][i], r ascending
__global__ void k_affine_rhs(const double* phi, int R, const double* terms, int64_t N, int B, double* out) {
    const int64_t tot = (int64_t)B * N;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(e / N);
        const int64_t i = e - (int64_t)b * N;
        double v = 0.0;
        for (int r = 0; r < R; ++r) v = fma(phi[b * R + r], terms[(int64_t)r * N + i], v);
        out[e] = v;
    }
}

// affine right-hand side of a batch in the internal layout (rbs_set_rhs_terms):
// v[i][b] = sum_r phi[b][r] T[i][r] (r ascending) for i < N, b < B; 0 in the padding.
// T: the packed terms [N8][ldt] (node-major, one read per solve)
__global__ void k_fill_terms(double* __restrict__ v, int64_t N, int64_t N8, int Bp, int B,
                             const double* __restrict__ T, int ldt, int R, const double* __restrict__ phi) {
    const int64_t tot = N8 * Bp;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / Bp;
        const int b = (int)(t - i * Bp);
        double x = 0.0;
        if (i < N && b < B) {
            const double* Ti = T + i * ldt;
            for (int r = 0; r < R; ++r) x = fma(phi[b * R + r], __ldg(Ti + r), x);
        }
        v[t] = x;
    }
}

// terms f_r (R borrowed device vectors of length N) -> packed node-major T[N8][ldt]
struct TermPtrs {
    const double* p[64];
};
__global__ void k_pack_terms(TermPtrs f, int R, int64_t N, int64_t N8, int ldt, double* __restrict__ T) {
    const int64_t tot = N8 * ldt;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / ldt;
        const int r = (int)(t - i * ldt);
        T[t] = (i < N && r < R) ? f.p[r][i] : 0.0;
    }
}

// columns j0 .. j0+7 of a node-major [N8][ld] matrix -> [N8][8] (zero beyond ncol)
__global__ void k_take8(const double* __restrict__ A, int ld, int j0, int ncol, int64_t N8,
                        double* __restrict__ Z) {
    const int64_t tot = N8 * 8;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t >> 3;
        const int k = (int)(t & 7);
        Z[t] = j0 + k < ncol ? A[i * ld + j0 + k] : 0.0;
    }
}

// Cell-label operator (rbs_set_operator_labels) as face coefficients: a face's
// coefficient for term q is the fraction of the 2^(dim-1) cells sharing it that carry
// label q, so kappa_e = sum_q theta_q F_q[e] is the cell average of theta_label(cell)
// (DESIGN.md AMB-1, AMB-24).  labels: (m+1)^dim cells, x fastest; F: [Q][dim][nf].
__global__ void k_labels_to_faces(const uint8_t* __restrict__ lab, int dim, int m, int Q,
                                  double* __restrict__ F) {
    const int64_t M = m, M1 = m + 1;
    const int64_t nf = M1 * (dim == 3 ? M * M : M);
    const int64_t tot = (int64_t)dim * nf;
    const double w = dim == 3 ? 0.25 : 0.5;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int d = (int)(t / nf);
        const int64_t idx = t - d * nf;
        // decode the face (layout in include/rbs.h): the cell index along d is a (0..m);
        // the two transverse node coordinates u, v (1..m) give cells u-1, u (and v-1, v)
        int64_t a, u, v = 1;
        if (d == 0) {             // idx = a + (m+1)((J-1) + m(K-1))
            a = idx % M1;
            const int64_t r = idx / M1;
            u = r % M + 1;        // J
            v = r / M + 1;        // K
        } else if (d == 1) {      // idx = (I-1) + m(a + (m+1)(K-1))
            u = idx % M + 1;      // I
            const int64_t r = idx / M;
            a = r % M1;
            v = r / M1 + 1;       // K
        } else {                  // idx = (I-1) + m((J-1) + m a)
            u = idx % M + 1;      // I
            const int64_t r = idx / M;
            v = r % M + 1;        // J
            a = r / M;
        }
        for (int q = 0; q < Q; ++q) F[((int64_t)q * dim + d) * nf + idx] = 0.0;
        const int nv = dim == 3 ? 2 : 1;
        for (int du = 0; du < 2; ++du)
            for (int dv = 0; dv < nv; ++dv) {
                int64_t c[3];
                const int64_t cu = u - 1 + du, cv = dim == 3 ? v - 1 + dv : 0;
                if (d == 0) { c[0] = a; c[1] = cu; c[2] = cv; }
                else if (d == 1) { c[0] = cu; c[1] = a; c[2] = cv; }
                else { c[0] = cu; c[1] = cv; c[2] = a; }
                const int q = lab[c[0] + M1 * (c[1] + M1 * c[2])];
                if (q < Q) F[((int64_t)q * dim + d) * nf + idx] += w;
            }
    }
}

// LAST pass of the smoother: y^T r, y^T y partials of this CTA and RBCG Step 10
// (beta = y_{k+1}^T r_{k+1} / y_k^T r_k) in the last CTA (AMB-11)
__device__ __forceinline__ void gs_step10(const GSArgs& a, double yr, double yy) {
    __shared__ double s_a[kFlat], s_b[kFlat];
    __shared__ double s_yr[kMaxBatch], s_yy[kMaxBatch];
    __shared__ int s_last;
    const SolveState& s = a.s;
    s_a[threadIdx.x] = yr;
    s_b[threadIdx.x] = yy;
    __syncthreads();
    if (threadIdx.x < a.Bp) {
        double sr = 0.0, sy = 0.0;
        for (int t = threadIdx.x; t < kFlat; t += a.Bp) {
            sr += s_a[t];
            sy += s_b[t];
        }
        s.partF[((int64_t)threadIdx.x * 2 + 0) * s.nctf + a.col0 + blockIdx.x] = sr;
        s.partF[((int64_t)threadIdx.x * 2 + 1) * s.nctf + a.col0 + blockIdx.x] = sy;
    }
    if (!a.ext && cta_is_last(s.ticket, &s_last)) {
        cta_sum_slot(s, 0, s_a, s_yr);
        cta_sum_slot(s, 1, s_a, s_yy);
        if (threadIdx.x < s.Bp) {
            const int bb = threadIdx.x;
            if (s.active[bb]) {
                const double r1 = s_yr[bb], y2 = s_yy[bb];
                if (!(r1 > s.delta * sqrt(y2) * sqrt(s.rr[bb]))) {
                    s.status[bb] = isfinite(r1) ? Q_PRECOND : Q_NONFINITE;
                    s.active[bb] = 0;
                    s.beta[bb] = 0.0;
                } else {
                    s.beta[bb] = a.init ? 0.0 : r1 / s.rho[bb];
                    s.rho[bb] = r1;
                }
            }
        }
        __threadfence();
        const int any = cta_any_active(s);
        if (threadIdx.x == 0) {
            *(volatile int*)s.done = any ? 0 : 1;
            if (!a.init) *(volatile int*)s.kcount = *(volatile int*)s.kcount + 1;
        }
        release_ticket(s.ticket);
    }
}

template <int DIM, bool LAST>
__global__ void __launch_bounds__(kFlat, 2) k_gs(GSArgs a) {
    if (a.done && ld_flag(a.done)) return;
    extern __shared__ double smem[];
    double* s_th = smem;
    int* s_act = (int*)(s_th + a.g.Q * a.Bp);
    for (int t = threadIdx.x; t < a.g.Q * a.Bp; t += kFlat) s_th[t] = a.theta[t];
    for (int t = threadIdx.x; t < a.Bp; t += kFlat) s_act[t] = a.active[t];
    __syncthreads();
    double yr = 0.0, yy = 0.0;
    const int64_t stride = (int64_t)gridDim.x * kFlat;
    const int b = threadIdx.x & (a.Bp - 1);
    if (s_act[b]) {
        for (int64_t e0 = blockIdx.x * (int64_t)kFlat + threadIdx.x; e0 < a.NB;
             e0 += kGsUnroll * stride) {
            double nb[kGsUnroll][2 * DIM], rhs[kGsUnroll], yo[kGsUnroll];
            int I[kGsUnroll], J[kGsUnroll], K[kGsUnroll];
            bool upd[kGsUnroll], ok[kGsUnroll];
#pragma unroll
            for (int u = 0; u < kGsUnroll; ++u) {
                const int64_t e = e0 + u * stride;
                ok[u] = e < a.NB;
                upd[u] = false;
                rhs[u] = a.rconst;
                yo[u] = 0.0;
                if (ok[u]) {
                    const int64_t i = e >> a.lgB;
                    node_coords(a.g, (uint32_t)i, I[u], J[u], K[u]);
                    upd[u] = ((I[u] + J[u] + (DIM == 3 ? K[u] : 0)) & 1) == a.color;
                    if (a.Rhs && (upd[u] || LAST)) rhs[u] = __ldg(a.Rhs + e);
                    if (upd[u]) node_nbrs<DIM>(a.g, a.Y, a.Bp, i, b, I[u], J[u], K[u], nb[u]);
                    else if (LAST) yo[u] = a.Y[e];
                }
            }
#pragma unroll
            for (int u = 0; u < kGsUnroll; ++u) {
                if (upd[u]) {
                    double k[2 * DIM];
                    node_kappa<DIM>(a.g, s_th, a.Bp, b, I[u], J[u], K[u], k);
                    yo[u] = gs_value<DIM>(a.g, k, rhs[u], nb[u]);
                    a.Y[e0 + u * stride] = yo[u];
                }
                if (LAST && ok[u] && (DIM == 2 || owned(a.g, K[u]))) {
                    yr = fma(yo[u], rhs[u], yr);
                    yy = fma(yo[u], yo[u], yy);
                }
            }
        }
    }
    if (LAST) gs_step10(a, yr, yy);
}

// ---------------------------------------------------------------------------
// Red-black half-sweep for 3D grids, row-pencil form: each group of Bp lanes (one
// query per lane) walks a (J, K) row of nodes in x, keeping the x-neighbours in
// registers (one new load per node) and updating the nodes of the sweep's colour
// with the same arithmetic as k_gs (node_kappa, gs_value; eq8,
// AMB-5/6).  Nodes inside one block take the block's theta without the cell-average
// (bitwise the same, see node_kappa).  LAST: y^T r, y^T y over every owned node.
// Requires Bp <= 32.
// ---------------------------------------------------------------------------


template <bool LAST, int kGsSeg, bool FACES>
__global__ void __launch_bounds__(kFlat, kGsSeg <= 2 ? 2 : 1) k_gs3r(GSArgs a) {
    if (a.done && ld_flag(a.done)) return;
    extern __shared__ double smem[];
    double* s_th = smem;
    int* s_act = (int*)(s_th + a.g.Q * a.Bp);
    for (int t = threadIdx.x; t < a.g.Q * a.Bp; t += kFlat) s_th[t] = a.theta[t];
    for (int t = threadIdx.x; t < a.Bp; t += kFlat) s_act[t] = a.active[t];
    __syncthreads();
    const Geo& g = a.g;
    const int Bp = a.Bp, m = g.m;
    const int lane = threadIdx.x & 31, rpw = 32 >> a.lgB;
    const int sub = lane >> a.lgB, b = lane & (Bp - 1);
    const int nseg = (m + kGsSeg - 1) / kGsSeg;
    const int64_t items = (int64_t)m * g.mz * nseg;
    const int64_t nw = ((int64_t)gridDim.x * kFlat) >> 5;
    const int64_t w0 = (blockIdx.x * (int64_t)kFlat + threadIdx.x) >> 5;
    const int64_t sy = (int64_t)m * Bp, sz = sy * m;
    double yr = 0.0, yy = 0.0;
    if (s_act[b]) {
        for (int64_t it = w0 * rpw + sub; it < items; it += nw * rpw) {
            const int64_t row = it / nseg;
            const int x0 = 1 + (int)(it - row * nseg) * kGsSeg;
            const int J = (int)(row % m) + 1, Kl = (int)(row / m), K = Kl + 1 + g.kofs;
            double* Yr = a.Y + ((int64_t)Kl * m * m + (int64_t)(J - 1) * m) * Bp + b;   // node x at Yr[(x-1)Bp]
            const double* Rr = a.Rhs ? a.Rhs + ((int64_t)Kl * m * m + (int64_t)(J - 1) * m) * Bp + b : nullptr;
            const bool hym = J > 1, hyp = J < m, hzm = has_zm(g, K), hzp = has_zp(g, K);
            const int px = (a.color - J - K) & 1;          // parity of the active x
            // ---- all loads of the segment first (x-window, y/z neighbours, rhs) ----
            double yv[kGsSeg + 2], q[kGsSeg][4], rh[kGsSeg];
#pragma unroll
            for (int j = 0; j < kGsSeg + 2; ++j) {
                const int x = x0 - 1 + j;
                yv[j] = (x >= 1 && x <= m) ? __ldg(Yr + (int64_t)(x - 1) * Bp) : 0.0;
            }
#pragma unroll
            for (int j = 0; j < kGsSeg; ++j) {
                const int x = x0 + j;
                const int64_t o = (int64_t)(x - 1) * Bp;
                const bool in = x <= m, act = in && ((x ^ px) & 1) == 0;
                q[j][0] = act && hym ? __ldg(Yr + o - sy) : 0.0;
                q[j][1] = act && hyp ? __ldg(Yr + o + sy) : 0.0;
                q[j][2] = act && hzm ? __ldg(Yr + o - sz) : 0.0;
                q[j][3] = act && hzp ? __ldg(Yr + o + sz) : 0.0;
                rh[j] = (Rr && in && (act || LAST)) ? __ldg(Rr + o) : a.rconst;
            }
            // ---- updates of the sweep's colour ----------------------------------------
            const int by0 = axis_block(g, J - 1, g.py) * g.px, by1 = axis_block(g, J, g.py) * g.px;
            const int pxy = g.px * g.py;
            const int bz0 = axis_block(g, K - 1, g.pz) * pxy, bz1 = axis_block(g, K, g.pz) * pxy;
            const bool rowu = !g.faces && by0 == by1 && bz0 == bz1;
            const bool own = owned(g, K);
#pragma unroll
            for (int j = 0; j < kGsSeg; ++j) {
                const int x = x0 + j;
                if (x > m) break;
                if (((x ^ px) & 1) == 0) {
                    double nb[6] = {yv[j], yv[j + 2], q[j][0], q[j][1], q[j][2], q[j][3]}, k[6];
                    const int bxl = axis_block(g, x - 1, g.px), bxr = axis_block(g, x, g.px);
                    if (FACES) {            // face operator: inline face loads (AMB-23)
                        node_kappa_faces<3>(g, s_th, Bp, b, x, J, K, k);
                    } else if (rowu && bxl == bxr) {
                        const double c = s_th[(bxr + by0 + bz0) * Bp + b];
#pragma unroll
                        for (int e = 0; e < 6; ++e) k[e] = c;
                    } else {
                        node_kappa3_call(g, s_th, Bp, b, x, J, K, k);
                    }
                    const double v = gs_value<3>(g, k, rh[j], nb);
                    Yr[(int64_t)(x - 1) * Bp] = v;
                    if (LAST && own) {
                        yr = fma(v, rh[j], yr);
                        yy = fma(v, v, yy);
                    }
                } else if (LAST && own) {
                    yr = fma(yv[j + 1], rh[j], yr);
                    yy = fma(yv[j + 1], yv[j + 1], yy);
                }
            }
        }
    }
    if (LAST) gs_step10(a, yr, yy);
}

// ---------------------------------------------------------------------------
// Damped Jacobi sweep ("the smoother (Jacobi or Gauss-Seidel)"):
//   y_out = y_in + omega (g - y_in), g = the Gauss-Seidel point value of y_in,
// i.e. y_in + omega D^-1 (b - A y_in).  Ping-pong buffers; frozen lanes copy.
// ---------------------------------------------------------------------------
template <int DIM, bool LAST>
__global__ void __launch_bounds__(kFlat, 2) k_jac(GSArgs a) {
    if (a.done && ld_flag(a.done)) return;
    extern __shared__ double smem[];
    double* s_th = smem;
    int* s_act = (int*)(s_th + a.g.Q * a.Bp);
    for (int t = threadIdx.x; t < a.g.Q * a.Bp; t += kFlat) s_th[t] = a.theta[t];
    for (int t = threadIdx.x; t < a.Bp; t += kFlat) s_act[t] = a.active[t];
    __syncthreads();
    double yr = 0.0, yy = 0.0;
    const int64_t stride = (int64_t)gridDim.x * kFlat;
    const int b = threadIdx.x & (a.Bp - 1);
    const bool act = s_act[b] != 0;
    for (int64_t e0 = blockIdx.x * (int64_t)kFlat + threadIdx.x; e0 < a.NB; e0 += kGsUnroll * stride) {
        double nb[kGsUnroll][2 * DIM], rhs[kGsUnroll], yi[kGsUnroll];
        int I[kGsUnroll], J[kGsUnroll], K[kGsUnroll];
        bool ok[kGsUnroll];
#pragma unroll
        for (int u = 0; u < kGsUnroll; ++u) {
            const int64_t e = e0 + u * stride;
            ok[u] = e < a.NB;
            rhs[u] = a.rconst;
            yi[u] = 0.0;
            if (ok[u]) {
                const int64_t i = e >> a.lgB;
                node_coords(a.g, (uint32_t)i, I[u], J[u], K[u]);
                yi[u] = a.Yin[e];
                if (act) {
                    if (a.Rhs) rhs[u] = __ldg(a.Rhs + e);
                    node_nbrs<DIM>(a.g, a.Yin, a.Bp, i, b, I[u], J[u], K[u], nb[u]);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kGsUnroll; ++u) {
            if (!ok[u]) continue;
            double yo = yi[u];
            if (act) {
                double k[2 * DIM];
                node_kappa<DIM>(a.g, s_th, a.Bp, b, I[u], J[u], K[u], k);
                const double gv = gs_value<DIM>(a.g, k, rhs[u], nb[u]);
                yo = yi[u] + a.omega * (gv - yi[u]);
                if (LAST && (DIM == 2 || owned(a.g, K[u]))) {
                    yr = fma(yo, rhs[u], yr);
                    yy = fma(yo, yo, yy);
                }
            }
            a.Y[e0 + u * stride] = yo;
        }
    }
    if (LAST) gs_step10(a, yr, yy);
}

// ---------------------------------------------------------------------------
// RBCG Step 11 + Step 5:
//   p_new = y + beta p_old (recomputed on the halo), q = A p_new,
//   sigma partial = p_new^T q; the last CTA computes alpha = rho / sigma with
//   the MAXIT / CURVATURE checks.  p is double-buffered.
// ---------------------------------------------------------------------------
struct CGPArgs {
    Geo g;
    int Bp, lgB;
    int64_t NB;
    const double* theta;
    const int* active;
    const double* beta;
    const double* Y;
    const double* Pold;
    double* Pnew;
    SolveState s;
    const int* done;
    int col0;                 // first partial column (mesh slabs)
    int ext;                  // 1 = partials only, Step 5 by k_slab_alpha
};

constexpr int kCgpUnroll = 2;

// sigma partials of this CTA and RBCG Step 5 (alpha = rho / p^T A p) with
// the MAXIT / CURVATURE checks in the last CTA (AMB-11)
__device__ __forceinline__ void cgp_step5(const CGPArgs& a, double sig) {
    __shared__ double s_a[kFlat];
    __shared__ double s_sig[kMaxBatch];
    __shared__ int s_last;
    const SolveState& s = a.s;
    s_a[threadIdx.x] = sig;
    __syncthreads();
    if (threadIdx.x < a.Bp) {
        double t0 = 0.0;
        for (int t = threadIdx.x; t < kFlat; t += a.Bp) t0 += s_a[t];
        s.partF[((int64_t)threadIdx.x * 2 + 0) * s.nctf + a.col0 + blockIdx.x] = t0;
    }
    if (!a.ext && cta_is_last(s.ticket, &s_last)) {
        cta_sum_slot(s, 0, s_a, s_sig);
        const int k = ld_flag(s.kcount);
        if (threadIdx.x < s.Bp) {
            const int bb = threadIdx.x;
            double al = 0.0;
            if (s.active[bb]) {
                const double sg = s_sig[bb];
                if (k >= s.maxit) { s.status[bb] = Q_MAXIT; s.its[bb] = k; s.active[bb] = 0; }
                else if (!(sg > 0.0)) {
                    s.status[bb] = isfinite(sg) ? Q_CURVATURE : Q_NONFINITE;
                    s.its[bb] = k;
                    s.active[bb] = 0;
                } else al = s.rho[bb] / sg;
            }
            s.alpha[bb] = al;
        }
        __threadfence();
        update_done(s);
        release_ticket(s.ticket);
    }
}

template <int DIM>
__global__ void __launch_bounds__(kFlat, 2) k_cgp(CGPArgs a) {
    if (a.done && ld_flag(a.done)) return;
    extern __shared__ double smem[];
    double* s_th = smem;
    int* s_act = (int*)(s_th + a.g.Q * a.Bp);
    for (int t = threadIdx.x; t < a.g.Q * a.Bp; t += kFlat) s_th[t] = a.theta[t];
    for (int t = threadIdx.x; t < a.Bp; t += kFlat) s_act[t] = a.active[t];
    __syncthreads();
    double sig = 0.0;
    const int64_t stride = (int64_t)gridDim.x * kFlat;
    const int b = threadIdx.x & (a.Bp - 1);
    if (s_act[b]) {
        const double bet = a.beta[b];
        const int64_t sy = (int64_t)a.g.m * a.Bp, sz = sy * a.g.m;
        for (int64_t e0 = blockIdx.x * (int64_t)kFlat + threadIdx.x; e0 < a.NB;
             e0 += kCgpUnroll * stride) {
            double yv[kCgpUnroll][2 * DIM + 1], pv[kCgpUnroll][2 * DIM + 1];
            int I[kCgpUnroll], J[kCgpUnroll], K[kCgpUnroll];
            bool ok[kCgpUnroll];
#pragma unroll
            for (int u = 0; u < kCgpUnroll; ++u) {
                const int64_t e = e0 + u * stride;
                ok[u] = e < a.NB;
                if (ok[u]) {
                    const int64_t i = e >> a.lgB;
                    node_coords(a.g, (uint32_t)i, I[u], J[u], K[u]);
                    const int64_t off[6] = {-a.Bp, a.Bp, -sy, sy, -sz, sz};
                    const bool in[6] = {I[u] > 1, I[u] < a.g.m, J[u] > 1, J[u] < a.g.m,
                                        has_zm(a.g, K[u]), has_zp(a.g, K[u])};
                    yv[u][0] = __ldg(a.Y + e);
                    pv[u][0] = __ldg(a.Pold + e);
#pragma unroll
                    for (int d = 0; d < 2 * DIM; ++d) {
                        yv[u][d + 1] = in[d] ? __ldg(a.Y + e + off[d]) : 0.0;
                        pv[u][d + 1] = in[d] ? __ldg(a.Pold + e + off[d]) : 0.0;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kCgpUnroll; ++u)
                if (ok[u]) {
                    double k[2 * DIM], nb[2 * DIM];
                    node_kappa<DIM>(a.g, s_th, a.Bp, b, I[u], J[u], K[u], k);
                    const double pp = fma(bet, pv[u][0], yv[u][0]);
#pragma unroll
                    for (int d = 0; d < 2 * DIM; ++d) nb[d] = fma(bet, pv[u][d + 1], yv[u][d + 1]);
                    const double q = stencil_apply<DIM>(a.g, k, pp, nb);
                    a.Pnew[e0 + u * stride] = pp;
                    if (DIM == 2 || owned(a.g, K[u])) sig = fma(pp, q, sig);
                }
        }
    }
    cgp_step5(a, sig);
}

// ---------------------------------------------------------------------------
// RBCG Step 11 + Step 5 for 3D grids in two passes (instead of recomputing p_new on
// the six neighbours of every node): k_pnew3 streams p_new = y + beta p_old
// for every node; k_sigma3r forms sigma = p_new^T A p_new (Step 5,
// PAPER.md:269) in k_gs3r's row segments (x window + y/z neighbours loaded together)
// and computes alpha in the last CTA.  Per node the same arithmetic as k_cgp<3>.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_pnew3(const double* __restrict__ Y, const double* __restrict__ Pold,
                                               double* __restrict__ Pnew, const double* __restrict__ beta,
                                               const int* __restrict__ active, int64_t NB2, int Bp,
                                               const int* done) {
    if (done && ld_flag(done)) return;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < NB2; e += stride) {
        const int b = (int)((2 * e) & (Bp - 1));          // lanes b, b+1 of one node
        const double2 y = __ldg(reinterpret_cast<const double2*>(Y) + e);
        const double2 p = __ldg(reinterpret_cast<const double2*>(Pold) + e);
        const bool a0 = active[b] != 0, a1 = active[b + 1] != 0;
        if (!a0 && !a1) continue;
        double2 o = reinterpret_cast<double2*>(Pnew)[e];
        if (a0) o.x = fma(beta[b], p.x, y.x);
        if (a1) o.y = fma(beta[b + 1], p.y, y.y);
        reinterpret_cast<double2*>(Pnew)[e] = o;
    }
}

template <int SEG, bool FACES>
__global__ void __launch_bounds__(kFlat, 1) k_sigma3r(CGPArgs a) {
    if (a.done && ld_flag(a.done)) return;
    extern __shared__ double smem[];
    double* s_th = smem;
    int* s_act = (int*)(s_th + a.g.Q * a.Bp);
    for (int t = threadIdx.x; t < a.g.Q * a.Bp; t += kFlat) s_th[t] = a.theta[t];
    for (int t = threadIdx.x; t < a.Bp; t += kFlat) s_act[t] = a.active[t];
    __syncthreads();
    const Geo& g = a.g;
    const int Bp = a.Bp, m = g.m;
    const int lane = threadIdx.x & 31, rpw = 32 >> a.lgB;
    const int sub = lane >> a.lgB, b = lane & (Bp - 1);
    const int nseg = (m + SEG - 1) / SEG;
    const int64_t items = (int64_t)m * g.mz * nseg;
    const int64_t nw = ((int64_t)gridDim.x * kFlat) >> 5;
    const int64_t w0 = (blockIdx.x * (int64_t)kFlat + threadIdx.x) >> 5;
    const int64_t sy = (int64_t)m * Bp, sz = sy * m;
    const double* P = a.Pnew;
    double sig = 0.0;
    if (s_act[b]) {
        for (int64_t it = w0 * rpw + sub; it < items; it += nw * rpw) {
            const int64_t row = it / nseg;
            const int x0 = 1 + (int)(it - row * nseg) * SEG;
            const int J = (int)(row % m) + 1, Kl = (int)(row / m), K = Kl + 1 + g.kofs;
            const double* Pr = P + ((int64_t)Kl * m * m + (int64_t)(J - 1) * m) * Bp + b;
            const bool hym = J > 1, hyp = J < m, hzm = has_zm(g, K), hzp = has_zp(g, K);
            double pw[SEG + 2], q[SEG][4];
#pragma unroll
            for (int j = 0; j < SEG + 2; ++j) {
                const int x = x0 - 1 + j;
                pw[j] = (x >= 1 && x <= m) ? __ldg(Pr + (int64_t)(x - 1) * Bp) : 0.0;
            }
#pragma unroll
            for (int j = 0; j < SEG; ++j) {
                const int x = x0 + j;
                const int64_t o = (int64_t)(x - 1) * Bp;
                const bool in = x <= m;
                q[j][0] = in && hym ? __ldg(Pr + o - sy) : 0.0;
                q[j][1] = in && hyp ? __ldg(Pr + o + sy) : 0.0;
                q[j][2] = in && hzm ? __ldg(Pr + o - sz) : 0.0;
                q[j][3] = in && hzp ? __ldg(Pr + o + sz) : 0.0;
            }
            const int by0 = axis_block(g, J - 1, g.py) * g.px, by1 = axis_block(g, J, g.py) * g.px;
            const int pxy = g.px * g.py;
            const int bz0 = axis_block(g, K - 1, g.pz) * pxy, bz1 = axis_block(g, K, g.pz) * pxy;
            const bool rowu = !g.faces && by0 == by1 && bz0 == bz1;
            const bool own = owned(g, K);
#pragma unroll
            for (int j = 0; j < SEG; ++j) {
                const int x = x0 + j;
                if (x > m) break;
                double k[6];
                const int bxl = axis_block(g, x - 1, g.px), bxr = axis_block(g, x, g.px);
                if (FACES) {
                    node_kappa_faces<3>(g, s_th, Bp, b, x, J, K, k);
                } else if (rowu && bxl == bxr) {
                    const double c = s_th[(bxr + by0 + bz0) * Bp + b];
#pragma unroll
                    for (int e = 0; e < 6; ++e) k[e] = c;
                } else {
                    node_kappa3_call(g, s_th, Bp, b, x, J, K, k);
                }
                const double nb[6] = {pw[j], pw[j + 2], q[j][0], q[j][1], q[j][2], q[j][3]};
                const double qv = stencil_apply<3>(g, k, pw[j + 1], nb);
                if (own) sig = fma(pw[j + 1], qv, sig);
            }
        }
    }
    cgp_step5(a, sig);
}

// ---------------------------------------------------------------------------
// Stage 2 of W^T r / ||r||^2 + stop test + reduced solve (RBCG Steps 7-9,
// RBI Steps 2-5).  One CTA per query.  All partial loads are issued at once
// (each thread sums a fixed chunk of one row, then the chunks are combined in
// a fixed order); the reduced solve e = A_n(mu)^{-1} r_n is a matvec with the
// inverse formed once per query at setup.
// ---------------------------------------------------------------------------
constexpr int kRsThreads = 512;
constexpr int kRsChunks = 32;     // chunks per row (one warp lane each in the second stage)
constexpr int kRsPer = 12;        // columns of a chunk loaded together

// solve_only = 1: e = A_n^{-1} r_n only -- no stop test, no state change (the coarse
// correction inside the symmetric two-level preconditioner, RBS_PRECOND_SYM); 2: the
// same, and e is also reported as a_n (the first application)
__global__ void __launch_bounds__(kRsThreads) k_reduce_solve(SolveState s, int solve_only = 0) {
    __shared__ double s_rn[kMaxN + 1];
    __shared__ double s_chunk[(kMaxN + 1) * kRsChunks];
    __shared__ double s_e[kMaxN * 8];
    __shared__ double s_prev;
    __shared__ int s_go, s_last, s_na;
    const int b = blockIdx.x, tid = threadIdx.x;
    const int rows = s.npad + 1, nr = s.n + 1;     // rows 0..n-1 and the rr row (npad)
    // A_n^{-1} row slice of this thread for the fixed-order matvec below (constant during
    // the solve: loaded before the dependency wait, so it overlaps the previous pass)
    const int mi = tid >> 3, ml = tid & 7;
    double ai[kMaxN / 8];
    {
        const bool mv = !s.tri && mi < s.n && b < s.B;
        const double* Ai = s.Ainv + (int64_t)b * s.npad * s.npad + mi * s.npad;
#pragma unroll
        for (int k = 0; k < kMaxN / 8; ++k) ai[k] = (mv && ml + 8 * k < s.n) ? __ldcg(Ai + ml + 8 * k) : 0.0;
    }
    pdl_wait();                       // the partials and the flags come from the previous pass
    if (ld_flag(s.done)) return;
    pdl_trigger();                    // the next pass may start its prologue on the idle SMs
    const bool act = s.active[b] != 0;
    if (act) {
        // two-stage fixed-order sums: 32 chunks of <= 10 columns per row (all loads of a
        // chunk in flight at once), then one warp per row combines its 32 chunks
        const int per = (s.nct + kRsChunks - 1) / kRsChunks;
        for (int t = tid; t < nr * kRsChunks; t += kRsThreads) {
            const int r = t / kRsChunks, c = t - r * kRsChunks;
            const int j = r < s.n ? r : s.npad;
            const double* p = s.partP + ((int64_t)b * rows + j) * s.nct;
            const int c0 = c * per, c1 = min(s.nct, c0 + per);
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            for (int k0 = c0; k0 < c1; k0 += kRsPer) {
                double v[kRsPer];
#pragma unroll
                for (int u = 0; u < kRsPer; ++u) v[u] = k0 + u < c1 ? __ldcg(p + k0 + u) : 0.0;
#pragma unroll
                for (int u = 0; u < kRsPer; u += 4) {
                    a0 += v[u];
                    a1 += v[u + 1];
                    a2 += v[u + 2];
                    a3 += v[u + 3];
                }
            }
            s_chunk[r * kRsChunks + c] = (a0 + a1) + (a2 + a3);
        }
        __syncthreads();
        for (int r = tid >> 5; r < nr; r += kRsThreads / 32) {
            double v = s_chunk[r * kRsChunks + (tid & 31)];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if ((tid & 31) == 0) s_rn[r < s.n ? r : s.npad] = v;
        }
        __syncthreads();
        if (tid == 0 && solve_only) s_go = 1;
        if (tid == 0 && !solve_only) {
            const double rr2 = s_rn[s.npad];
            const double h = sqrt(rr2) / s.fnorm[b];
            const int it = ld_flag(s.kcount) + 1;
            if (s.hist) s.hist[(int64_t)b * (s.maxit + 1) + it] = h;
            s.its[b] = it;
            s.relres[b] = h;
            s_prev = s.rr[b];                 // ||r_k||^2 (adaptive-n rule)
            s.rr[b] = rr2;
            int go = 1;
            if (!isfinite(h)) { s.status[b] = Q_NONFINITE; go = 0; }
            else if (h < s.tol) { s.status[b] = Q_CONVERGED; go = 0; }
            else if (s.method == 0 && it >= s.maxit) { s.status[b] = Q_MAXIT; go = 0; }
            if (!go) s.active[b] = 0;
            s_go = go;
        }
        __syncthreads();
        if (s.tri) {
            // active dimension (adaptive-n rule after the x-update), then
            // e = A_{na}^{-1} r_n[0..na) with the leading block of L (AMB-19), zero beyond
            if (tid == 0) {
                int na = s.na[b];
                const double prev = s_prev;
                if (!solve_only && s_go && s.gamma > 0.0 && s.method == 1 && na < s.n &&
                    prev < s.gamma * s.gamma * s_rn[s.npad])
                    ++na;
                s.na[b] = na;
                s_na = na;
            }
            __syncthreads();
            if (tid < 32) {
                const int na = s_na;
                const double* Lb = s.L + (int64_t)b * s.npad * s.npad;
                double z0 = (s_go && tid < na) ? s_rn[tid] : 0.0;
                double z1 = (s_go && tid + 32 < na) ? s_rn[tid + 32] : 0.0;
                if (s_go) warp_chol_solve(Lb, s.npad, na, &z0, &z1, tid);
                if (tid < s.n) s.E[tid * s.Bp + b] = tid < na ? z0 : 0.0;
                if (tid + 32 < s.n) s.E[(tid + 32) * s.Bp + b] = tid + 32 < na ? z1 : 0.0;
                if (solve_only == 2) {                     // first coarse correction
                    if (tid < s.n) s.a_n[(int64_t)b * s.npad + tid] = tid < na ? z0 : 0.0;
                    if (tid + 32 < s.n) s.a_n[(int64_t)b * s.npad + tid + 32] = tid + 32 < na ? z1 : 0.0;
                }
            }
        } else {
        // e = A_n^{-1} r_n: row i by 8 threads (fixed order), frozen lanes get e = 0
        if (mi < s.n) {
            double v = 0.0;
            if (s_go) {
#pragma unroll
                for (int k = 0; k < kMaxN / 8; ++k)
                    if (ml + 8 * k < s.n) v = fma(ai[k], s_rn[ml + 8 * k], v);
            }
            s_e[tid] = v;
        }
        __syncthreads();
        if (tid < s.n) {
            double v = 0.0;
            for (int l = 0; l < 8; ++l) v += s_e[tid * 8 + l];
            s.E[tid * s.Bp + b] = v;
            if (solve_only == 2) s.a_n[(int64_t)b * s.npad + tid] = v;   // first coarse correction
        }
        }
    }
    // RBI: the iteration counter and the done flag in the last CTA.  RBCG skips the ticket
    // (an L2 round trip chain per iteration): the smoother pass that follows recomputes the
    // done flag in its last CTA, so a batch whose last query converged here costs one more
    // (all-lanes-frozen) smoother pass per solve instead
    if (!solve_only && s.method == 0 && cta_is_last(s.ticket, &s_last)) {
        const int any = cta_any_active(s);
        if (threadIdx.x == 0) {
            *(volatile int*)s.done = any ? 0 : 1;
            *(volatile int*)s.kcount = ld_flag(s.kcount) + 1;
        }
        release_ticket(s.ticket);
    }
}

// Polak-Ribiere beta (RBS_BETA_PR, NEXT(3)): per-CTA partials of y^T r_old over a
// contiguous node range (fixed order), part[b][2][nctf] slot 0 ...
__global__ void __launch_bounds__(256) k_dot_pr(const double* __restrict__ Y, const double* __restrict__ Ro,
                                                int64_t N, int Bp, SolveState s) {
    __shared__ double s_p[256];
    if (ld_flag(s.done)) return;
    const int tid = threadIdx.x, b = tid % Bp, gsz = 256 / Bp, k = tid / Bp;
    const int64_t n0 = N * blockIdx.x / gridDim.x, n1 = N * (blockIdx.x + 1) / gridDim.x;
    double acc = 0.0;
    for (int64_t i = n0 + k; i < n1; i += gsz) acc = fma(Y[i * Bp + b], Ro[i * Bp + b], acc);
    s_p[tid] = acc;
    __syncthreads();
    if (tid < Bp) {
        double v = 0.0;
        for (int u = 0; u < gsz; ++u) v += s_p[u * Bp + tid];
        s.partF[((int64_t)tid * 2 + 0) * s.nctf + blockIdx.x] = v;
    }
}

// ... then one CTA: d = y_{k+1}^T r_k (fixed-order sum of the partials) and
// beta = (rho_{k+1} - d) / rho_k (the smoother's Step-10 epilogue already set
// rho = rho_{k+1}; rho_k was saved in rho_prev before it)
__global__ void __launch_bounds__(256) k_beta_pr(SolveState s, const double* __restrict__ rho_prev, int ncta) {
    __shared__ double s_buf[256], s_d[kMaxBatch];
    if (ld_flag(s.done)) return;
    cta_sum_slot(s, 0, s_buf, s_d, ncta);
    if (threadIdx.x < s.Bp && s.active[threadIdx.x]) {
        const int b = threadIdx.x;
        s.beta[b] = (s.rho[b] - s_d[b]) / rho_prev[b];
    }
}

// generic stage 2: out[b][j] = sum_c part[b][j][c], j < rows (one CTA per b)
__global__ void __launch_bounds__(128) k_reduce_rows(const double* part, int rows, int nct,
                                                     double* out) {
    const int b = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = warp; j < rows; j += 4) {
        const double v = warp_sum_row(part + ((int64_t)b * rows + j) * nct, nct, lane);
        if (lane == 0) out[(int64_t)b * rows + j] = v;
    }
}

// ---------------------------------------------------------------------------
// Once per query (eq12b, 69): A_n(theta) = sum_q theta_q
// A_{n,q}; right-looking Cholesky in shared memory; a_n = A_n^{-1} f_n
// (first RB correction, PAPER.md:171 / AMB-12); state init.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_setup_reduced(SolveState s, int rbi) {
    __shared__ double sA[kMaxN * kMaxN];
    __shared__ int s_fail;
    const int b = blockIdx.x, tid = threadIdx.x;
    const int n = s.n, ld = s.npad;
    if (b >= s.B) {
        if (tid == 0) { s.active[b] = 0; s.status[b] = Q_MAXIT; s.its[b] = 0; s.alpha[b] = 0.0;
                        s.beta[b] = 0.0; s.rho[b] = 0.0; s.fnorm[b] = 1.0; s.rr[b] = 0.0; }
        return;
    }
    for (int t = tid; t < n * n; t += blockDim.x) {
        const int i = t / n, j = t - i * n;
        double v = 0.0;
        for (int q = 0; q < s.Q; ++q) v = fma(s.theta[q * s.Bp + b], s.ANq[((int64_t)q * ld + i) * ld + j], v);
        sA[i * ld + j] = v;
    }
    if (tid == 0) s_fail = -1;
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        if (tid == 0) {
            const double d = sA[k * ld + k];
            if (!(d > 0.0)) s_fail = k;
            else sA[k * ld + k] = sqrt(d);
        }
        __syncthreads();
        if (s_fail >= 0) break;
        const double dk = sA[k * ld + k];
        for (int i = k + 1 + tid; i < n; i += blockDim.x) sA[i * ld + k] /= dk;
        __syncthreads();
        const int m = n - k - 1;  // trailing (i,j), k < j <= i < n
        for (int t = tid; t < m * m; t += blockDim.x) {
            const int i = k + 1 + t / m, j = k + 1 + t % m;
            if (j <= i) sA[i * ld + j] -= sA[i * ld + k] * sA[j * ld + k];
        }
        __syncthreads();
    }
    double* L = s.L + (int64_t)b * ld * ld;
    for (int t = tid; t < n * ld; t += blockDim.x) {
        const int i = t / ld, j = t - i * ld;
        L[t] = (j <= i && j < n) ? sA[i * ld + j] : 0.0;
    }
    const double ff = s.fproj[(int64_t)b * (ld + 1) + ld];
    const double fnorm = sqrt(ff);
    if (tid == 0) {
        s.fnorm[b] = fnorm > 0.0 ? fnorm : 1.0;
        s.rr[b] = ff;
        s.alpha[b] = 0.0;
        s.beta[b] = 0.0;
        s.rho[b] = 0.0;
        s.its[b] = 0;
        s.relres[b] = fnorm > 0.0 ? 1.0 : 0.0;
        s.pivot[b] = s_fail;
        if (s.hist) s.hist[(int64_t)b * (s.maxit + 1)] = fnorm > 0.0 ? 1.0 : 0.0;
        int act = 1, st = Q_MAXIT;
        if (s_fail >= 0) { act = 0; st = Q_NOT_SPD; }
        else if (!isfinite(fnorm)) { act = 0; st = Q_NONFINITE; }   // before f = 0 (AMB-11)
        else if (!(fnorm > 0.0)) { act = 0; st = Q_CONVERGED; }
        else if (rbi && 1.0 < s.tol) { act = 0; st = Q_CONVERGED; }
        else if (rbi && s.maxit <= 0) { act = 0; st = Q_MAXIT; }
        s.active[b] = act;
        s.status[b] = st;
    }
    __syncthreads();
    // A_n^{-1} = L^{-T} L^{-1}: thread j solves column j (L z = e_j, L^T x = z)
    if (s_fail < 0 && s.Ainv) {
        double* Ai = s.Ainv + (int64_t)b * ld * ld;
        for (int j = tid; j < ld; j += blockDim.x) {
            if (j >= n) {
                for (int i = 0; i < ld; ++i) Ai[i * ld + j] = 0.0;
                continue;
            }
            for (int i = 0; i < n; ++i) {
                double v = (i == j) ? 1.0 : 0.0;
                for (int k = j; k < i; ++k) v -= sA[i * ld + k] * Ai[k * ld + j];
                Ai[i * ld + j] = i < j ? 0.0 : v / sA[i * ld + i];
            }
            for (int i = n - 1; i >= 0; --i) {
                double v = Ai[i * ld + j];
                for (int k = i + 1; k < n; ++k) v -= sA[k * ld + i] * Ai[k * ld + j];
                Ai[i * ld + j] = v / sA[i * ld + i];
            }
            for (int i = n; i < ld; ++i) Ai[i * ld + j] = 0.0;
        }
    }
    const int na0 = (s.na0 > 0 && s.na0 < n) ? s.na0 : n;   // zero-initialised state: all of W
    if (tid == 0 && s.na) s.na[b] = na0;
    if (s_fail < 0 && n > 0 && tid < 32) {
        // sA holds the factor in its lower triangle (only that part is read); the first
        // correction uses the active dimension na0 (leading block, AMB-19)
        const int na = na0;
        const double* fn = s.fproj + (int64_t)b * (ld + 1);
        double z0 = tid < na ? fn[tid] : 0.0, z1 = tid + 32 < na ? fn[tid + 32] : 0.0;
        warp_chol_solve(sA, ld, na, &z0, &z1, tid);
        if (tid < n) { z0 = tid < na ? z0 : 0.0; s.E[tid * s.Bp + b] = z0; s.a_n[(int64_t)b * ld + tid] = z0; }
        if (tid + 32 < n) {
            z1 = tid + 32 < na ? z1 : 0.0;
            s.E[(tid + 32) * s.Bp + b] = z1;
            s.a_n[(int64_t)b * ld + tid + 32] = z1;
        }
    }
}

// ---------------------------------------------------------------------------
// layout / init helpers
// ---------------------------------------------------------------------------
// W column-major (ldw) -> node-major [N8][ldwi], zero padded
__global__ void k_pack_W(const double* __restrict__ W, int64_t ldw, int64_t N, int64_t N8, int n,
                         int ldwi, double* __restrict__ Wi) {
    const int64_t tot = N8 * ldwi;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / ldwi;
        const int j = (int)(t - i * ldwi);
        Wi[t] = (i < N && j < n) ? W[(int64_t)j * ldw + i] : 0.0;
    }
}

// node-major [N8][ldwi] -> column-major N x n
__global__ void k_unpack_W(const double* __restrict__ Wi, int64_t N, int n, int ldwi,
                           double* __restrict__ W) {
    const int64_t tot = N * n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / N, i = t - j * N;
        W[t] = Wi[i * ldwi + j];
    }
}

// dst <- src (tot doubles) unless the solve's done flag is set: the Jacobi ping-pong's copy-back
// inside the iteration graph (after the last query froze the sweeps are no-ops and the
// scratch buffer is not the iterate any more)
__global__ void k_copy_unless_done(double* __restrict__ dst, const double* __restrict__ src, int64_t tot,
                                   const int* done) {
    if (done && ld_flag(done)) return;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x)
        dst[t] = src[t];
}

// v[N8][Bp] <- value (or from src [B][N] query-major when src != nullptr)
__global__ void k_fill_batch(double* __restrict__ v, int64_t N, int64_t N8, int Bp, int B,
                             const double* __restrict__ src, double value) {
    const int64_t tot = N8 * Bp;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / Bp;
        const int b = (int)(t - i * Bp);
        double x = 0.0;
        if (i < N && b < B) x = src ? src[(int64_t)b * N + i] : value;
        v[t] = x;
    }
}

// out[B][ldo] (query-major) <- v[N8][Bp] for N nodes; tiled transpose through shared memory
__global__ void k_transpose_out(const double* __restrict__ v, int64_t N, int Bp, int B,
                                double* __restrict__ out, int64_t ldo) {
    __shared__ double tile[32][kMaxBatch + 1];
    const int64_t i0 = (int64_t)blockIdx.x * 32;
    for (int t = threadIdx.x; t < 32 * Bp; t += blockDim.x) {
        const int r = t / Bp, b = t - r * Bp;
        tile[r][b] = (i0 + r < N) ? v[(i0 + r) * Bp + b] : 0.0;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 32 * B; t += blockDim.x) {
        const int b = t >> 5, r = t & 31;
        if (i0 + r < N) out[(int64_t)b * ldo + i0 + r] = tile[r][b];
    }
}

// offline: Z[i][j] = (A_q W[:,j])_i for the columns of the packed basis
// offline: Z[i][jj] = (A_q W[:, j0+jj])_i, jj < 8, for the packed basis
template <int DIM>
__global__ void __launch_bounds__(kThreads) k_apply_Aq(Geo g, int q, const double* __restrict__ Wi,
                                                       int npad, int j0, double* __restrict__ Z) {
    __shared__ double s_th[64];
    for (int t = threadIdx.x; t < g.Q; t += blockDim.x) s_th[t] = (t == q) ? 1.0 : 0.0;
    __syncthreads();
    const int64_t tot = g.N * 8;
    for (int64_t e = blockIdx.x * (int64_t)kThreads + threadIdx.x; e < tot;
         e += (int64_t)gridDim.x * kThreads) {
        const int64_t i = e >> 3;
        const int j = j0 + (int)(e & 7);
        int I, J, K;
        node_coords(g, (uint32_t)i, I, J, K);
        double k[2 * DIM], nb[2 * DIM];
        node_kappa<DIM>(g, s_th, 1, 0, I, J, K, k);
        node_nbrs<DIM>(g, Wi, npad, i, j, I, J, K, nb);
        Z[e] = stencil_apply<DIM>(g, k, Wi[i * npad + j], nb);
    }
}

// ---------------------------------------------------------------------------
// Mesh-slab mode: the passes write per-CTA partials of every
// slab into one column range each; these single-CTA kernels sum all columns in
// a fixed order and run the scalar step of the RBCG iteration.
//   k_slab_alpha: Step 5 alpha = rho / (p^T A p), MAXIT / CURVATURE
//   k_slab_beta:  Step 10 rho' = y^T r, PRECOND, beta = rho'/rho
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512) k_slab_alpha(SolveState s, int ncols) {
    if (ld_flag(s.done)) return;
    __shared__ double s_a[512];
    __shared__ double s_sig[kMaxBatch];
    cta_sum_slot(s, 0, s_a, s_sig, ncols);
    const int k = ld_flag(s.kcount);
    if (threadIdx.x < s.Bp) {
        const int bb = threadIdx.x;
        double al = 0.0;
        if (s.active[bb]) {
            const double sg = s_sig[bb];
            if (k >= s.maxit) { s.status[bb] = Q_MAXIT; s.its[bb] = k; s.active[bb] = 0; }
            else if (!(sg > 0.0)) {
                s.status[bb] = isfinite(sg) ? Q_CURVATURE : Q_NONFINITE;
                s.its[bb] = k;
                s.active[bb] = 0;
            } else al = s.rho[bb] / sg;
        }
        s.alpha[bb] = al;
    }
    __syncthreads();
    update_done(s);
}

__global__ void __launch_bounds__(512) k_slab_beta(SolveState s, int ncols, int init) {
    if (ld_flag(s.done)) return;
    __shared__ double s_a[512];
    __shared__ double s_yr[kMaxBatch], s_yy[kMaxBatch];
    cta_sum_slot(s, 0, s_a, s_yr, ncols);
    cta_sum_slot(s, 1, s_a, s_yy, ncols);
    if (threadIdx.x < s.Bp) {
        const int bb = threadIdx.x;
        if (s.active[bb]) {
            const double r1 = s_yr[bb], y2 = s_yy[bb];
            if (!(r1 > s.delta * sqrt(y2) * sqrt(s.rr[bb]))) {
                s.status[bb] = isfinite(r1) ? Q_PRECOND : Q_NONFINITE;
                s.active[bb] = 0;
                s.beta[bb] = 0.0;
            } else {
                s.beta[bb] = init ? 0.0 : r1 / s.rho[bb];
                s.rho[bb] = r1;
            }
        }
    }
    __syncthreads();
    const int any = cta_any_active(s);
    if (threadIdx.x == 0) {
        *(volatile int*)s.done = any ? 0 : 1;
        if (!init) *(volatile int*)s.kcount = *(volatile int*)s.kcount + 1;
    }
}

__global__ void k_update_done(const int* active, int Bp, int* done) {
    int any = 0;
    for (int b = 0; b < Bp; ++b) any |= active[b];
    *done = any ? 0 : 1;
}

}  // namespace rbs
