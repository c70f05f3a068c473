// march.cuh -- row-marching (2.5D-blocked) passes for 2D grids on sm_100a.
//
// A CTA owns a strip of TX nodes in x (plus a halo) and a segment of rows in
// y, and marches up the rows.  Row segments of the node-major batch vectors
// (contiguous in memory: nodes of one grid row are adjacent) are streamed
// into a shared-memory ring with cp.async.bulk (TMA bulk copies, SASS UBLKCP)
// completing on mbarriers, several rows ahead of the compute, so every byte
// is read from HBM once and all stencil reuse is served from shared memory.
//
// k_smooth_march fuses, per arriving row J_in:
//   y0(J_in)   = W e           (prolongation, eq7, DMMA)
//                (+ x_old when accumulating: RBI Step 6)
//   half-sweep s of the smoother on row J_in-1-s   (s = 0..S-1, AMB-5/6)
//   row J_in-S is final: stored, and y^T r / y^T y partials accumulated
// The lag of one row per half-sweep is exactly the red-black dependency, so
// the whole symmetric sweep R,B,R is one pass; the x-halo of S nodes is
// recomputed (bitwise identical to the neighbour's values).
#pragma once
#include "kernels.cuh"

namespace rbs {

// ---- mbarrier / bulk-copy primitives -----------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra LAB_WAIT%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

constexpr int kMarchThreads = 512;
constexpr int kMaxSweeps = 5;    // half-sweeps per smoother application (halo width)
constexpr int kPF = 2;           // rows prefetched ahead of the compute

// strip / segment partition of a 2D grid: nsx strips of TX nodes, nsy row segments
struct MarchPart {
    int nsx, nsy, rows_per_seg;
};

struct SmoothMarchArgs {
    Geo g;
    int Bp, npad, ldw;
    MarchPart part;
    const double* W;          // [N8][npad]
    const double* E;          // [npad][Bp]
    const double* Xold;       // accumulate: y0 = x_old + W e (RBI); else nullptr
    const double* Rhs;        // smoother right-hand side rows, or nullptr -> rconst
    double rconst;
    double* Y;                // output [N8][Bp]
    const double* theta;      // [Q][Bp]
    const int* active;
    int S;                    // number of half-sweeps
    int seq[kMaxSweeps];      // their colours
    int has_e;                // npad > 0
    int last;                 // LAST: y^T rhs, y^T y partials + Step 10 in the last CTA
    int init;
    SolveState s;
    const int* done;
};

// dynamic shared memory layout of k_smooth_march (R rows per step, 1 step prefetch)
constexpr int kRows = 2;

template <int TX>
struct SmoothSmem {
    int TW, RY, RR, RW, tiles;
    size_t yring, rring, wring, xring, es, cb, th, bars, total;
    __host__ __device__ SmoothSmem(int Bp, int npad, int ldw, int Q, int S, bool has_rhs, bool acc) {
        TW = TX + 2 * S;
        tiles = (TW + 7) / 8;
        RY = kRows + S + 1;
        RR = 2 * kRows + S;
        RW = 2 * kRows;
        size_t off = 0;
        auto take = [&](size_t bytes) { size_t o = off; off = (off + bytes + 127) & ~size_t(127); return o; };
        yring = take((size_t)RY * TW * Bp * 8);
        rring = take(has_rhs ? (size_t)RR * TW * Bp * 8 : 0);
        wring = take((size_t)RW * tiles * 8 * ldw * 8);
        xring = take(acc ? (size_t)RW * TW * Bp * 8 : 0);
        es = take((size_t)npad * (Bp + 4) * 8);      // row stride Bp + 4: conflict-free B fragments
        cb = take((size_t)2 * (TW + 2) * 4);
        th = take((size_t)Q * Bp * 8);
        bars = take(8 * 2 + 64);
        total = off;
    }
};

// (x mod n) for -n <= x < 2n without a division
__device__ __forceinline__ int wrapn(int x, int n) { return x >= n ? x - n : (x < 0 ? x + n : x); }

template <int TX>
__global__ void __launch_bounds__(kMarchThreads, 1) k_smooth_march(SmoothMarchArgs a) {
    if (a.done && ld_flag(a.done)) return;
    extern __shared__ __align__(128) unsigned char sm[];
    const int Bp = a.Bp, npad = a.npad, S = a.S, m = a.g.m;
    const bool has_rhs = a.Rhs != nullptr, acc = a.Xold != nullptr;
    SmoothSmem<TX> L(Bp, npad, a.ldw, a.g.Q, S, has_rhs, acc);
    const int ldw = a.ldw, Bpe = Bp + 4;
    double* yring = (double*)(sm + L.yring);
    double* rring = (double*)(sm + L.rring);
    double* wring = (double*)(sm + L.wring);
    double* xring = (double*)(sm + L.xring);
    double* Es = (double*)(sm + L.es);
    double* th = (double*)(sm + L.th);
    int* cbx = (int*)(sm + L.cb);      // [col][2]: x-blocks of cells I-1, I of window column col
    uint64_t* bars = (uint64_t*)(sm + L.bars);
    __shared__ int s_act[kMaxBatch];
    __shared__ double s_a[kMarchThreads], s_b[kMarchThreads];
    __shared__ double s_yr[kMaxBatch], s_yy[kMaxBatch];
    __shared__ int s_last;

    const int tid = threadIdx.x, H = S, TW = L.TW, RY = L.RY, RR = L.RR;
    const int sx = blockIdx.x % a.part.nsx, sy = blockIdx.x / a.part.nsx;
    const int x0 = 1 + sx * TX;                       // first owned node (1-based)
    const int y0 = 1 + sy * a.part.rows_per_seg;
    const int y1 = min(m + 1, y0 + a.part.rows_per_seg);   // exclusive
    const int xlo = x0 - H;                           // node of window column 0
    const int Imin = max(1, xlo), Imax = min(m, x0 + TX - 1 + H);
    const int ncopy = Imax - Imin + 1, coff = Imin - xlo;
    const int cmin = Imin - xlo, cmax = Imax - xlo;   // valid window columns

    // ---- init: zero the rings (invalid halo columns stay zero), stage E, theta
    for (size_t t = tid; t < (L.es - L.yring) / 8; t += kMarchThreads) ((double*)(sm + L.yring))[t] = 0.0;
    for (int t = tid; t < npad * Bp; t += kMarchThreads) {
        const int j = t / Bp, bb = t - j * Bp;
        Es[j * Bpe + bb] = a.has_e ? a.E[t] : 0.0;
    }
    for (int col = tid; col < L.TW; col += kMarchThreads) {
        const int I = min(max(xlo + col, 1), m);
        cbx[2 * col] = axis_block(a.g, I - 1, a.g.px);
        cbx[2 * col + 1] = axis_block(a.g, I, a.g.px);
    }
    for (int t = tid; t < a.g.Q * Bp; t += kMarchThreads) th[t] = a.theta[t];
    for (int t = tid; t < Bp; t += kMarchThreads) s_act[t] = a.active[t];
    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_fence_init();
    }
    __syncthreads();

    const int Jfirst = y0 - H, Jlast = y1 - 1 + H;   // rows whose y0 is formed
    const int nsteps = (Jlast - Jfirst + kRows) / kRows;
    const size_t wrow = (size_t)L.tiles * 8 * ldw;    // doubles per W slot
    const size_t vrow = (size_t)TW * Bp;              // doubles per vector slot
    const uint32_t wb = a.has_e ? (uint32_t)ncopy * ldw * 8 : 0u;
    const uint32_t vb = (uint32_t)ncopy * Bp * 8;
    // loads of step t: rows Jfirst + t*R + k, k < R (thread 0 only)
    auto issue = [&](int t) {
        uint64_t* bar = &bars[t & 1];
        uint32_t bytes = 0;
        for (int k = 0; k < kRows; ++k) {
            const int J = Jfirst + t * kRows + k;
            if (J >= 1 && J <= m && J <= Jlast) bytes += wb + (has_rhs ? vb : 0u) + (acc ? vb : 0u);
        }
        fence_async_smem();
        mbar_expect_tx(bar, bytes);
        for (int k = 0; k < kRows; ++k) {
            const int J = Jfirst + t * kRows + k;
            if (J < 1 || J > m || J > Jlast) continue;
            const int64_t n0 = (int64_t)(J - 1) * m + (Imin - 1);
            const int ws = (t & 1) * kRows + k;            // W / x slot
            const int u = t * kRows + k;                   // row index relative to Jfirst
            const int rs = u % RR;                         // r slot (once per row, thread 0)
            if (a.has_e) bulk_g2s(wring + ws * wrow + (size_t)coff * ldw, a.W + n0 * ldw, wb, bar);
            if (has_rhs) bulk_g2s(rring + rs * vrow + (size_t)coff * Bp, a.Rhs + n0 * Bp, vb, bar);
            if (acc) bulk_g2s(xring + ws * vrow + (size_t)coff * Bp, a.Xold + n0 * Bp, vb, bar);
        }
    };
    if (tid == 0) issue(0);

    const int warp = tid >> 5, lane = tid & 31;
    const int lgB = 31 - __clz(Bp), nbt = Bp >> 3, lgnbt = 31 - __clz(nbt);
    const int b = tid & (Bp - 1);           // fixed query per thread
    const int cstride = kMarchThreads >> lgB;
    const int cfirst = tid >> lgB;
    const bool qact = s_act[b] != 0;
    const int npairs = L.tiles * nbt, nk = npad >> 2;
    double yr = 0.0, yy = 0.0;

    int ysb = 0;   // y slot of row Jfirst + t*R
    int rsb = 0;   // r slot of row Jfirst + t*R
    for (int t = 0; t < nsteps; ++t) {
        const int Jb = Jfirst + t * kRows;
        if (tid == 0 && t + 1 < nsteps) issue(t + 1);
        mbar_wait(&bars[t & 1], (uint32_t)((t >> 1) & 1));
        // ---- y0 for rows Jb .. Jb+R-1 (DMMA: M = 8 nodes, N = 8 queries, K = 4)
        for (int k = 0; k < kRows; ++k) {
            const int J = Jb + k;
            if (!(J >= 1 && J <= m && J <= Jlast)) {
                double* ynew = yring + (size_t)wrapn(ysb + k, RY) * vrow;
                for (size_t e = tid; e < vrow; e += kMarchThreads) ynew[e] = 0.0;
            }
        }
        for (int task = warp; task < kRows * npairs; task += kMarchThreads / 32) {
            int k = 0, pr = task;
            while (pr >= npairs) { pr -= npairs; ++k; }
            const int J = Jb + k;
            if (J >= 1 && J <= m && J <= Jlast) {
                double* ynew = yring + (size_t)wrapn(ysb + k, RY) * vrow;
                const double* Ws = wring + ((t & 1) * kRows + k) * wrow;
                const double* Xs = xring + ((t & 1) * kRows + k) * vrow;
                {
                    const int bt = pr & (nbt - 1), tile = pr >> lgnbt;
                    double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
                    const double* wr = Ws + (size_t)(tile * 8 + (lane >> 2)) * ldw + (lane & 3);
                    const double* ec = Es + (lane & 3) * Bpe + bt * 8 + (lane >> 2);
                    int kk = 0;
                    for (; kk + 1 < nk; kk += 2) {
                        dmma_8x8x4(d0, d1, wr[kk * 4], ec[kk * 4 * Bpe]);
                        dmma_8x8x4(e0, e1, wr[kk * 4 + 4], ec[(kk + 1) * 4 * Bpe]);
                    }
                    if (kk < nk) dmma_8x8x4(d0, d1, wr[kk * 4], ec[kk * 4 * Bpe]);
                    d0 += e0;
                    d1 += e1;
                    const int col = tile * 8 + (lane >> 2);
                    if (col >= cmin && col <= cmax) {
                        const int bb = bt * 8 + 2 * (lane & 3);
                        if (acc) {
                            d0 += Xs[(size_t)col * Bp + bb];
                            d1 += Xs[(size_t)col * Bp + bb + 1];
                        }
                        *reinterpret_cast<double2*>(ynew + (size_t)col * Bp + bb) = make_double2(d0, d1);
                    }
                }
            }
        }
        __syncthreads();
        // ---- half-sweeps: sweep s on rows Jb-1-s .. Jb+R-2-s, window columns s+1 .. TW-2-s
        for (int s = 0; s < S; ++s) {
            const int hw = H - 1 - s;
            const int c0 = max(s + 1, cmin), c1 = min(TW - 2 - s, cmax);
            const int color = a.seq[s];
            if (qact) {
#pragma unroll
                for (int k = 0; k < kRows; ++k) {
                    const int J = Jb - 1 - s + k;
                    if (J < y0 - hw || J > y1 - 1 + hw || J < 1 || J > m) continue;
                    const int sl = wrapn(ysb - 1 - s + k, RY);
                    double* yc = yring + (size_t)sl * vrow;
                    const double* ydn = yring + (size_t)wrapn(sl - 1, RY) * vrow;
                    const double* yup = yring + (size_t)wrapn(sl + 1, RY) * vrow;
                    const double* rs = rring + (size_t)wrapn(rsb - 1 - s + k, RR) * vrow;
                    const int cs = c0 + ((color - (xlo + c0 + J)) & 1);   // first column of `color`
                    const int by0 = axis_block(a.g, J - 1, a.g.py) * a.g.px;
                    const int by1 = axis_block(a.g, J, a.g.py) * a.g.px;
                    for (int col = cs + 2 * cfirst; col <= c1; col += 2 * cstride) {
                        double kap[4], nb[4];
                        kappa2_blocks(th, Bp, b, cbx[2 * col], cbx[2 * col + 1], by0, by1, kap);
                        const size_t e = (size_t)col * Bp + b;
                        nb[0] = yc[e - Bp];
                        nb[1] = yc[e + Bp];
                        nb[2] = ydn[e];
                        nb[3] = yup[e];
                        const double rhs = has_rhs ? rs[e] : a.rconst;
                        yc[e] = gs_value<2>(a.g, kap, rhs, nb);
                    }
                }
            }
            __syncthreads();
        }
        // ---- rows Jb-S .. Jb-S+R-1 are final
#pragma unroll
        for (int k = 0; k < kRows; ++k) {
            const int Jo = Jb - S + k;
            if (Jo < y0 || Jo >= y1) continue;    // all lanes: a frozen RBI lane has e = 0
            const double* yo = yring + (size_t)wrapn(ysb - S + k, RY) * vrow;
            const double* rs = rring + (size_t)wrapn(rsb - S + k, RR) * vrow;
            const int c0 = H, c1 = min(H + TX - 1, cmax);
            double* yg = a.Y + ((int64_t)(Jo - 1) * m + (xlo - 1)) * Bp;
            for (int col = c0 + cfirst; col <= c1; col += cstride) {
                const size_t e = (size_t)col * Bp + b;
                const double v = yo[e];
                yg[e] = v;
                if (a.last) {
                    const double rv = has_rhs ? rs[e] : a.rconst;
                    yr = fma(v, rv, yr);
                    yy = fma(v, v, yy);
                }
            }
        }
        ysb = wrapn(ysb + kRows, RY);
        rsb = wrapn(rsb + kRows, RR);
        __syncthreads();   // every read of this step is done before slots are re-armed
    }
    if (!a.last) return;
    // ---- partials and RBCG Step 10 in the last CTA (as in k_gs<LAST>) --------
    SolveState& s = a.s;
    s_a[tid] = yr;
    s_b[tid] = yy;
    __syncthreads();
    if (tid < Bp) {
        double sr = 0.0, sq = 0.0;
        for (int t = tid; t < kMarchThreads; t += Bp) {
            sr += s_a[t];
            sq += s_b[t];
        }
        s.partF[((int64_t)tid * 2 + 0) * s.nctf + blockIdx.x] = sr;
        s.partF[((int64_t)tid * 2 + 1) * s.nctf + blockIdx.x] = sq;
    }
    if (cta_is_last(s.ticket, &s_last)) {
        cta_sum_slot(s, 0, s_a, s_yr);
        cta_sum_slot(s, 1, s_a, s_yy);
        if (tid < s.Bp) {
            const int bb = tid;
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
        if (tid == 0) {
            *(volatile int*)s.done = any ? 0 : 1;
            if (!a.init) *(volatile int*)s.kcount = *(volatile int*)s.kcount + 1;
        }
        release_ticket(s.ticket);
    }
}

}  // namespace rbs

namespace rbs {

// ---------------------------------------------------------------------------
// k_resid_march: the projection pass as a row march (2D).
//   MODE_CG    (RBCG Steps 6-8): q = A p, x += alpha p,
//              r -= alpha q (x, r stored), v = r
//   MODE_RESID (RBI Step 2): v = f - A x (not stored)
// Per step (row J): stage A forms v on row J (stencil from the p / x ring,
// halo 1) and parks it in shared memory; stage B contracts row J-1 with W on
// the FP64 tensor cores (D[j][b] += W[node][j] v[node][b], W^T v, eq5).  The
// stages touch different rows, so one barrier per row suffices.  Each warp
// owns fixed (j-tile, b-tile) accumulators for the whole march, so the
// per-CTA partials need no combination: deterministic.
// ---------------------------------------------------------------------------
constexpr int kRmTX = 32;
constexpr int kRmPF = 2;

struct ResidMarchArgs {
    Geo g;
    int Bp, npad, ldw;
    MarchPart mp;
    const double* W;          // [N8][ldw]
    const double* theta;      // [Q][Bp]
    const int* active;        // [Bp] or nullptr
    const double* alpha;      // MODE_CG
    const double* P;          // MODE_CG stencil input
    double* X;                // MODE_CG rw / MODE_RESID stencil input
    double* R;                // MODE_CG rw
    const double* V;          // MODE_RESID rhs rows or nullptr -> vconst
    double vconst;
    double* part;             // [Bp][npad+1][nct]
    int nct;
    const int* done;
};

struct ResidSmem {
    size_t sring, xring, rring, vring, wring, th, bars, total;
    __host__ __device__ ResidSmem(int Bp, int ldw, int Q, int mode, bool has_v) {
        size_t off = 0;
        auto take = [&](size_t bytes) { size_t o = off; off = (off + bytes + 127) & ~size_t(127); return o; };
        const size_t row1 = (size_t)(kRmTX + 2) * Bp * 8, row0 = (size_t)kRmTX * Bp * 8;
        sring = take((3 + kRmPF) * row1);                                 // stencil input, halo 1
        xring = take(mode == 0 ? (2 + kRmPF) * row0 : 0);                 // x (CG)
        rring = take(mode == 0 ? (2 + kRmPF) * row0 : 0);                 // r (CG)
        vring = take(mode == 1 && has_v ? (2 + kRmPF) * row0 : 0);        // rhs rows (RESID)
        wring = take((size_t)(3 + kRmPF) * kRmTX * ldw * 8);
        th = take((size_t)Q * Bp * 8 + 2 * (size_t)kRmTX * (Bp + 4) * 8);  // theta + new-v rows
        bars = take(8 * (kRmPF + 1) + 64);
        total = off;
    }
};

template <int MODE>
__global__ void __launch_bounds__(kMarchThreads, 1) k_resid_march(ResidMarchArgs a) {
    if (a.done && ld_flag(a.done)) return;
    extern __shared__ __align__(128) unsigned char sm[];
    const int Bp = a.Bp, npad = a.npad, ldw = a.ldw, m = a.g.m, Bpv = Bp + 4;
    const bool has_v = a.V != nullptr;
    ResidSmem L(Bp, ldw, a.g.Q, MODE, has_v);
    double* sring = (double*)(sm + L.sring);
    double* xring = (double*)(sm + L.xring);
    double* rring = (double*)(sm + L.rring);
    double* vring = (double*)(sm + L.vring);
    double* wring = (double*)(sm + L.wring);
    double* th = (double*)(sm + L.th);
    double* vnew = th + a.g.Q * Bp;            // 2 rows of [kRmTX][Bp+4]
    uint64_t* bars = (uint64_t*)(sm + L.bars);
    __shared__ int s_act[kMaxBatch];
    __shared__ double s_alpha[kMaxBatch];
    __shared__ int s_cbx[2 * (kRmTX + 2)];
    __shared__ double s_rr[kMarchThreads];

    const int tid = threadIdx.x;
    const int sx = blockIdx.x % a.mp.nsx, sy = blockIdx.x / a.mp.nsx;
    const int x0 = 1 + sx * kRmTX;
    const int y0 = 1 + sy * a.mp.rows_per_seg;
    const int y1 = min(m + 1, y0 + a.mp.rows_per_seg);
    const int xlo = x0 - 1;                        // window column 0 = node x0-1
    const int Imin = max(1, xlo), Imax = min(m, x0 + kRmTX);   // stencil input range
    const int nc = min(kRmTX, m - x0 + 1);                       // owned nodes
    const int ncs = Imax - Imin + 1, coffs = Imin - xlo;
    const size_t row1 = (size_t)(kRmTX + 2) * Bp, row0 = (size_t)kRmTX * Bp, wrowd = (size_t)kRmTX * ldw;

    for (size_t t = tid; t < (L.th - L.sring) / 8; t += kMarchThreads) ((double*)(sm + L.sring))[t] = 0.0;
    for (int t = tid; t < a.g.Q * Bp; t += kMarchThreads) th[t] = a.theta[t];
    for (int t = tid; t < 2 * kRmTX * Bpv; t += kMarchThreads) vnew[t] = 0.0;
    for (int t = tid; t < Bp; t += kMarchThreads) {
        s_act[t] = a.active ? a.active[t] : 1;
        s_alpha[t] = MODE == 0 ? a.alpha[t] : 0.0;
    }
    for (int col = tid; col < kRmTX + 2; col += kMarchThreads) {
        const int I = min(max(xlo + col, 1), m);
        s_cbx[2 * col] = axis_block(a.g, I - 1, a.g.px);
        s_cbx[2 * col + 1] = axis_block(a.g, I, a.g.px);
    }
    if (tid == 0) {
        for (int k = 0; k <= kRmPF; ++k) mbar_init(&bars[k], 1);
        mbar_fence_init();
    }
    __syncthreads();

    const double* Sin = MODE == 0 ? a.P : a.X;      // stencil input
    // step t handles stage A on row J = y0 - 1 + t (t = 0 loads row y0-1 only) and
    // stage B on row J - 1; the ring row index of row J is u = J - (y0 - 1).
    const int Jbase = y0 - 1;
    const int nsteps = (y1 - y0) + 2;                // J = y0-1 .. y1 = ring rows 0 .. nsteps-1
    auto issue = [&](int u) {                        // loads of ring row u (row Jbase + u)
        const int J = Jbase + u;
        uint64_t* bar = &bars[u % (kRmPF + 1)];
        const bool srow = J >= 1 && J <= m;                  // stencil row (halo rows too)
        const bool crow = J >= y0 && J < y1;                 // owned row: centre data + W
        uint32_t bytes = 0;
        const uint32_t sb = (uint32_t)ncs * Bp * 8, cb = (uint32_t)nc * Bp * 8, wb = (uint32_t)nc * ldw * 8;
        if (srow) bytes += sb;
        if (crow) bytes += wb + (MODE == 0 ? 2 * cb : (has_v ? cb : 0u));
        fence_async_smem();
        mbar_expect_tx(bar, bytes);
        if (srow) {
            const int64_t n0 = (int64_t)(J - 1) * m + (Imin - 1);
            bulk_g2s(sring + (u % (3 + kRmPF)) * row1 + (size_t)coffs * Bp, Sin + n0 * Bp, sb, bar);
        }
        if (crow) {
            const int64_t n0 = (int64_t)(J - 1) * m + (x0 - 1);
            const int cs = u % (2 + kRmPF);
            bulk_g2s(wring + (u % (3 + kRmPF)) * wrowd, a.W + n0 * ldw, wb, bar);
            if (MODE == 0) {
                bulk_g2s(xring + cs * row0, a.X + n0 * Bp, cb, bar);
                bulk_g2s(rring + cs * row0, a.R + n0 * Bp, cb, bar);
            } else if (has_v) {
                bulk_g2s(vring + cs * row0, a.V + n0 * Bp, cb, bar);
            }
        }
    };
    // ring row u holds row Jbase + u; stage A on row J needs rows J-1..J+1 -> u+1 must be loaded
    if (tid == 0)
        for (int u = 0; u <= kRmPF && u < nsteps; ++u) issue(u);

    const int warp = tid >> 5, lane = tid & 31;
    const int lgB = 31 - __clz(Bp), nbt = Bp >> 3, lgnbt = 31 - __clz(nbt);
    const int b = tid & (Bp - 1), cfirst = tid >> lgB, cstride = kMarchThreads >> lgB;
    const bool qact = s_act[b] != 0;
    const double al = s_alpha[b];
    const int npairs = (npad >> 3) * nbt;
    double acc[4][2];
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k][0] = acc[k][1] = 0.0;
    double rr = 0.0;

    for (int t = 0; t < nsteps; ++t) {
        const int J = Jbase + t;                 // stage A row (u = t); ring row t+1 = J+1
        // row t+PF+1 re-arms the barrier of row t: that phase must have completed
        // (waited here at t = 0, at step t-1 otherwise) before thread 0 re-arms it
        if (t == 0) mbar_wait(&bars[0], 0u);
        if (tid == 0 && t + kRmPF + 1 < nsteps) issue(t + kRmPF + 1);
        if (t + 1 < nsteps) mbar_wait(&bars[(t + 1) % (kRmPF + 1)], (uint32_t)(((t + 1) / (kRmPF + 1)) & 1));
        // zero stencil rows outside the domain (no copy was issued for them)
        if (t + 1 < nsteps && (J + 1 < 1 || J + 1 > m)) {
            double* z = sring + ((t + 1) % (3 + kRmPF)) * row1;
            for (size_t e = tid; e < row1; e += kMarchThreads) z[e] = 0.0;
            __syncthreads();
        }
        // ---- stage A: row J (owned rows only)
        double* vA = vnew + (size_t)(t & 1) * kRmTX * Bpv;
        if (J >= y0 && J < y1 && qact) {
            const double* sc = sring + (t % (3 + kRmPF)) * row1;
            const double* sd = sring + ((t + 3 + kRmPF - 1) % (3 + kRmPF)) * row1;
            const double* su = sring + ((t + 1) % (3 + kRmPF)) * row1;
            const int cs = t % (2 + kRmPF);
            const double* xs = xring + cs * row0;
            const double* rs = rring + cs * row0;
            const double* vs = vring + cs * row0;
            const int by0 = axis_block(a.g, J - 1, a.g.py) * a.g.px, by1 = axis_block(a.g, J, a.g.py) * a.g.px;
            double* xg = a.X + ((int64_t)(J - 1) * m + (x0 - 1)) * Bp;
            double* rg = a.R + ((int64_t)(J - 1) * m + (x0 - 1)) * Bp;
            for (int c = cfirst; c < nc; c += cstride) {
                const size_t e = (size_t)(c + 1) * Bp + b;     // stencil window index
                double kap[4], nb[4];
                kappa2_blocks(th, Bp, b, s_cbx[2 * (c + 1)], s_cbx[2 * (c + 1) + 1], by0, by1, kap);
                nb[0] = sc[e - Bp];
                nb[1] = sc[e + Bp];
                nb[2] = sd[e];
                nb[3] = su[e];
                const double q = stencil_apply<2>(a.g, kap, sc[e], nb);
                const size_t o = (size_t)c * Bp + b;
                double v;
                if (MODE == 0) {
                    const double xv = fma(al, sc[e], xs[o]);
                    v = fma(-al, q, rs[o]);
                    xg[o] = xv;
                    rg[o] = v;
                } else {
                    v = (has_v ? vs[o] : a.vconst) - q;
                }
                vA[c * Bpv + b] = v;
                rr = fma(v, v, rr);
            }
        } else if (J >= y0 && J < y1) {
            for (int c = cfirst; c < nc; c += cstride) vA[c * Bpv + b] = 0.0;
        }
        // ---- stage B: W^T v on row J-1 (DMMA, K = 4 nodes per step)
        const int JB = J - 1;
        if (JB >= y0 && JB < y1) {
            const double* vB = vnew + (size_t)((t + 1) & 1) * kRmTX * Bpv;
            const double* Ws = wring + ((t - 1 + 3 + kRmPF) % (3 + kRmPF)) * wrowd;
            const int nks = (nc + 3) >> 2;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int pr = warp + k * (kMarchThreads / 32);
                if (pr < npairs) {
                    const int bt = pr & (nbt - 1), jt = pr >> lgnbt;
                    const double* wa = Ws + (size_t)(lane & 3) * ldw + jt * 8 + (lane >> 2);
                    const double* vb = vB + (size_t)(lane & 3) * Bpv + bt * 8 + (lane >> 2);
                    for (int ks = 0; ks < nks; ++ks)
                        dmma_8x8x4(acc[k][0], acc[k][1], wa[(size_t)ks * 4 * ldw], vb[(size_t)ks * 4 * Bpv]);
                }
            }
        }
        __syncthreads();
    }
    // ---- per-CTA partials: (j, b) owned by exactly one warp-task
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int pr = warp + k * (kMarchThreads / 32);
        if (pr < npairs) {
            const int bt = pr & (nbt - 1), jt = pr >> lgnbt;
            const int j = jt * 8 + (lane >> 2), bb = bt * 8 + 2 * (lane & 3);
            a.part[((int64_t)bb * (npad + 1) + j) * a.nct + blockIdx.x] = acc[k][0];
            a.part[((int64_t)(bb + 1) * (npad + 1) + j) * a.nct + blockIdx.x] = acc[k][1];
        }
    }
    s_rr[tid] = rr;
    __syncthreads();
    if (tid < Bp) {
        double v = 0.0;
        for (int u = tid; u < kMarchThreads; u += Bp) v += s_rr[u];
        a.part[((int64_t)tid * (npad + 1) + npad) * a.nct + blockIdx.x] = v;
    }
}

}  // namespace rbs
