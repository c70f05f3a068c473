// march2.cuh -- lean row-marching passes for 2D grids (sm_100a), v2.
//
// The three streaming passes of an RBCG iteration on a 2D grid (and the two
// of an RBI iteration), each as a row march: a CTA owns a strip of 32 columns
// (+ halo) and a segment of rows and walks up the rows; row windows of the
// node-major batch vectors arrive by TMA bulk copy (cp.async.bulk, SASS
// UBLKCP) into shared-memory rings completing on mbarriers, so every byte is
// read from HBM once and every stencil / temporal-blocking reuse is served
// from shared memory.  Every pass has ONE barrier per row.
//
// v1 (march.cuh) was issue-bound at 150-400 thread-instructions per
// node-query (ncu, profiles/r1_v1_ncu_c2.md); this version is templated on
// the padded batch BP and on the number of half-sweeps S so every ring stride
// is a compile-time constant and per-row bases are hoisted out of the element
// loops; nodes whose four cells lie in one block (all but the block
// interfaces) use one table lookup instead of the four cell averages.
//
//   k_cgp2      RBCG Step 11 + sigma of Step 5
//   k_resid2    RBCG Steps 6-8 + W^T r / RBI Step 2+4
//   k_smooth2   prolongation + smoother (+ y^T r)
#pragma once
#include "march.cuh"

namespace rbs {

// RBS_CLK: per-warp cycle accounting of k_smooth2 (instrumented builds only, tools/s2clk.py)
#ifdef RBS_CLK
__device__ unsigned long long g_s2clk[148 * 16 * 6];
__device__ unsigned long long g_s2t[148 * 3];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define S2CLK_ENTRY if (threadIdx.x == 0 && blockIdx.x < 148) g_s2t[blockIdx.x * 3] = gtimer();
#define S2CLK_DECL unsigned long long c_[6] = {0, 0, 0, 0, 0, 0}; long long t_ = clock64(), u_; \
    if (threadIdx.x == 0 && blockIdx.x < 148) g_s2t[blockIdx.x * 3 + 1] = gtimer();
#define S2CLK(k) do { u_ = clock64(); c_[k] += (unsigned long long)(u_ - t_); t_ = u_; } while (0)
#define S2CLK_FLUSH do { if (threadIdx.x == 0 && blockIdx.x < 148) g_s2t[blockIdx.x * 3 + 2] = gtimer(); \
    if (lane == 0 && blockIdx.x < 148) for (int k_ = 0; k_ < 6; ++k_) \
    atomicAdd(&g_s2clk[(blockIdx.x * 16 + warp) * 6 + k_], c_[k_]); } while (0)
#else
#define S2CLK_ENTRY
#define S2CLK_DECL
#define S2CLK(k) do {} while (0)
#define S2CLK_FLUSH do {} while (0)
#endif
constexpr int kMT = kMarchThreads;        // 512 threads, 16 warps
constexpr int kNW = kMT / 32;

template <int BP>
struct LgB {
    static constexpr int v = BP == 8 ? 3 : BP == 16 ? 4 : BP == 32 ? 5 : 6;
};

// explicit 32-bit shared-memory accesses: the hot loops keep one u32 base per
// ring row in a register instead of letting the compiler rematerialise the
// shared window base for every access (ncu: ~25 extra instructions per element)
__device__ __forceinline__ double ldsd(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void stsd(uint32_t a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void stsd2(uint32_t a, double v0, double v1) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v0), "d"(v1) : "memory");
}

// (A p)_P for a node whose 4 cells are in one block: scale*theta*(4 p - sum nb)
__device__ __forceinline__ double stencil_uniform(double st, double c, double n0, double n1, double n2,
                                                  double n3) {
    return st * fma(4.0, c, -((n0 + n1) + (n2 + n3)));
}

// per-column block info of a window: bx of the left cell | bx of the right cell << 8,
// and -1 / bx for the "uniform in x" test
__device__ __forceinline__ void fill_colinfo(const Geo& g, int xlo, int ncols, int* cinfo, int* cuni) {
    for (int col = threadIdx.x; col < ncols; col += blockDim.x) {
        const int I = min(max(xlo + col, 1), g.m);
        const int b0 = axis_block(g, I - 1, g.px), b1 = axis_block(g, I, g.px);
        cinfo[col] = b0 | (b1 << 8);
        cuni[col] = b0 == b1 ? b0 : -1;
    }
}

// per-row y-block offsets: rb[u] = by(cell row Jfirst + u - 1) * px, u in [0, nr)
__device__ __forceinline__ void fill_rowinfo(const Geo& g, int Jfirst, int nr, int* rb) {
    for (int u = threadIdx.x; u < nr; u += blockDim.x) {
        const int a = min(max(Jfirst + u - 1, 0), g.m);
        rb[u] = axis_block(g, a, g.py) * g.px;
    }
}

// ===========================================================================
// k_smooth2<BP, S>: per arriving row Jb (step t):
//   lag 0       y0(Jb) = W e (+ x_old)              DMMA (eq7)
//   lag 2(s+1)  half-sweep s on row Jb - 2(s+1)     (eq8, AMB-5/6)
//   lag 2S+1    row final: stored, y^T r, y^T y
// Half-sweep s reads rows R-1..R+1, whose opposite-colour nodes were last
// written by half-sweep s-1 (two rows up, an earlier step) and are next
// written by s+1 (two rows down, a later step): no two stages of a step touch
// the same row, so the red-black order is exact with one barrier per row.
// ===========================================================================
constexpr int kS2TX = 32;       // strip width (24 when the rings of 32 do not fit)
constexpr int kS2YR = 8;         // y ring rows (lags 0 .. 2S+1 <= 7)
constexpr int kS2RR = 8;         // r ring rows (issued at lag 0, last read at lag 2S+1)
// W / x_old ring rows: template parameter WR of k_smooth2 (3: prefetch distance 2;
// 2: distance 1, when the 3-row ring would push the strip width down to 24)
constexpr int kS2NTW = 4;                 // tensor warps
constexpr int kS2NVT = kMT - 32 * kS2NTW; // vector threads (384)

// dynamic shared memory (doubles):
//   y ring 8 | r ring 8 (has_rhs) | x_old ring 3 (acc) | E (npad x (Bp+4)) |
//   W ring 3 x (tiles*8 x ldw) | theta | h^2/(4 theta)
struct Smooth2Smem {
    int vrow, xo, eo, wo, tho, cho, wrow;
    size_t total;
    __host__ __device__ Smooth2Smem(int TX, int S, int Bp, int ldw, int Q, bool has_rhs, bool acc, int npad,
                                    int WR = 3) {
        const int TW = TX + 2 * S, tiles = (TW + 7) / 8;
        vrow = TW * Bp;
        wrow = tiles * 8 * ldw;
        xo = (kS2YR + (has_rhs ? kS2RR : 0)) * vrow;
        eo = xo + (acc ? WR * vrow : 0);
        wo = eo + ((npad * (Bp + 4) + 15) & ~15);
        tho = wo + WR * wrow;
        cho = tho + Q * Bp;
        total = (size_t)(cho + Q * Bp) * 8;
    }
};

// Warp roles: warps 0..3 (tensor warps) run the prolongation of the arriving
// row on the FP64 tensor pipe (1 DMMA / 16 cycles / SMSP bounds the pass);
// warps 4..15 (vector warps) are split into S groups, group s running
// half-sweep s (one column of every column pair has the sweep's colour), and
// all 12 share the output row.  Every shared-memory load of a step is issued
// before any update of that step.
template <int BP, int S, bool HAS_RHS, int TX, int WR, int NKC = 0>
__global__ void __launch_bounds__(kMT, 1) k_smooth2(SmoothMarchArgs a) {
    // NKC > 0: the basis width npad / 4 fixed at compile time, so the k loop of the
    // prolongation unrolls completely (no loop-carried branch; loads scheduled ahead)
    constexpr int kS2WR = WR, kS2D = WR - 1;
    S2CLK_ENTRY
    constexpr int LGB = LgB<BP>::v;
    constexpr int TW = TX + 2 * S;
    constexpr int VROW = TW * BP;
    constexpr int TILES = (TW + 7) / 8;
    constexpr int NBT = BP / 8;
    constexpr int NPAIRS = TW / 2;
    constexpr int GW = S > 0 ? (kS2NVT / 32) / S : 1;        // warps per sweep group
    constexpr int GT = GW * 32;                              // threads per sweep group
    constexpr int PPI = GT >> LGB;                           // pairs per slot round
    // the output row is stored by the vector threads of groups >= OG: with three half-sweeps
    // group 0 (the widest cone) skips it, so the per-row work of the groups evens out
    constexpr int OG = S == 3 ? 1 : 0;
    constexpr int NOT = kS2NVT - OG * GT;                   // output threads
    constexpr int JO = (TX * BP + NOT - 1) / NOT;           // output slots per thread
    constexpr int YR = 0, RR = kS2YR * VROW;
    extern __shared__ __align__(128) double smd[];
    __shared__ int s_ci[TW], s_cu[TW];
    __shared__ __align__(8) uint64_t wbar[kS2WR], rbar[kS2RR];
    __shared__ int s_act[kMaxBatch];
    __shared__ double s_yr[kMaxBatch], s_yy[kMaxBatch];
    __shared__ int s_last;
    const int m = a.g.m, ldw = a.ldw, npad = a.npad;
    constexpr bool has_rhs = HAS_RHS;
    const bool acc = a.Xold != nullptr;
    const uint32_t sbase = smem_u32(smd);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int sx = blockIdx.x % a.part.nsx, sy = blockIdx.x / a.part.nsx;
    const int x0 = 1 + sx * TX;
    const int y0 = 1 + sy * a.part.rows_per_seg;
    const int y1 = min(m + 1, y0 + a.part.rows_per_seg);   // exclusive
    const int xlo = x0 - S;                                  // node of window column 0
    const int Imin = max(1, xlo), Imax = min(m, x0 + TX - 1 + S);
    const int ncopy = Imax - Imin + 1, coff = Imin - xlo;
    const int cmin = Imin - xlo, cmax = Imax - xlo;          // valid window columns
    const int Jfirst = y0 - S;                               // row of step 0
    const int JlastP = y1 - 1 + S;                           // last prolongated row
    const int nsteps = (y1 - y0) + 3 * S + 1;                // last output row y1-1 at lag 2S+1
    const Smooth2Smem L(TX, S, BP, ldw, a.g.Q, has_rhs, acc, npad, WR);
    const int XO = L.xo, EO = L.eo, WO = L.wo, THO = L.tho, CHO = L.cho, WROW = L.wrow;

    // ---- init: zero the rings (Dirichlet columns/rows stay zero), tables ------
    for (int t = tid; t < EO; t += kMT) smd[t] = 0.0;
    for (int t = tid; t < kS2WR * WROW; t += kMT) smd[WO + t] = 0.0;
    for (int t = tid; t < a.g.Q * BP; t += kMT) {
        const double v = a.theta[t];
        smd[THO + t] = v;
        smd[CHO + t] = a.g.h2 / (4.0 * v);
    }
    fill_colinfo(a.g, xlo, TW, s_ci, s_cu);
    if (tid == 0) {
        for (int k = 0; k < kS2WR; ++k) mbar_init(&wbar[k], 1);
        for (int k = 0; k < kS2RR; ++k) mbar_init(&rbar[k], 1);
        mbar_fence_init();
    }
    pdl_wait();                       // E, the active flags, r and x_old come from earlier passes
    if (a.done && ld_flag(a.done)) return;
    for (int t = tid; t < WO - EO; t += kMT) {
        const int j = t / (BP + 4), bb = t - j * (BP + 4);
        smd[EO + t] = (a.has_e && j < npad && bb < BP) ? a.E[j * BP + bb] : 0.0;
    }
    for (int t = tid; t < BP; t += kMT) s_act[t] = a.active[t];
    __syncthreads();

    const uint32_t wb = a.has_e ? (uint32_t)ncopy * ldw * 8 : 0u;
    const uint32_t vb = (uint32_t)ncopy * BP * 8;
    auto issue_w = [&](int u) {          // W (+ x_old) of row Jfirst + u (thread 0)
        const int J = Jfirst + u;
        const bool in = J >= 1 && J <= m;
        const int ws = u % kS2WR;
        uint64_t* bar = &wbar[ws];
        fence_async_smem();
        mbar_expect_tx(bar, in ? wb + (acc ? vb : 0u) : 0u);
        if (!in) return;
        const int64_t n0 = (int64_t)(J - 1) * m + (Imin - 1);
        if (a.has_e) bulk_g2s(smd + WO + ws * WROW + coff * ldw, a.W + n0 * ldw, wb, bar);
        if (acc) bulk_g2s(smd + XO + ws * VROW + coff * BP, a.Xold + n0 * BP, vb, bar);
    };
    auto issue_r = [&](int u) {          // smoother rhs row Jfirst + u (thread 0)
        const int J = Jfirst + u;
        const bool in = J >= 1 && J <= m;
        const int rs = u & (kS2RR - 1);
        uint64_t* bar = &rbar[rs];
        fence_async_smem();
        mbar_expect_tx(bar, in ? vb : 0u);
        if (!in) return;
        const int64_t n0 = (int64_t)(J - 1) * m + (Imin - 1);
        bulk_g2s(smd + RR + rs * VROW + coff * BP, a.Rhs + n0 * BP, vb, bar);
    };
    if (tid == 0)
        for (int u = 0; u < kS2D && Jfirst + u <= JlastP; ++u) issue_w(u);

    const bool tensor = warp < kS2NTW;
    const int b = tid & (BP - 1);
    const bool qact = s_act[b] != 0;
    const double rconst = a.rconst;
    double yr = 0.0, yy = 0.0;
    // ---- tensor warps: query tile bt, tiles tile0 + k*TSTEP ----------------------
    constexpr int LGNBT = LGB - 3;
    constexpr int TSTEP = kS2NTW >> LGNBT;
    const int nk = NKC > 0 ? NKC : npad >> 2;
    const int bt = warp & (NBT - 1), tile0 = warp >> LGNBT;
    constexpr int TPW = (TILES + TSTEP - 1) / TSTEP;                 // tiles per tensor warp
    const int eoff = EO + (lane & 3) * (BP + 4) + bt * 8 + (lane >> 2);   // B fragments (E)
    // ---- vector threads: sweep group, pair slots, output slots (loop-invariant) --
    const int vtid = tid - 32 * kS2NTW;
    const int grp = S > 0 ? min(vtid / GT, S - 1) : 0;
    const int tg = vtid - grp * GT;
    const int p0 = tg >> LGB;                                 // first pair of this thread
    const int sgi = S > 0 ? grp : 0;
    const int c0g = max(sgi + 1, cmin), c1g = min(TW - 2 - sgi, cmax);
    const int hwg = S - 1 - sgi;
    const int rlog = max(1, y0 - hwg), rhig = min(m, y1 - 1 + hwg);
    const int colg = a.seq[sgi] - xlo;                       // colour term of this group's sweep
    // block column info of this thread's nodes (both parities) in registers: the
    // h^2/(4 theta) load of a node does not wait on a column-table load
    constexpr int ITER = (NPAIRS + PPI - 1) / PPI;
    int cu0[ITER], cu1[ITER];
#pragma unroll
    for (int i = 0; i < ITER; ++i) {
        const int pp = p0 + i * PPI;
        cu0[i] = pp < NPAIRS ? s_cu[2 * pp] : -1;
        cu1[i] = pp < NPAIRS ? s_cu[2 * pp + 1] : -1;
    }
    const int nco = min(S + TX - 1, cmax) - S + 1;        // owned output columns
    double* yg = a.Y + ((int64_t)(Jfirst - (2 * S + 1) - 1) * m + (x0 - 1)) * BP;

    S2CLK_DECL
    for (int t = 0; t < nsteps; ++t, yg += (int64_t)m * BP) {
        const int Jb = Jfirst + t;
        if (tid == 0) {
            if (Jb + kS2D <= JlastP) issue_w(t + kS2D);
            if (has_rhs && Jb <= JlastP) issue_r(t);
        }
        S2CLK(0);
        if (tensor) {
            // ---- stage P: y0 of row Jb (lag 0) --------------------------------
            if (Jb <= JlastP) {
                const int ws = t % kS2WR;
                mbar_wait(&wbar[ws], (uint32_t)((t / kS2WR) & 1));
                S2CLK(1);
                const int yn = YR + (t & (kS2YR - 1)) * VROW;
                const int xs = XO + ws * VROW;
                if (Jb < 1 || Jb > m) {
                    for (int e = tid; e < VROW; e += 32 * kS2NTW) smd[yn + e] = 0.0;
                } else if (!a.has_e) {
                    for (int e = tid + cmin * BP; e < (cmax + 1) * BP; e += 32 * kS2NTW)
                        smd[yn + e] = acc ? smd[xs + e] : 0.0;
                } else {
                    // all tiles of this warp at once: TPW independent accumulator chains,
                    // the E fragment of each k-step shared by the tiles
                    const uint32_t wsb = sbase + 8u * (WO + ws * WROW + (tile0 * 8 + (lane >> 2)) * ldw + (lane & 3));
                    const uint32_t tstr = 8u * TSTEP * 8 * ldw;
                    uint32_t ea = sbase + 8u * eoff;
                    double d0[TPW], d1[TPW];
#pragma unroll
                    for (int i = 0; i < TPW; ++i) d0[i] = d1[i] = 0.0;
#pragma unroll (NKC > 0 ? NKC / 2 : 1)
                    for (int kk = 0; kk < nk; kk += 2, ea += 8u * 8 * (BP + 4)) {
                        const double e0 = ldsd(ea), e1 = ldsd(ea + 8u * 4 * (BP + 4));
                        double wa[TPW], wb2[TPW];
#pragma unroll
                        for (int i = 0; i < TPW; ++i) {
                            const bool tv = TPW * TSTEP == TILES || tile0 + i * TSTEP < TILES;
                            const uint32_t w = wsb + (tv ? i : 0) * tstr + 32u * kk;
                            wa[i] = ldsd(w);
                            wb2[i] = ldsd(w + 32u);
                        }
#pragma unroll
                        for (int i = 0; i < TPW; ++i)
                            if (TPW * TSTEP == TILES || tile0 + i * TSTEP < TILES) dmma_8x8x4(d0[i], d1[i], wa[i], e0);
#pragma unroll
                        for (int i = 0; i < TPW; ++i)
                            if (TPW * TSTEP == TILES || tile0 + i * TSTEP < TILES) dmma_8x8x4(d0[i], d1[i], wb2[i], e1);
                    }
#pragma unroll
                    for (int i = 0; i < TPW; ++i) {
                        const int col = (tile0 + i * TSTEP) * 8 + (lane >> 2);
                        if (col >= cmin && col <= cmax) {
                            const int o = col * BP + bt * 8 + 2 * (lane & 3);
                            double v0 = d0[i], v1 = d1[i];
                            if (acc) {
                                v0 += smd[xs + o];
                                v1 += smd[xs + o + 1];
                            }
                            *reinterpret_cast<double2*>(smd + yn + o) = make_double2(v0, v1);
                        }
                    }
                }
            }
        } else {
            // r of row Jb - RL (issued at its lag 0) is first read at lag RL
            constexpr int RL = S == 0 ? 1 : 2;
            if (has_rhs && t >= RL && Jb - RL <= JlastP)
                mbar_wait(&rbar[(t - RL) & (kS2RR - 1)], (uint32_t)(((t - RL) >> 3) & 1));
            S2CLK(1);
            // ---- half-sweep of this group on row R = Jb - 2(grp+1) ----------------
            const int R = Jb - 2 * (sgi + 1);
            if (S > 0 && R >= rlog && R <= rhig && qact) {
                const int par = (colg - R) & 1;
                const int sl = (t - 2 * (sgi + 1)) & (kS2YR - 1);
                const uint32_t yc = sbase + 8u * (YR + sl * VROW + b);
                const uint32_t ydn = sbase + 8u * (YR + ((sl - 1) & (kS2YR - 1)) * VROW + b);
                const uint32_t yup = sbase + 8u * (YR + ((sl + 1) & (kS2YR - 1)) * VROW + b);
                const uint32_t rrw = sbase + 8u * (RR + ((t - 2 * (sgi + 1)) & (kS2RR - 1)) * VROW + b);
                const int by0 = axis_block(a.g, R - 1, a.g.py) * a.g.px;
                const int by1 = axis_block(a.g, R, a.g.py) * a.g.px;
                const bool rowu = by0 == by1;
                const uint32_t chb = sbase + 8u * (CHO + by0 * BP + b);
#pragma unroll
                for (int i = 0; i < ITER; ++i) {
                    const int p = p0 + i * PPI;
                    const int col = 2 * p + par;
                    if (p >= NPAIRS || col < c0g || col > c1g) continue;
                    const int cu = par ? cu1[i] : cu0[i];
                    const uint32_t o = 8u * col * BP;
                    const double n0 = ldsd(yc + o - 8 * BP), n1 = ldsd(yc + o + 8 * BP);
                    const double n2 = ldsd(ydn + o), n3 = ldsd(yup + o);
                    const double rh = HAS_RHS ? ldsd(rrw + o) : rconst;
                    double v;
                    if (rowu && cu >= 0) {
                        v = fma(ldsd(chb + 8u * cu * BP), rh, 0.25 * ((n0 + n1) + (n2 + n3)));
                    } else {
                        const int ci = s_ci[col];
                        double kap[4], nb[4] = {n0, n1, n2, n3};
                        kappa2_blocks(smd + THO, BP, b, ci & 0xff, ci >> 8, by0, by1, kap);
                        v = gs_value<2>(a.g, kap, rh, nb);
                    }
                    stsd(yc + o, v);
                }
            }
            S2CLK(2);
            // ---- output row Ro = Jb - (2S+1): stores + y^T r, y^T y -----------------
            const int Ro = Jb - (2 * S + 1);
            const int ot = vtid - OG * GT;
            if (ot >= 0 && Ro >= y0 && Ro < y1) {
                const uint32_t yo = sbase + 8u * (YR + ((t - (2 * S + 1)) & (kS2YR - 1)) * VROW + S * BP);
                const uint32_t ro = sbase + 8u * (RR + ((t - (2 * S + 1)) & (kS2RR - 1)) * VROW + S * BP);
#pragma unroll
                for (int j = 0; j < JO; ++j) {
                    const int e = ot + j * NOT;
                    if ((e >> LGB) >= nco) break;
                    const double v = ldsd(yo + 8u * e);
                    yg[e] = v;
                    if (a.last) {
                        const double rv = HAS_RHS ? ldsd(ro + 8u * e) : rconst;
                        yr = fma(v, rv, yr);
                        yy = fma(v, v, yy);
                    }
                }
            }
        }
        S2CLK(3);
        __syncthreads();
        S2CLK(4);
    }
    S2CLK_FLUSH;
    pdl_trigger();
    if (!a.last) return;
    // ---- partials and RBCG Step 10 in the last CTA (rings are dead) ----------
    double* s_a = smd;
    double* s_b = smd + kMT;
    SolveState& s = a.s;
    s_a[tid] = yr;
    s_b[tid] = yy;
    __syncthreads();
    if (tid < BP) {
        double sr = 0.0, sq = 0.0;
        for (int u = tid; u < kMT; u += BP) {
            sr += s_a[u];
            sq += s_b[u];
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

// ===========================================================================
// k_cgp2<BP>: RBCG Step 11 + the sigma of Step 5.
//   lag 0: p_new = y + beta p_old on the arriving row (window of 34 columns),
//          stored for the owned columns
//   lag 2: q = A p_new on row Jb - 2 (its rows were formed in earlier steps),
//          sigma partial += p_new . q
// The last CTA forms alpha = rho / sigma with the MAXIT / CURVATURE checks.
// ===========================================================================
constexpr int kC2TX = 32;
constexpr int kC2D = 3;          // prefetch distance (rows)
constexpr int kC2R = 4;          // raw y / p_old ring rows (>= D + 1, pow2)
constexpr int kC2P = 4;          // p_new ring rows (lags 0..3)

struct CGP2Args {
    Geo g;
    int Bp;
    MarchPart part;
    const double* theta;
    const int* active;
    const double* beta;
    const double* Y;
    const double* Pold;
    double* Pnew;
    SolveState s;
    const int* done;
};

// dynamic shared memory (doubles): y ring | p ring | p_new ring | scale*theta table
__host__ __device__ inline size_t cgp2_smem_bytes(int Bp, int Q) {
    return ((size_t)(kC2R + kC2R + kC2P) * (kC2TX + 2) * Bp + (size_t)Q * Bp) * 8;
}

template <int BP>
__global__ void __launch_bounds__(kMT, 2) k_cgp2(CGP2Args a) {
    constexpr int LGB = LgB<BP>::v;
    constexpr int TW = kC2TX + 2;
    constexpr int VROW = TW * BP;
    constexpr int YR = 0, PR = kC2R * VROW, NR = 2 * kC2R * VROW, ST = NR + kC2P * VROW;
    constexpr int JA = (TW * BP + kMT - 1) / kMT;      // p_new slots per thread
    constexpr int JB = (kC2TX * BP + kMT - 1) / kMT;   // stencil slots per thread
    extern __shared__ __align__(128) double smd[];
    __shared__ int s_ci[TW], s_cu[TW];
    __shared__ __align__(8) uint64_t bars[kC2R];
    __shared__ double s_a[kMT];
    __shared__ double s_sig[kMaxBatch];
    __shared__ int s_last;
    const int m = a.g.m;
    const int tid = threadIdx.x;
    const int sx = blockIdx.x % a.part.nsx, sy = blockIdx.x / a.part.nsx;
    const int x0 = 1 + sx * kC2TX;
    const int y0 = 1 + sy * a.part.rows_per_seg;
    const int y1 = min(m + 1, y0 + a.part.rows_per_seg);
    const int xlo = x0 - 1;
    const int Imin = max(1, xlo), Imax = min(m, x0 + kC2TX);
    const int ncopy = Imax - Imin + 1, coff = Imin - xlo;
    const int cmin = Imin - xlo, cmax = Imax - xlo;
    const int nown = min(kC2TX, cmax);                 // owned window columns 1..nown
    const int Jfirst = y0 - 1;                         // rows y0-1 .. y1 are formed
    const int nform = y1 - y0 + 2;
    const int nsteps = y1 - y0 + 3;                    // stencil row y1-1 at lag 2

    for (int t = tid; t < ST; t += kMT) smd[t] = 0.0;
    for (int t = tid; t < a.g.Q * BP; t += kMT) smd[ST + t] = a.g.scale * a.theta[t];
    fill_colinfo(a.g, xlo, TW, s_ci, s_cu);
    if (tid == 0) {
        for (int k = 0; k < kC2R; ++k) mbar_init(&bars[k], 1);
        mbar_fence_init();
    }
    pdl_wait();                       // y, p_old, beta and the flags come from earlier passes
    if (a.done && ld_flag(a.done)) return;
    __syncthreads();
    const uint32_t vb = (uint32_t)ncopy * BP * 8;
    auto issue = [&](int u) {
        const int J = Jfirst + u;
        const bool in = J >= 1 && J <= m;
        uint64_t* bar = &bars[u & (kC2R - 1)];
        fence_async_smem();
        mbar_expect_tx(bar, in ? 2 * vb : 0u);
        if (!in) return;
        const int64_t n0 = (int64_t)(J - 1) * m + (Imin - 1);
        const int so = (u & (kC2R - 1)) * VROW + coff * BP;
        bulk_g2s(smd + YR + so, a.Y + n0 * BP, vb, bar);
        bulk_g2s(smd + PR + so, a.Pold + n0 * BP, vb, bar);
    };
    if (tid == 0)
        for (int u = 0; u < kC2D && u < nform; ++u) issue(u);

    const int b = tid & (BP - 1);
    const double bet = a.beta[b];
    // loop-invariant slot data
    int oa[JA];
    bool va[JA], wa[JA];
#pragma unroll
    for (int j = 0; j < JA; ++j) {
        oa[j] = tid + cmin * BP + j * kMT;
        va[j] = oa[j] < (cmax + 1) * BP;
        wa[j] = oa[j] >= BP && oa[j] < (nown + 1) * BP;
        if (!va[j]) oa[j] = 0;
    }
    int ob[JB], cub[JB], cib[JB];
    bool vbq[JB];
#pragma unroll
    for (int j = 0; j < JB; ++j) {
        const int item = (tid >> LGB) + j * (kMT >> LGB);
        vbq[j] = item < nown;
        const int col = vbq[j] ? item + 1 : 1;
        ob[j] = col * BP + b;
        cub[j] = s_cu[col];
        cib[j] = s_ci[col];
    }
    const uint32_t sbase = smem_u32(smd);
    double sig = 0.0;
    double* pg = a.Pnew + ((int64_t)(Jfirst - 1) * m + (xlo - 1)) * BP;
    for (int t = 0; t < nsteps; ++t, pg += (int64_t)m * BP) {
        const int Jb = Jfirst + t;
        if (tid == 0 && t + kC2D < nform) issue(t + kC2D);
        const bool arow = t < nform;
        if (arow) mbar_wait(&bars[t & (kC2R - 1)], (uint32_t)((t / kC2R) & 1));
        const bool ain = arow && Jb >= 1 && Jb <= m;
        const int ya = YR + (t & (kC2R - 1)) * VROW, pa = PR + (t & (kC2R - 1)) * VROW;
        const int na = NR + (t & (kC2P - 1)) * VROW;
        // ---- loads: stage A (row Jb) and stage B (rows Jb-3 .. Jb-1) ---------
        double yv[JA], pv[JA];
        const uint32_t yA = sbase + 8u * ya, pA = sbase + 8u * pa, nA = sbase + 8u * na;
#pragma unroll
        for (int j = 0; j < JA; ++j) {
            yv[j] = ldsd(yA + 8u * oa[j]);
            pv[j] = ldsd(pA + 8u * oa[j]);
        }
        const int R = Jb - 2;
        const bool brow = R >= y0 && R < y1;
        const int nc_ = NR + ((t - 2) & (kC2P - 1)) * VROW, nd_ = NR + ((t - 3) & (kC2P - 1)) * VROW;
        const int nu_ = NR + ((t - 1) & (kC2P - 1)) * VROW;
        double qc[JB], q0[JB], q1[JB], q2[JB], q3[JB];
        const uint32_t cA = sbase + 8u * nc_, dA = sbase + 8u * nd_, uA = sbase + 8u * nu_;
#pragma unroll
        for (int j = 0; j < JB; ++j) {
            const uint32_t o = 8u * ob[j];
            qc[j] = ldsd(cA + o);
            q0[j] = ldsd(cA + o - 8 * BP);
            q1[j] = ldsd(cA + o + 8 * BP);
            q2[j] = ldsd(dA + o);
            q3[j] = ldsd(uA + o);
        }
        // ---- stage A: p_new = y + beta p_old -----------------------------------
        if (ain) {
#pragma unroll
            for (int j = 0; j < JA; ++j) {
                const double v = fma(bet, pv[j], yv[j]);
                if (va[j]) stsd(nA + 8u * oa[j], v);
                if (wa[j]) pg[oa[j]] = v;
            }
        } else if (arow) {
            for (int e = tid; e < VROW; e += kMT) smd[na + e] = 0.0;
        }
        // ---- stage B: sigma += p_new . (A p_new) on row R ----------------------
        if (brow) {
            const int by0 = axis_block(a.g, R - 1, a.g.py) * a.g.px, by1 = axis_block(a.g, R, a.g.py) * a.g.px;
            const bool rowu = by0 == by1;
#pragma unroll
            for (int j = 0; j < JB; ++j) {
                if (!vbq[j]) continue;
                double q;
                if (rowu && cub[j] >= 0) {
                    q = stencil_uniform(ldsd(sbase + 8u * (ST + (cub[j] + by0) * BP + b)), qc[j], q0[j], q1[j], q2[j],
                                        q3[j]);
                } else {
                    double kap[4], nb[4] = {q0[j], q1[j], q2[j], q3[j]};
                    kappa2_blocks(a.theta, BP, b, cib[j] & 0xff, cib[j] >> 8, by0, by1, kap);
                    q = stencil_apply<2>(a.g, kap, qc[j], nb);
                }
                sig = fma(qc[j], q, sig);
            }
        }
        __syncthreads();
    }
    pdl_trigger();
    // ---- partials; last CTA: alpha = rho / sigma, MAXIT / CURVATURE (Step 5)
    SolveState& s = a.s;
    s_a[tid] = sig;
    __syncthreads();
    if (tid < BP) {
        double t0 = 0.0;
        for (int u = tid; u < kMT; u += BP) t0 += s_a[u];
        s.partF[((int64_t)tid * 2 + 0) * s.nctf + blockIdx.x] = t0;
    }
    if (cta_is_last(s.ticket, &s_last)) {
        cta_sum_slot(s, 0, s_a, s_sig);
        const int k = ld_flag(s.kcount);
        if (tid < s.Bp) {
            const int bb = tid;
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

// ===========================================================================
// k_resid2<BP, MODE>: the projection pass as a row march.
//   MODE 0 (RBCG Steps 6-8): q = A p, x += alpha p,
//          r -= alpha q (x, r stored), v = r
//   MODE 1 (RBI Step 2): v = f - A x (not stored)
// Stage A (row J = y0-1+t) forms v and parks it in shared memory; stage B
// contracts the previous row's v with W on the FP64 tensor cores (W^T v,
// eq5), split into (j-tile, b-tile, k-quarter) tasks so the 16 warps carry
// equal DMMA loads; the quarters are combined in a fixed order at the end.
// ===========================================================================
// prefetch distance PF (rows): 2, or 1 when the rings of 2 do not fit (large n)
// dynamic shared memory (doubles): stencil ring | x ring | r (or f) ring |
//   parked v (2 rows, stride Bp+4) | W ring (ldw) | scale*theta
__host__ __device__ inline size_t resid2_smem_bytes(int PF, int Bp, int ldw, int Q) {
    const int NS = 3 + PF, NC = 2 + PF;
    const size_t fixed = (size_t)NS * (kRmTX + 2) * Bp + 2 * (size_t)NC * kRmTX * Bp +
                         2 * (size_t)kRmTX * (Bp + 4);
    return (fixed + (size_t)NS * kRmTX * ldw + (size_t)Q * Bp) * 8;
}

template <int BP, int MODE, int kR2PF>
__global__ void __launch_bounds__(kMT, 1) k_resid2(ResidMarchArgs a) {
    constexpr int kR2NS = 3 + kR2PF;     // stencil-input / W ring rows
    constexpr int kR2NC = 2 + kR2PF;     // x / r / f ring rows
    constexpr int LGB = LgB<BP>::v;
    constexpr int BPV = BP + 4;
    constexpr int NBT = BP / 8, LGNBT = LGB - 3;
    constexpr int ROW1 = (kRmTX + 2) * BP, ROW0 = kRmTX * BP;
    constexpr int SR = 0, XR = kR2NS * ROW1, RRg = XR + kR2NC * ROW0, VN = RRg + kR2NC * ROW0;
    constexpr int WR = VN + 2 * kRmTX * BPV;
    constexpr int JA = (kRmTX * BP + kMT - 1) / kMT;
    extern __shared__ __align__(128) double smd[];
    __shared__ int s_ci[kRmTX + 2], s_cu[kRmTX + 2];
    __shared__ __align__(8) uint64_t bars[kR2PF + 1];
    __shared__ int s_act[kMaxBatch];
    __shared__ double s_alpha[kMaxBatch];
    __shared__ double s_rr[kMT];
    const int npad = a.npad, ldw = a.ldw, m = a.g.m;
    const bool has_v = a.V != nullptr;
    const int tid = threadIdx.x;
    const int sx = blockIdx.x % a.mp.nsx, sy = blockIdx.x / a.mp.nsx;
    const int x0 = 1 + sx * kRmTX;
    const int y0 = 1 + sy * a.mp.rows_per_seg;
    const int y1 = min(m + 1, y0 + a.mp.rows_per_seg);
    const int xlo = x0 - 1;
    const int Imin = max(1, xlo), Imax = min(m, x0 + kRmTX);
    const int nc = min(kRmTX, m - x0 + 1);
    const int ncs = Imax - Imin + 1, coffs = Imin - xlo;
    const int Jbase = y0 - 1;
    const int nsteps = (y1 - y0) + 2;
    const int WROWD = kRmTX * ldw;
    const int STo = WR + kR2NS * WROWD;

    for (int t = tid; t < STo; t += kMT) smd[t] = 0.0;
    for (int t = tid; t < a.g.Q * BP; t += kMT) smd[STo + t] = a.g.scale * a.theta[t];
    fill_colinfo(a.g, xlo, kRmTX + 2, s_ci, s_cu);
    if (tid == 0) {
        for (int k = 0; k <= kR2PF; ++k) mbar_init(&bars[k], 1);
        mbar_fence_init();
    }
    pdl_wait();                       // p, x, r, alpha and the flags come from earlier passes
    if (a.done && ld_flag(a.done)) return;
    for (int t = tid; t < BP; t += kMT) {
        s_act[t] = a.active ? a.active[t] : 1;
        s_alpha[t] = MODE == 0 ? a.alpha[t] : 0.0;
    }
    __syncthreads();

    const double* Sin = MODE == 0 ? a.P : a.X;
    auto issue = [&](int u) {
        const int J = Jbase + u;
        uint64_t* bar = &bars[u % (kR2PF + 1)];
        const bool srow = J >= 1 && J <= m;
        const bool crow = J >= y0 && J < y1;
        const uint32_t sb = (uint32_t)ncs * BP * 8, cb = (uint32_t)nc * BP * 8, wb = (uint32_t)nc * ldw * 8;
        uint32_t bytes = 0;
        if (srow) bytes += sb;
        if (crow) bytes += wb + (MODE == 0 ? 2 * cb : (has_v ? cb : 0u));
        fence_async_smem();
        mbar_expect_tx(bar, bytes);
        if (srow) {
            const int64_t n0 = (int64_t)(J - 1) * m + (Imin - 1);
            bulk_g2s(smd + SR + (u % kR2NS) * ROW1 + coffs * BP, Sin + n0 * BP, sb, bar);
        }
        if (crow) {
            const int64_t n0 = (int64_t)(J - 1) * m + (x0 - 1);
            const int cs = u % kR2NC;
            bulk_g2s(smd + WR + (u % kR2NS) * WROWD, a.W + n0 * ldw, wb, bar);
            if (MODE == 0) {
                bulk_g2s(smd + XR + cs * ROW0, a.X + n0 * BP, cb, bar);
                bulk_g2s(smd + RRg + cs * ROW0, a.R + n0 * BP, cb, bar);
            } else if (has_v) {
                bulk_g2s(smd + RRg + cs * ROW0, a.V + n0 * BP, cb, bar);
            }
        }
    };
    if (tid == 0)
        for (int u = 0; u <= kR2PF && u < nsteps; ++u) issue(u);

    const int warp = tid >> 5, lane = tid & 31;
    const int b = tid & (BP - 1);
    const bool qact = s_act[b] != 0;
    const double al = s_alpha[b];
    const double vconst = a.vconst;
    // DMMA tasks (pair = (j-tile, b-tile), k-quarter of the 32-node row), contiguous per warp
    const int npairs = (npad >> 3) * NBT;
    const int ntask = npairs * 4;
    const int ntpw = (ntask + kNW - 1) / kNW;
    const int t0 = warp * ntpw;
    const int myn = max(0, min(ntpw, ntask - t0));
    int wofs[8], vofs[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int task = t0 + k;
        const int pr = task >> 2, kq = task & 3;
        const int btt = pr & (NBT - 1), jt = pr >> LGNBT;
        wofs[k] = (kq * 8 + (lane & 3)) * ldw + jt * 8 + (lane >> 2);
        vofs[k] = VN + (kq * 8 + (lane & 3)) * BPV + btt * 8 + (lane >> 2);
    }
    double acc[8][2];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k][0] = acc[k][1] = 0.0;
    // stage-A slots (loop-invariant): owned column c, its block info
    int oc[JA], ocu[JA], oci[JA];
    bool ov_[JA];
#pragma unroll
    for (int j = 0; j < JA; ++j) {
        const int c = (tid >> LGB) + j * (kMT >> LGB);
        ov_[j] = c < nc;
        oc[j] = ov_[j] ? c : 0;
        ocu[j] = s_cu[oc[j] + 1];
        oci[j] = s_ci[oc[j] + 1];
    }
    const uint32_t sbase = smem_u32(smd);
    double rr = 0.0;
    int sl_c = 0, sl_n = 1, sl_d = kR2NS - 1;    // ring slots of rows J, J+1, J-1 (mod NS)
    int sl_x = 0;                                // ring slot of row J (mod NC)
    double* xg = a.X + ((int64_t)(Jbase - 1) * m + (x0 - 1)) * BP + b;
    double* rg = a.R + ((int64_t)(Jbase - 1) * m + (x0 - 1)) * BP + b;

    for (int t = 0; t < nsteps; ++t, xg += (int64_t)m * BP, rg += (int64_t)m * BP) {
        const int J = Jbase + t;
        if (t == 0) mbar_wait(&bars[0], 0u);
        if (tid == 0 && t + kR2PF + 1 < nsteps) issue(t + kR2PF + 1);
        if (t + 1 < nsteps) mbar_wait(&bars[(t + 1) % (kR2PF + 1)], (uint32_t)(((t + 1) / (kR2PF + 1)) & 1));
        if (t + 1 < nsteps && (J + 1 < 1 || J + 1 > m)) {
            const int z = SR + sl_n * ROW1;
            for (int e = tid; e < ROW1; e += kMT) smd[z + e] = 0.0;
            __syncthreads();
        }
        // ---- stage A loads: row J -------------------------------------------------
        const bool arow = J >= y0 && J < y1;
        const int sc = SR + sl_c * ROW1 + BP + b, sd = SR + sl_d * ROW1 + BP + b;
        const int su = SR + sl_n * ROW1 + BP + b;
        const int xs = XR + sl_x * ROW0 + b, rs = RRg + sl_x * ROW0 + b;
        double pc[JA], q0[JA], q1[JA], q2[JA], q3[JA], xa[JA], ra[JA];
        const uint32_t scA = sbase + 8u * sc, sdA = sbase + 8u * sd, suA = sbase + 8u * su;
        const uint32_t xsA = sbase + 8u * xs, rsA = sbase + 8u * rs;
#pragma unroll
        for (int j = 0; j < JA; ++j) {
            const uint32_t o = 8u * oc[j] * BP;
            pc[j] = ldsd(scA + o);
            q0[j] = ldsd(scA + o - 8 * BP);
            q1[j] = ldsd(scA + o + 8 * BP);
            q2[j] = ldsd(sdA + o);
            q3[j] = ldsd(suA + o);
            if (MODE == 0) {
                xa[j] = ldsd(xsA + o);
                ra[j] = ldsd(rsA + o);
            } else {
                ra[j] = has_v ? ldsd(rsA + o) : vconst;
            }
        }
        // ---- stage B: W^T v on row J-1 (DMMA) -----------------------------------
        const int JB = J - 1;
        if (JB >= y0 && JB < y1) {
            const int vB = ((t + 1) & 1) * kRmTX * BPV;
            const int Ws = WR + sl_d * WROWD;
            const uint32_t WsA = sbase + 8u * Ws, vBA = sbase + 8u * vB;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (k >= myn) break;
                const uint32_t wa = WsA + 8u * wofs[k], vb = vBA + 8u * vofs[k];
                const double a0 = ldsd(wa), b0 = ldsd(vb), a1 = ldsd(wa + 32u * ldw), b1 = ldsd(vb + 32u * BPV);
                dmma_8x8x4(acc[k][0], acc[k][1], a0, b0);
                dmma_8x8x4(acc[k][0], acc[k][1], a1, b1);
            }
        }
        // ---- stage A compute / stores -------------------------------------------
        if (arow) {
            const int vA = VN + (t & 1) * kRmTX * BPV + b;
            const int by0 = axis_block(a.g, J - 1, a.g.py) * a.g.px, by1 = axis_block(a.g, J, a.g.py) * a.g.px;
            const bool rowu = by0 == by1;
#pragma unroll
            for (int j = 0; j < JA; ++j) {
                if (!ov_[j]) continue;
                const int o = oc[j] * BP;
                double v = 0.0;
                if (qact) {
                    double q;
                    if (rowu && ocu[j] >= 0) {
                        q = stencil_uniform(ldsd(sbase + 8u * (STo + (ocu[j] + by0) * BP + b)), pc[j], q0[j], q1[j],
                                            q2[j], q3[j]);
                    } else {
                        double kap[4], nb[4] = {q0[j], q1[j], q2[j], q3[j]};
                        kappa2_blocks(a.theta, BP, b, oci[j] & 0xff, oci[j] >> 8, by0, by1, kap);
                        q = stencil_apply<2>(a.g, kap, pc[j], nb);
                    }
                    if (MODE == 0) {
                        const double xv = fma(al, pc[j], xa[j]);
                        v = fma(-al, q, ra[j]);
                        xg[o] = xv;
                        rg[o] = v;
                    } else {
                        v = ra[j] - q;
                    }
                    rr = fma(v, v, rr);
                }
                stsd(sbase + 8u * (vA + oc[j] * BPV), v);
            }
        }
        __syncthreads();
        sl_d = sl_c;
        sl_c = sl_n;
        sl_n = sl_n + 1 == kR2NS ? 0 : sl_n + 1;
        sl_x = sl_x + 1 == kR2NC ? 0 : sl_x + 1;
    }
    pdl_trigger();
    // ---- per-CTA partials: the 4 k-quarters of each (j-tile, b-tile) in order
    double* s_q = smd;          // rings are dead: [ntask][64]
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (k >= myn) break;
        const int task = t0 + k;
        s_q[task * 64 + 2 * lane] = acc[k][0];
        s_q[task * 64 + 2 * lane + 1] = acc[k][1];
    }
    s_rr[tid] = rr;
    __syncthreads();
    for (int idx = tid; idx < npairs * 64; idx += kMT) {
        const int pr = idx >> 6, w = idx & 63;            // w = 2*lane + h
        const double v = ((s_q[(pr * 4 + 0) * 64 + w] + s_q[(pr * 4 + 1) * 64 + w]) +
                          s_q[(pr * 4 + 2) * 64 + w]) + s_q[(pr * 4 + 3) * 64 + w];
        const int ln = w >> 1, h = w & 1;
        const int btt = pr & (NBT - 1), jt = pr >> LGNBT;
        const int j = jt * 8 + (ln >> 2), bb = btt * 8 + 2 * (ln & 3) + h;
        a.part[((int64_t)bb * (npad + 1) + j) * a.nct + blockIdx.x] = v;
    }
    if (tid < BP) {
        double v = 0.0;
        for (int u = tid; u < kMT; u += BP) v += s_rr[u];
        a.part[((int64_t)tid * (npad + 1) + npad) * a.nct + blockIdx.x] = v;
    }
}

}  // namespace rbs

namespace rbs {
// ===========================================================================
// k_wtr<BP>: the projection W^T v and ||v||^2 as a stream over a contiguous node
// range per CTA (any dimension; the 3D second half of K2, eq5).
// Chunks of kWtCH nodes of W (ldw doubles per node) and v (BP per node) arrive by
// TMA bulk copies into a kWtD-slot ring (mbarriers, kWtD-1 chunks in flight); each
// chunk of v is first copied to a padded buffer (row stride BP+4: the DMMA B-fragment
// reads of a half-warp then hit 16 distinct 8-byte banks; the dense rows are 4-way
// conflicted) while ||v||^2 is accumulated; warps own (8-basis x 8-query) tiles with
// two accumulator chains (even / odd k-steps) and split the chunk's k-steps when there
// are fewer tiles than warps; chains, k-parts and the per-thread ||v||^2 terms are summed
// in a fixed order.  Partials go to part[b][j][col] exactly like k_proj (stage 2:
// k_reduce_solve).
// ===========================================================================
constexpr int kWtD = 4;

inline size_t wtr_smem_bytes(int Bp, int ldw, int ch) {
    return (size_t)kWtD * ch * (ldw + Bp) * 8 + (size_t)ch * (Bp + 4) * 8 + 256;
}

template <int BP, int kWtCH>
__global__ void __launch_bounds__(kMT, 2) k_wtr(ProjArgs a) {
    if (a.done && ld_flag(a.done)) return;
    extern __shared__ __align__(128) double smd[];
    __shared__ __align__(8) uint64_t bars[kWtD];
    __shared__ double s_red[kNW * 64];
    __shared__ double s_rr[kMT];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int npad = a.npad, ldw = a.ldw, ntile = npad >> 3;
    constexpr int NBT = BP / 8;
    constexpr int LDV = BP + 4;                               // padded v row
    const int T = ntile * NBT;                                // output tiles
    const int KP = T >= kNW ? 1 : min(kWtCH / 4, kNW / T);   // k-parts per tile (k-steps split)
    const int64_t N = a.g.N;
    const int64_t n0 = N * blockIdx.x / gridDim.x, n1 = N * (blockIdx.x + 1) / gridDim.x;
    const int nch = (int)((n1 - n0 + kWtCH - 1) / kWtCH);
    const int slotW = kWtCH * ldw, slotV = kWtCH * BP;
    double* wr = smd;
    double* vr = smd + kWtD * slotW;
    double* vp = vr + kWtD * slotV;                           // padded copy of the current v chunk
    if (tid == 0) {
        for (int k = 0; k < kWtD; ++k) mbar_init(&bars[k], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int c) {             // chunk c -> slot c % kWtD (thread 0)
        const int64_t i0 = n0 + (int64_t)c * kWtCH;
        const int cnt = (int)(n1 - i0 < (int64_t)kWtCH ? n1 - i0 : (int64_t)kWtCH);
        const int sl = c % kWtD;
        uint64_t* bar = &bars[sl];
        fence_async_smem();
        const uint32_t bw = (uint32_t)cnt * ldw * 8, bv = (uint32_t)cnt * BP * 8;
        mbar_expect_tx(bar, bw + bv);
        bulk_g2s(wr + sl * slotW, a.W + i0 * ldw, bw, bar);
        bulk_g2s(vr + sl * slotV, a.V + i0 * BP, bv, bar);
    };
    if (tid == 0)
        for (int c = 0; c < kWtD - 1 && c < nch; ++c) issue(c);
    // this warp's tiles: t = warp % T' ... with k-part kp
    const int tslot = warp % (T * KP >= kNW ? kNW : T * KP);
    const bool wact = warp < T * KP || T >= kNW;
    const int kp = T >= kNW ? 0 : tslot / T;
    double acc[2][2], acc2[2][2];
#pragma unroll
    for (int u = 0; u < 2; ++u) acc[u][0] = acc[u][1] = acc2[u][0] = acc2[u][1] = 0.0;
    double rr = 0.0;
    for (int c = 0; c < nch; ++c) {
        if (tid == 0 && c + kWtD - 1 < nch) issue(c + kWtD - 1);
        const int sl = c % kWtD;
        mbar_wait(&bars[sl], (uint32_t)((c / kWtD) & 1));
        const int64_t i0 = n0 + (int64_t)c * kWtCH;
        const int cnt = (int)(n1 - i0 < (int64_t)kWtCH ? n1 - i0 : (int64_t)kWtCH);
        const double* W = wr + sl * slotW;
        const double* V = vr + sl * slotV;
        // padded copy + ||v||^2: element e (fixed node/query per thread); rows past cnt are 0
        for (int e = tid; e < kWtCH * BP; e += kMT) {
            const int nd = e / BP, q = e - nd * BP;
            const double v = nd < cnt ? V[e] : 0.0;
            rr = fma(v, v, rr);
            vp[nd * LDV + q] = v;
        }
        __syncthreads();
        if (wact) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {      // T <= 32 tiles: at most two per warp
                const int t = T >= kNW ? warp + u * kNW : (u == 0 ? tslot % T : T);
                if (t >= T) continue;
                const int jt = t / NBT, bt = t - jt * NBT;
                for (int ks = kp; ks < kWtCH / 4; ks += 2 * KP) {
                    const int nd = ks * 4 + (lane & 3);           // node of this lane's k
                    const double wa = nd < cnt ? W[nd * ldw + jt * 8 + (lane >> 2)] : 0.0;   // A: basis x node
                    const double vb = vp[nd * LDV + bt * 8 + (lane >> 2)];                    // B: node x query
                    dmma_8x8x4(acc[u][0], acc[u][1], wa, vb);
                    const int ks2 = ks + KP;
                    if (ks2 < kWtCH / 4) {
                        const int nd2 = ks2 * 4 + (lane & 3);
                        const double wa2 = nd2 < cnt ? W[nd2 * ldw + jt * 8 + (lane >> 2)] : 0.0;
                        const double vb2 = vp[nd2 * LDV + bt * 8 + (lane >> 2)];
                        dmma_8x8x4(acc2[u][0], acc2[u][1], wa2, vb2);
                    }
                }
            }
        }
        __syncthreads();   // slot sl is reissued kWtD - 1 chunks later; vp is rewritten
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {          // the two chains, fixed order
        acc[u][0] += acc2[u][0];
        acc[u][1] += acc2[u][1];
    }
    // ---- fixed-order combine: k-parts of each tile, then partial columns -----
    const int rows = npad + 1;
    if (T >= kNW) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int t = warp + u * kNW;
            if (t >= T) continue;
            const int jt = t / NBT, bt = t - jt * NBT;
            const int j = jt * 8 + (lane >> 2), bb = bt * 8 + 2 * (lane & 3);
            a.part[((int64_t)bb * rows + j) * a.nct + a.col0 + blockIdx.x] = acc[u][0];
            a.part[((int64_t)(bb + 1) * rows + j) * a.nct + a.col0 + blockIdx.x] = acc[u][1];
        }
    } else {
        if (wact) {
            s_red[warp * 64 + 2 * lane] = acc[0][0];
            s_red[warp * 64 + 2 * lane + 1] = acc[0][1];
        }
        __syncthreads();
        for (int idx = tid; idx < T * 64; idx += kMT) {
            const int t = idx >> 6, w = idx & 63;
            double s = 0.0;
            for (int k = 0; k < KP; ++k) s += s_red[(k * T + t) * 64 + w];
            const int ln = w >> 1, h = w & 1;
            const int jt = t / NBT, bt = t - jt * NBT;
            const int j = jt * 8 + (ln >> 2), bb = bt * 8 + 2 * (ln & 3) + h;
            a.part[((int64_t)bb * rows + j) * a.nct + a.col0 + blockIdx.x] = s;
        }
    }
    s_rr[tid] = rr;
    __syncthreads();
    if (tid < BP) {
        double v = 0.0;
        for (int u = tid; u < kMT; u += BP) v += s_rr[u];
        a.part[((int64_t)tid * rows + npad) * a.nct + a.col0 + blockIdx.x] = v;
    }
}
}  // namespace rbs
