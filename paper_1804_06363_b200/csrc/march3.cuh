// march3.cuh -- K3 (prolongation + smoother) for 2D grids, v3: register windows.
//
// Same lagged row march and the same per-node arithmetic as k_smooth2
// (march2.cuh), a different division of labour built to minimise the
// instructions of a row step (ncu: the row march is issue-bound, and every
// instruction per warp-step costs ~0.17 us at c2):
//
//  * 512 threads = 16 column pairs x 32 queries: warp w owns window columns
//    2w, 2w+1 (lane = query) and keeps both columns of the last 8 rows in
//    registers.  A red-black half-sweep updates exactly one column of every
//    pair per row, so a pair does S updates per step; the vertical neighbours
//    and the pair's other column come from registers, only the far
//    x-neighbour from the shared y ring, where every update is also published.
//  * the same 16 warps run the prolongation y0 = W e (eq7) of the arriving row,
//    one 8x8 DMMA tile each (4 column tiles x 4 query tiles); the E fragments of
//    the warp's query tile stay in registers for the whole pass.  Half of the
//    warps (two per SM sub-partition) prolongate before their sweeps, the others
//    after, so the DMMA pipe overlaps the sweeps.  The y ring rows are padded to
//    40 doubles per column so the tiles' 16-byte stores are conflict-free.
//  * the step loop is unrolled by 8 (the ring length): every ring slot, window
//    register, barrier slot and phase is a compile-time constant.  The colour
//    parity is constant too: the partition keeps every strip origin and segment
//    origin at the same parity, so a symmetric sweep starting red updates column
//    A in half-sweep s of step t iff s + t is even.
//  * the output row (lag 2S+1) is stored from registers.
//
// Window = 32 columns (S-column halo each side), strip TX = 32 - 2S, row
// segments of even length.  One barrier per row; the red-black order is exact by
// k_smooth2's lag argument (half-sweep s on row Jb - 2(s+1); the rows a step
// reads and writes are disjoint).
//
//   k_smooth3   prolongation + smoother (+ y^T r, RBCG Step 10)
#pragma once
#include "march2.cuh"

namespace rbs {

constexpr int kS3TW = 32;           // window columns (16 pairs)
constexpr int kS3YR = 8;            // y ring rows (lags 0..7)
constexpr int kS3RR = 8;            // rhs ring rows (issued at lag 0, last read at lag 2S+1)
constexpr int kS3WR = 4;            // W (+ x_old) ring rows: prefetch distance 3
constexpr int kS3YS = 32 + 8;       // y ring column stride (doubles): conflict-free tile stores

// dynamic shared memory (doubles): y ring | rhs ring | x_old ring | W ring | theta | h^2/(4 theta)
struct Smooth3Smem {
    int vy, vr, ro, xo, wo, wrow, tho, cho;
    size_t total;
    __host__ __device__ Smooth3Smem(int ldw, int Q, bool has_rhs, bool acc) {
        vy = kS3TW * kS3YS;
        vr = kS3TW * 32;
        ro = kS3YR * vy;
        xo = ro + (has_rhs ? kS3RR * vr : 0);
        wo = xo + (acc ? kS3WR * vr : 0);
        wrow = kS3TW * ldw;
        tho = wo + kS3WR * wrow;
        cho = tho + Q * 32;
        total = (size_t)(cho + Q * 32) * 8;
    }
};

// Gauss-Seidel value of a block-interface node (cells of more than one block): the
// general cell-averaged coefficients, out of line (rare; keeps the unrolled steps small)
__device__ __noinline__ double gs_iface(const Geo& g, const double* th, int b, int ci, int by0, int by1,
                                        double rh, double nl, double nr, double nd, double nu) {
    double kap[4], nb[4] = {nl, nr, nd, nu};
    kappa2_blocks(th, 32, b, ci & 0xff, ci >> 8, by0, by1, kap);
    return gs_value<2>(g, kap, rh, nb);
}

// per-thread state of the march (registers after inlining: every array index is constant)
template <int S, int NKC>
struct S3State {
    double yA[8], yB[8];   // window: row with ring slot k of column A / B
    int cb[8];             // y-block * px of the cell row with ring slot k
    double ef[NKC];        // E fragments (B operand of the prolongation)
    double yr, yy;         // y^T r, y^T y partials
    double* yg;            // output pointer of the current output row (column 0, lane b)
    // per-thread constants
    int oA, oB, fA, fB, rA, rB, chA, chB, ciA, ciB, gA, gB;
    bool uA, uB;           // column's cells in one x-block (the uniform fast path)
    bool okA[S], okB[S];   // column valid for half-sweep s (and the query active)
    int tlo[S], thi[S];    // steps at which half-sweep s has a valid row
    int tolo, tohi;        // steps with an output row
    int tphi, tdlo, tdhi;  // steps with a prolongated row / with a row inside 1..m
    int wofs, tofs, xofs, WROW, THO;
    int Jfirst, JlastP, m, Imin, coff, ncopy;
    uint32_t wbar0, rbar0;
    bool issW, issR, tfirst, last;
};

// TMA row copies (one thread): W (+ x_old) of row J into W-ring slot ws; rhs row J into
// rhs-ring slot rs
template <bool ACC>
__device__ __forceinline__ void s3_issue_w(const SmoothMarchArgs& a, double* smd, int WO, int XO, int WROW,
                                           int J, int m, int Imin, int coff, int ncopy, int ws,
                                           uint64_t* wbar) {
    const bool in = J >= 1 && J <= m;
    const uint32_t wb = (uint32_t)ncopy * a.ldw * 8, vb = (uint32_t)ncopy * 32 * 8;
    uint64_t* bar = wbar + ws;
    fence_async_smem();
    mbar_expect_tx(bar, in ? wb + (ACC ? vb : 0u) : 0u);
    if (!in) return;
    const int64_t n0 = (int64_t)(J - 1) * m + (Imin - 1);
    bulk_g2s(smd + WO + ws * WROW + coff * a.ldw, a.W + n0 * a.ldw, wb, bar);
    if (ACC) bulk_g2s(smd + XO + ws * kS3TW * 32 + coff * 32, a.Xold + n0 * 32, vb, bar);
}
__device__ __forceinline__ void s3_issue_r(const SmoothMarchArgs& a, double* smd, int RO, int J, int m,
                                           int Imin, int coff, int ncopy, int rs, uint64_t* rbar) {
    const bool in = J >= 1 && J <= m;
    const uint32_t vb = (uint32_t)ncopy * 32 * 8;
    uint64_t* bar = rbar + rs;
    fence_async_smem();
    mbar_expect_tx(bar, in ? vb : 0u);
    if (!in) return;
    const int64_t n0 = (int64_t)(J - 1) * m + (Imin - 1);
    bulk_g2s(smd + RO + rs * kS3TW * 32 + coff * 32, a.Rhs + n0 * 32, vb, bar);
}

// one row step t = t0 + ROT (t0 a multiple of 8)
template <int S, bool HAS_RHS, bool ACC, int NKC, int ROT>
__device__ __forceinline__ void s3_step(S3State<S, NKC>& st, const SmoothMarchArgs& a, double* smd,
                                        uint64_t* wbar, uint64_t* rbar, int t0) {
    constexpr int LO = 2 * S + 1;
    constexpr int VY = kS3TW * kS3YS, VR = kS3TW * 32, RO = kS3YR * VY;
    constexpr int XO = RO + (HAS_RHS ? kS3RR * VR : 0), WO = XO + (ACC ? kS3WR * VR : 0);
    constexpr int WR = kS3WR, D = WR - 1;
    constexpr int WS = ROT & (WR - 1);            // W ring slot of this step's row (WR | 8)
    constexpr int WPH = (ROT / WR) & 1;           // its phase (t0 / WR is even)
    const int t = t0 + ROT;
    const int Jb = st.Jfirst + t;
    // ---- TMA: W (+ x_old) of row Jb + D, rhs row Jb --------------------------------------
    if (st.issW && Jb + D <= st.JlastP)
        s3_issue_w<ACC>(a, smd, WO, XO, st.WROW, Jb + D, st.m, st.Imin, st.coff, st.ncopy, (ROT + D) & (WR - 1),
                        wbar);
    if (HAS_RHS && st.issR && Jb <= st.JlastP)
        s3_issue_r(a, smd, RO, Jb, st.m, st.Imin, st.coff, st.ncopy, ROT, rbar);
    // ---- row Jb - 1 (formed last step) enters the window; block of cell row Jb - 2 -------
    constexpr int S1 = (ROT - 1) & 7, S2 = (ROT - 2) & 7;
    st.yA[S1] = smd[S1 * VY + st.oA];
    st.yB[S1] = smd[S1 * VY + st.oB];
    st.cb[S2] = axis_block(a.g, min(max(Jb - 2, 0), st.m), a.g.py) * a.g.px;

#define RBS_S3_TENSOR                                                                           \
    if (t <= st.tphi) { /* prolongation of row Jb (lag 0): one DMMA tile per warp */           \
        double d0 = 0.0, d1 = 0.0;                                                              \
        if (t >= st.tdlo && t <= st.tdhi) {                                                     \
            if (a.has_e) {                                                                      \
                const double* wr = smd + WS * st.WROW + st.wofs;                                \
                _Pragma("unroll") for (int k = 0; k < NKC; ++k) dmma_8x8x4(d0, d1, wr[4 * k], st.ef[k]); \
            }                                                                                   \
            if (ACC) {                                                                          \
                d0 += smd[WS * VR + st.xofs];                                                   \
                d1 += smd[WS * VR + st.xofs + 1];                                               \
            }                                                                                   \
        }                                                                                       \
        *reinterpret_cast<double2*>(smd + ROT * VY + st.tofs) = make_double2(d0, d1);           \
    }
    if (st.tfirst) { RBS_S3_TENSOR }
    // ---- half-sweeps: s on row R = Jb - 2(s+1); column A iff s + ROT is even ------------
    // all shared loads of the three updates first (independent rows), then the values,
    // then the stores: one load latency per step instead of one per half-sweep
    bool go[S];
    double far[S], rh[S], ch[S];
    int by0[S], by1[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int SL = (ROT - 2 * (s + 1)) & 7;        // ring slot / window index of row R
        const bool upA = ((s + ROT) & 1) == 0;        // compile time
        go[s] = (upA ? st.okA[s] : st.okB[s]) && t >= st.tlo[s] && t <= st.thi[s];
        by0[s] = st.cb[(SL - 1) & 7];
        by1[s] = st.cb[SL];
        far[s] = rh[s] = ch[s] = 0.0;
        if (go[s]) {
            far[s] = smd[SL * VY + (upA ? st.fA : st.fB)];
            rh[s] = HAS_RHS ? smd[SL * VR + (upA ? st.rA : st.rB)] : a.rconst;
            ch[s] = smd[(upA ? st.chA : st.chB) + by0[s] * 32];
        }
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
        if (!go[s]) continue;
        const int SL = (ROT - 2 * (s + 1)) & 7;
        const bool upA = ((s + ROT) & 1) == 0;
        const double own = upA ? st.yB[SL] : st.yA[SL];        // the pair's other column, row R
        const double nd = upA ? st.yA[(SL - 1) & 7] : st.yB[(SL - 1) & 7];   // row R - 1
        const double nu = upA ? st.yA[(SL + 1) & 7] : st.yB[(SL + 1) & 7];   // row R + 1
        double v;
        if (by0[s] == by1[s] && (upA ? st.uA : st.uB)) {
            // k_smooth2's uniform-node formula; the stencil sum commutes, so the far
            // neighbour's side does not matter
            v = fma(ch[s], rh[s], 0.25 * ((far[s] + own) + (nd + nu)));
        } else {
            v = gs_iface(a.g, smd + st.THO, threadIdx.x & 31, upA ? st.ciA : st.ciB, by0[s], by1[s], rh[s],
                         upA ? far[s] : own, upA ? own : far[s], nd, nu);
        }
        smd[SL * VY + (upA ? st.oA : st.oB)] = v;
        if (upA) st.yA[SL] = v;
        else st.yB[SL] = v;
    }
    // ---- output row Ro = Jb - (2S+1): stores (+ y^T r, y^T y) from registers ------------
    if (t >= st.tolo && t <= st.tohi) {
        constexpr int SO = (ROT - LO) & 7;
        if (st.gA >= 0) {
            const double v = st.yA[SO];
            st.yg[(int64_t)st.gA * 32] = v;
            if (st.last) {
                const double rv = HAS_RHS ? smd[SO * VR + st.rA] : a.rconst;
                st.yr = fma(v, rv, st.yr);
                st.yy = fma(v, v, st.yy);
            }
        }
        if (st.gB >= 0) {
            const double v = st.yB[SO];
            st.yg[(int64_t)st.gB * 32] = v;
            if (st.last) {
                const double rv = HAS_RHS ? smd[SO * VR + st.rB] : a.rconst;
                st.yr = fma(v, rv, st.yr);
                st.yy = fma(v, v, st.yy);
            }
        }
    }
    if (!st.tfirst) { RBS_S3_TENSOR }
#undef RBS_S3_TENSOR
    st.yg += (int64_t)st.m * 32;
    // one thread waits for the rows the next step reads (W (+ x_old) of row Jb + 1, rhs of
    // row Jb - 1); the barrier then publishes them to every thread
    if (st.issW) {
        constexpr int WS1 = (ROT + 1) & (WR - 1), WPH1 = ((ROT + 1) / WR) & 1;
        if (t + 1 <= st.tphi) mbar_wait_u32(st.wbar0 + 8u * WS1, (uint32_t)WPH1);
        if (HAS_RHS && t + 1 >= 2 && Jb - 1 <= st.JlastP)
            mbar_wait_u32(st.rbar0 + 8u * ((ROT - 1) & 7), (uint32_t)(((t - 1) >> 3) & 1));
    }
    __syncthreads();
}

// S: half-sweeps (alternating colours starting red); HAS_RHS: smoother rhs rows (RBCG: r)
// else a.rconst; ACC: y0 = x_old + W e (RBI Steps 6-7); NKC: npad / 4
template <int S, bool HAS_RHS, bool ACC, int NKC>
__global__ void __launch_bounds__(kMT, 1) k_smooth3(SmoothMarchArgs a) {
    constexpr int BP = 32, TW = kS3TW, TX = TW - 2 * S, YS = kS3YS;
    constexpr int WR = kS3WR, D = WR - 1;
    constexpr int LO = 2 * S + 1;                 // lag of the output row
    constexpr int VY = kS3TW * kS3YS, VR = kS3TW * 32, RO = kS3YR * VY;
    constexpr int XO = RO + (HAS_RHS ? kS3RR * VR : 0), WO = XO + (ACC ? kS3WR * VR : 0);
    (void)VY;
    if (a.done && ld_flag(a.done)) return;
    extern __shared__ __align__(128) double smd[];
    __shared__ int s_ci[TW], s_cu[TW];
    __shared__ __align__(8) uint64_t wbar[WR], rbar[kS3RR];
    __shared__ double s_yr[kMaxBatch], s_yy[kMaxBatch];
    __shared__ int s_last;
    const int m = a.g.m, ldw = a.ldw;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int sx = blockIdx.x % a.part.nsx, sy = blockIdx.x / a.part.nsx;
    const int x0 = 1 + sx * TX;
    const int y0 = 1 + sy * a.part.rows_per_seg;
    const int y1 = min(m + 1, y0 + a.part.rows_per_seg);   // exclusive
    const int xlo = x0 - S;                                  // node of window column 0
    const int Imin = max(1, xlo), Imax = min(m, x0 + TX - 1 + S);
    const int cmin = Imin - xlo, cmax = Imax - xlo;          // valid window columns
    const int Jfirst = y0 - S;                               // row of step 0
    const int nsteps = (y1 - y0) + 3 * S + 1;
    const Smooth3Smem L(ldw, a.g.Q, HAS_RHS, ACC);

    // ---- init: zero the rings (Dirichlet columns / rows stay zero), tables --------
    for (int t = tid; t < L.tho; t += kMT) smd[t] = 0.0;
    for (int t = tid; t < a.g.Q * BP; t += kMT) {
        const double v = a.theta[t];
        smd[L.tho + t] = v;
        smd[L.cho + t] = a.g.h2 / (4.0 * v);
    }
    fill_colinfo(a.g, xlo, TW, s_ci, s_cu);
    if (tid == 0) {
        for (int k = 0; k < WR; ++k) mbar_init(&wbar[k], 1);
        for (int k = 0; k < kS3RR; ++k) mbar_init(&rbar[k], 1);
        mbar_fence_init();
    }
    S3State<S, NKC> st;
    const int ct = warp >> 2, bt = warp & 3;
#pragma unroll
    for (int k = 0; k < NKC; ++k) st.ef[k] = a.E[(4 * k + (lane & 3)) * BP + bt * 8 + (lane >> 2)];
    __syncthreads();

    st.m = m;
    st.Jfirst = Jfirst;
    st.JlastP = y1 - 1 + S;
    st.Imin = Imin;
    st.coff = Imin - xlo;
    st.ncopy = Imax - Imin + 1;
    st.WROW = L.wrow;
    st.THO = L.tho;
    st.wbar0 = smem_u32(&wbar[0]);
    st.rbar0 = smem_u32(&rbar[0]);
    st.issW = tid == 0;
    st.issR = tid == 32;
    st.tfirst = warp < 8;
    st.last = a.last != 0;
    if (tid == 0) {
        for (int u = 0; u < D && Jfirst + u <= st.JlastP; ++u)
            s3_issue_w<ACC>(a, smd, WO, XO, st.WROW, Jfirst + u, m, Imin, st.coff, st.ncopy, u, wbar);
        mbar_wait_u32(st.wbar0, 0u);   // step 0's row (later steps: the waiter before each barrier)
    }
    __syncthreads();

    // ---- this thread: column pair (cA, cB) = (2 warp, 2 warp + 1), query b = lane ----
    const int b = lane;
    const int cA = 2 * warp, cB = cA + 1;
    const bool qact = a.active[b] != 0;
    const int cuA = s_cu[cA], cuB = s_cu[cB];
    st.ciA = s_ci[cA];
    st.ciB = s_ci[cB];
    st.uA = cuA >= 0;
    st.uB = cuB >= 0;
    st.chA = L.cho + max(cuA, 0) * BP + b;
    st.chB = L.cho + max(cuB, 0) * BP + b;
    st.oA = cA * YS + b;
    st.oB = cB * YS + b;
    st.fA = (cA - 1) * YS + b;
    st.fB = (cB + 1) * YS + b;
    st.rA = RO + cA * BP + b;
    st.rB = RO + cB * BP + b;
    st.gA = (cA >= S && cA < S + TX && cA <= cmax) ? cA : -1;
    st.gB = (cB >= S && cB < S + TX && cB <= cmax) ? cB : -1;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int c0 = max(s + 1, cmin), c1 = min(TW - 2 - s, cmax);
        const int hw = S - 1 - s;
        const int rlo = max(1, y0 - hw), rhi = min(m, y1 - 1 + hw);
        st.tlo[s] = rlo + 2 * (s + 1) - Jfirst;
        st.thi[s] = rhi + 2 * (s + 1) - Jfirst;
        st.okA[s] = qact && cA >= c0 && cA <= c1;
        st.okB[s] = qact && cB >= c0 && cB <= c1;
    }
    st.tolo = y0 + LO - Jfirst;
    st.tohi = y1 - 1 + LO - Jfirst;
    st.tphi = st.JlastP - Jfirst;
    st.tdlo = 1 - Jfirst;
    st.tdhi = m - Jfirst;
    st.wofs = WO + (ct * 8 + (lane >> 2)) * ldw + (lane & 3);
    st.tofs = (ct * 8 + (lane >> 2)) * YS + bt * 8 + 2 * (lane & 3);
    st.xofs = XO + (ct * 8 + (lane >> 2)) * BP + bt * 8 + 2 * (lane & 3);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        st.yA[k] = st.yB[k] = 0.0;
        st.cb[k] = 0;
    }
    st.yr = st.yy = 0.0;
    st.yg = a.Y + ((int64_t)(Jfirst - LO - 1) * m + (xlo - 1)) * BP + b;

    // steps padded to a multiple of 8: the extra steps are past every row range (no
    // copies, sweeps or stores), only their barriers run
    for (int t0 = 0; t0 < nsteps; t0 += 8) {
        s3_step<S, HAS_RHS, ACC, NKC, 0>(st, a, smd, wbar, rbar, t0);
        s3_step<S, HAS_RHS, ACC, NKC, 1>(st, a, smd, wbar, rbar, t0);
        s3_step<S, HAS_RHS, ACC, NKC, 2>(st, a, smd, wbar, rbar, t0);
        s3_step<S, HAS_RHS, ACC, NKC, 3>(st, a, smd, wbar, rbar, t0);
        s3_step<S, HAS_RHS, ACC, NKC, 4>(st, a, smd, wbar, rbar, t0);
        s3_step<S, HAS_RHS, ACC, NKC, 5>(st, a, smd, wbar, rbar, t0);
        s3_step<S, HAS_RHS, ACC, NKC, 6>(st, a, smd, wbar, rbar, t0);
        s3_step<S, HAS_RHS, ACC, NKC, 7>(st, a, smd, wbar, rbar, t0);
    }
    if (!a.last) return;
    // ---- partials and RBCG Step 10 in the last CTA (rings are dead) ----------------
    double* s_a = smd;
    double* s_b = smd + kMT;
    SolveState& s = a.s;
    s_a[tid] = st.yr;
    s_b[tid] = st.yy;
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

}  // namespace rbs
