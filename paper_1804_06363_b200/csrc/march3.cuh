// march3.cuh -- K3 (prolongation + smoother) for 2D grids, v3: register windows.
//
// Same lagged row march and the same arithmetic as k_smooth2 (march2.cuh), a
// different division of labour that moves the smoother's vertical stencil
// reuse from shared memory into registers:
//
//  * 512 threads = 16 column pairs x 32 queries: warp w owns window columns
//    2w, 2w+1 (lane = query) and keeps both columns of the rows Jb-(2S+1) ..
//    Jb-1 in registers.  A red-black half-sweep updates exactly one column of
//    every pair per row, so a pair does S updates per step; the vertical
//    neighbours and the pair's other column come from registers, only the far
//    x-neighbour from the shared y ring (where every update is also published).
//    Per update: 3 shared loads (x-neighbour, rhs, h^2/(4 theta)) + 1 store,
//    against 6 + 1 in k_smooth2.
//  * the same 16 warps run the prolongation y0 = W e (eq7) of the arriving row
//    as one 8x8 DMMA tile each (4 column tiles x 4 query tiles); the E fragments
//    of the warp's query tile stay in registers for the whole pass, so a DMMA
//    needs one W fragment load.  The y ring rows are padded to 40 doubles per
//    column so the tiles' 16-byte fragment stores are conflict-free.
//  * the output row (lag 2S+1) is stored from registers.
//
// Window = 32 columns (S-column halo each side), strip TX = 32 - 2S.  One
// barrier per row; the red-black order is exact by the same lag argument as
// k_smooth2 (half-sweep s on row Jb - 2(s+1), the rows a step reads and writes
// are disjoint), and the per-node formulas are k_smooth2's, so the result is
// bitwise identical to k_smooth2 (tests/test_gpu_parity.py).
//
//   k_smooth3   prolongation + smoother (+ y^T r, RBCG Step 10)
#pragma once
#include <type_traits>

#include "march2.cuh"

namespace rbs {

constexpr int kS3TW = 32;           // window columns (16 pairs)
constexpr int kS3YR = 8;            // y ring rows (lags 0..7)
constexpr int kS3RR = 8;            // rhs ring rows (issued at lag 0, last read at lag 2S+1)
constexpr int kS3WR = 3;            // W (+ x_old) ring rows: prefetch distance 2
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

// S: half-sweeps (1..3); HAS_RHS: smoother rhs rows (RBCG: r) else a.rconst;
// ACC: y0 = x_old + W e (RBI Step 6-7); NKC: npad / 4 (k-steps of the prolongation)
template <int S, bool HAS_RHS, bool ACC, int NKC>
__global__ void __launch_bounds__(kMT, 1) k_smooth3(SmoothMarchArgs a) {
    constexpr int BP = 32, TW = kS3TW, TX = TW - 2 * S, YS = kS3YS;
    constexpr int WR = kS3WR, D = WR - 1;
    constexpr int LO = 2 * S + 1;                 // lag of the output row
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
    const int ncopy = Imax - Imin + 1, coff = Imin - xlo;
    const int cmin = Imin - xlo, cmax = Imax - xlo;          // valid window columns
    const int Jfirst = y0 - S;                               // row of step 0
    const int JlastP = y1 - 1 + S;                           // last prolongated row
    const int nsteps = (y1 - y0) + 3 * S + 1;
    const Smooth3Smem L(ldw, a.g.Q, HAS_RHS, ACC);
    // ring bases are compile-time constants (the same values as Smooth3Smem)
    constexpr int VY = kS3TW * kS3YS, VR = kS3TW * 32, RO = kS3YR * VY;
    constexpr int XO = RO + (HAS_RHS ? kS3RR * VR : 0), WO = XO + (ACC ? kS3WR * VR : 0);
    const int THO = L.tho, CHO = L.cho, WROW = L.wrow;

    // ---- init: zero the rings (Dirichlet columns / rows stay zero), tables --------
    for (int t = tid; t < THO; t += kMT) smd[t] = 0.0;
    for (int t = tid; t < a.g.Q * BP; t += kMT) {
        const double v = a.theta[t];
        smd[THO + t] = v;
        smd[CHO + t] = a.g.h2 / (4.0 * v);
    }
    fill_colinfo(a.g, xlo, TW, s_ci, s_cu);
    if (tid == 0) {
        for (int k = 0; k < WR; ++k) mbar_init(&wbar[k], 1);
        for (int k = 0; k < kS3RR; ++k) mbar_init(&rbar[k], 1);
        mbar_fence_init();
    }
    // E fragments of this warp's query tile (B operand: E[k][query]) for the whole pass
    const int ct = warp >> 2, bt = warp & 3;
    double ef[NKC];
#pragma unroll
    for (int k = 0; k < NKC; ++k) ef[k] = a.E[(4 * k + (lane & 3)) * BP + bt * 8 + (lane >> 2)];
    __syncthreads();

    const uint32_t wb = (uint32_t)ncopy * ldw * 8;
    const uint32_t vb = (uint32_t)ncopy * BP * 8;
    auto issue_w = [&](int u) {          // W (+ x_old) of row Jfirst + u (thread 0)
        const int J = Jfirst + u;
        const bool in = J >= 1 && J <= m;
        const int ws = u % WR;
        uint64_t* bar = &wbar[ws];
        fence_async_smem();
        mbar_expect_tx(bar, in ? wb + (ACC ? vb : 0u) : 0u);
        if (!in) return;
        const int64_t n0 = (int64_t)(J - 1) * m + (Imin - 1);
        bulk_g2s(smd + WO + ws * WROW + coff * ldw, a.W + n0 * ldw, wb, bar);
        if (ACC) bulk_g2s(smd + XO + ws * VR + coff * BP, a.Xold + n0 * BP, vb, bar);
    };
    auto issue_r = [&](int u) {          // smoother rhs row Jfirst + u (thread 0)
        const int J = Jfirst + u;
        const bool in = J >= 1 && J <= m;
        const int rs = u & (kS3RR - 1);
        uint64_t* bar = &rbar[rs];
        fence_async_smem();
        mbar_expect_tx(bar, in ? vb : 0u);
        if (!in) return;
        const int64_t n0 = (int64_t)(J - 1) * m + (Imin - 1);
        bulk_g2s(smd + RO + rs * VR + coff * BP, a.Rhs + n0 * BP, vb, bar);
    };
    if (tid == 0)
        for (int u = 0; u < D && Jfirst + u <= JlastP; ++u) issue_w(u);

    // ---- this thread: column pair (cA, cB) = (2 warp, 2 warp + 1), query b = lane ----
    const int b = lane;
    const int cA = 2 * warp, cB = cA + 1;
    const bool qact = a.active[b] != 0;
    const double rconst = a.rconst;
    const int cuA = s_cu[cA], cuB = s_cu[cB], ciA = s_ci[cA], ciB = s_ci[cB];
    // half-sweep s: rows of the dependency cone, and whether each column of the pair is
    // in its valid column range (the S - s halo columns shrink by one per half-sweep)
    int rlos[S], rhis[S];
    bool okA[S], okB[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int c0 = max(s + 1, cmin), c1 = min(TW - 2 - s, cmax);
        const int hw = S - 1 - s;
        rlos[s] = max(1, y0 - hw);
        rhis[s] = min(m, y1 - 1 + hw);
        okA[s] = qact && cA >= c0 && cA <= c1;
        okB[s] = qact && cB >= c0 && cB <= c1;
    }
    // Roles instead of columns: at step t half-sweeps 0, 2 update the pair's column P and
    // half-sweep 1 its column Q, where P = A iff q0 + t is even (consecutive half-sweeps
    // alternate colours: color_seq drops repeats; node I = xlo + c on row R = Jb - 2(s+1)
    // has the sweep's colour iff I + R - seq[s] is even).  P and Q swap every step, and
    // the window shift moves each register to the other role, so every register index is
    // a constant.  The stencil sum 0.25 ((n_l + n_r) + (n_d + n_u)) needs no side (IEEE
    // addition commutes); only the interface path needs left / right.
    const int q0 = (a.seq[0] - xlo - Jfirst) & 1;
    // window: row Jb - L of column P / Q in yP/yQ[L], L = 1 .. LO
    double yP[LO + 1], yQ[LO + 1];
    int cbr[2 * S];                // y-block (x px) of cell rows Jb-2, Jb-3, .., Jb-1-2S
#pragma unroll
    for (int k = 0; k <= LO; ++k) yP[k] = yQ[k] = 0.0;
#pragma unroll
    for (int k = 0; k < 2 * S; ++k) cbr[k] = 0;
    double yr = 0.0, yy = 0.0;
    double* yg = a.Y + ((int64_t)(Jfirst - LO - 1) * m + (xlo - 1)) * BP + b;
    const int wofs = WO + (ct * 8 + (lane >> 2)) * ldw + (lane & 3);            // A fragment (W)
    const int tofs = (ct * 8 + (lane >> 2)) * YS + bt * 8 + 2 * (lane & 3);      // D fragment (y0)
    const int xofs = XO + (ct * 8 + (lane >> 2)) * BP + bt * 8 + 2 * (lane & 3); // x_old fragment
    // per-role data, swapped every step: own y-ring offset, far x-neighbour offset, rhs
    // ring offset, column block info, output column (or -1), "P is the left column"
    const int oA = cA * YS + b, oB = cB * YS + b;
    const int fA = (cA - 1) * YS + b, fB = (cB + 1) * YS + b;
    const int rA = RO + cA * BP + b, rB = RO + cB * BP + b;
    const bool ownA = cA >= S && cA < S + TX && cA <= cmax;
    const bool ownB = cB >= S && cB < S + TX && cB <= cmax;
    const bool pa0 = q0 == 0;     // step 0: P = A
    int oP = pa0 ? oA : oB, oQ = pa0 ? oB : oA, fP = pa0 ? fA : fB, fQ = pa0 ? fB : fA;
    int rP = pa0 ? rA : rB, rQ = pa0 ? rB : rA;
    int cuP = pa0 ? cuA : cuB, cuQ = pa0 ? cuB : cuA, ciP = pa0 ? ciA : ciB, ciQ = pa0 ? ciB : ciA;
    int gP = pa0 ? (ownA ? cA : -1) : (ownB ? cB : -1), gQ = pa0 ? (ownB ? cB : -1) : (ownA ? cA : -1);
    bool pleft = pa0;
    // validity of each role's column per half-sweep (s even: P, s odd: Q)
    bool okP[S], okQ[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        okP[s] = pa0 ? okA[s] : okB[s];
        okQ[s] = pa0 ? okB[s] : okA[s];
    }
    const int chb = CHO + b;
    const bool issW = tid == 0, issR = tid == 32;
    const bool tfirst = warp < 8;
    const uint32_t wbar0 = smem_u32(&wbar[0]), rbar0 = smem_u32(&rbar[0]);
    int ws = 0, wph = 0;           // W ring slot / phase of row Jb

    for (int t = 0; t < nsteps; ++t) {
        const int Jb = Jfirst + t;
        const int sl = t & 7;
        if (issW && Jb + D <= JlastP) issue_w(t + D);
        if (HAS_RHS && issR && Jb <= JlastP) issue_r(t);
        // ---- roles swap: window shift moves P <-> Q; row Jb - 1 (formed last step) enters ----
        if (t > 0) {
#pragma unroll
            for (int k = LO; k >= 2; --k) {
                const double tp = yP[k - 1];
                yP[k] = yQ[k - 1];
                yQ[k] = tp;
            }
            int ti;
            ti = oP; oP = oQ; oQ = ti;
            ti = fP; fP = fQ; fQ = ti;
            ti = rP; rP = rQ; rQ = ti;
            ti = cuP; cuP = cuQ; cuQ = ti;
            ti = ciP; ciP = ciQ; ciQ = ti;
            ti = gP; gP = gQ; gQ = ti;
            pleft = !pleft;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const bool tb = okP[s];
                okP[s] = okQ[s];
                okQ[s] = tb;
            }
        }
        {
            const int y1o = ((sl - 1) & 7) * VY;
            yP[1] = smd[y1o + oP];
            yQ[1] = smd[y1o + oQ];
        }
#pragma unroll
        for (int k = 2 * S - 1; k >= 1; --k) cbr[k] = cbr[k - 1];
        cbr[0] = axis_block(a.g, min(max(Jb - 2, 0), m), a.g.py) * a.g.px;

        // the two halves of a step are independent (the sweeps read rows formed in
        // earlier steps only): half of the warps (two per SM sub-partition) prolongate
        // first, the others sweep first, so the DMMA pipe and the sweeps overlap
#define RBS_S3_TENSOR                                                                         \
        if (Jb <= JlastP) {  /* prolongation of row Jb (lag 0): one DMMA tile per warp */     \
            mbar_wait_u32(wbar0 + 8u * ws, (uint32_t)wph);                                   \
            double d0 = 0.0, d1 = 0.0;                                                        \
            if (Jb >= 1 && Jb <= m) {                                                         \
                if (a.has_e && !(a.dbg & 1)) {                                                \
                    const double* wr = smd + ws * WROW + wofs;                                \
                    _Pragma("unroll") for (int k = 0; k < NKC; ++k)                            \
                        dmma_8x8x4(d0, d1, wr[4 * k], ef[k]);                                 \
                }                                                                             \
                if (ACC) {                                                                    \
                    d0 += smd[ws * VR + xofs];                                                \
                    d1 += smd[ws * VR + xofs + 1];                                            \
                }                                                                             \
            }                                                                                 \
            *reinterpret_cast<double2*>(smd + sl * VY + tofs) = make_double2(d0, d1);         \
        }
        if (tfirst) { RBS_S3_TENSOR }
        // ---- half-sweeps: s on row R = Jb - 2(s+1), role P (s even) / Q (s odd) --------
        if (HAS_RHS && t >= 2 && Jb - 2 <= JlastP)
            mbar_wait_u32(rbar0 + 8u * ((sl - 2) & 7), (uint32_t)(((t - 2) >> 3) & 1));
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (a.dbg & 2) break;
            const int Ls = 2 * (s + 1);
            const int R = Jb - Ls;
            const bool isP = (s & 1) == 0;                   // compile time
            if (!(isP ? okP[s] : okQ[s]) || R < rlos[s] || R > rhis[s]) continue;
            const int SL = (sl - Ls) & 7;
            const int yrow = SL * VY;
            const double far = smd[yrow + (isP ? fP : fQ)];
            const double own = isP ? yQ[Ls] : yP[Ls];       // the pair's other column, row R
            const double nd = isP ? yP[Ls + 1] : yQ[Ls + 1]; // row R - 1
            const double nu = isP ? yP[Ls - 1] : yQ[Ls - 1]; // row R + 1
            const double rh = HAS_RHS ? smd[SL * VR + (isP ? rP : rQ)] : rconst;
            const int by0 = cbr[2 * s + 1], by1 = cbr[2 * s];
            const int cu = isP ? cuP : cuQ;
            double v;
            if (by0 == by1 && cu >= 0) {
                v = fma(smd[chb + (cu + by0) * BP], rh, 0.25 * ((far + own) + (nd + nu)));
            } else {
                const bool left = isP ? pleft : !pleft;      // the updated column is the pair's left
                v = gs_iface(a.g, smd + THO, b, isP ? ciP : ciQ, by0, by1, rh, left ? far : own,
                             left ? own : far, nd, nu);
            }
            smd[yrow + (isP ? oP : oQ)] = v;
            if (isP) yP[Ls] = v;
            else yQ[Ls] = v;
        }
        // ---- output row Ro = Jb - (2S+1): stores (+ y^T r, y^T y) from registers -----
        const int Ro = Jb - LO;
        if (Ro >= y0 && Ro < y1 && !(a.dbg & 4)) {
            const int so = ((sl - LO) & 7) * VR;
            if (gP >= 0) {
                const double v = yP[LO];
                yg[(int64_t)gP * BP] = v;
                if (a.last) {
                    const double rv = HAS_RHS ? smd[so + rP] : rconst;
                    yr = fma(v, rv, yr);
                    yy = fma(v, v, yy);
                }
            }
            if (gQ >= 0) {
                const double v = yQ[LO];
                yg[(int64_t)gQ * BP] = v;
                if (a.last) {
                    const double rv = HAS_RHS ? smd[so + rQ] : rconst;
                    yr = fma(v, rv, yr);
                    yy = fma(v, v, yy);
                }
            }
        }
        if (!tfirst) { RBS_S3_TENSOR }
#undef RBS_S3_TENSOR
        ws = ws + 1 == WR ? 0 : ws + 1;
        wph ^= ws == 0 ? 1 : 0;
        yg += (int64_t)m * BP;
        __syncthreads();
    }
    if (!a.last) return;
    // ---- partials and RBCG Step 10 in the last CTA (rings are dead) ----------------
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

}  // namespace rbs
