/*
 * oracle.c -- plain CPU fp64 oracle (TEST INFRASTRUCTURE ONLY; see oracle.h).
 *
 * Every function follows the paper step by step,
 * in its order and notation, with the readings listed in DESIGN.md ("Readings
 * of the paper", AMB-1..AMB-21).  No blocking, fusion or reordering.
 * Built with -O2 -ffp-contract=off (every operation rounded, AMB-21).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Grid and affine operator: PAPER.md:98-103 (eq12) with DESIGN.md AMB-1..4. */
/* ------------------------------------------------------------------------ */

/* block index of cell a along an axis with p blocks: the cell centre
 * (a + 1/2) h lies in block floor((a + 1/2) h p)  (AMB-2, exact in integers). */
static int axis_block(int64_t a, int64_t m, int p)
{
    return (int)(((2 * a + 1) * (int64_t)p) / (2 * (m + 1)));
}

/* theta of cell (a,b,c) */
static double cell_theta(int dim, int64_t m, const int* blocks, const double* theta,
                         int64_t a, int64_t b, int64_t c)
{
    int q = axis_block(a, m, blocks[0]) + blocks[0] * axis_block(b, m, blocks[1]);
    if (dim == 3) q += blocks[0] * blocks[1] * axis_block(c, m, blocks[2]);
    return theta[q];
}

/* General affine operator (NEXT(4), DESIGN.md AMB-23): face coefficients
 * kappa_e(theta) = sum_q theta_q F_q[e] given per face (or_set_faces), selected
 * by blocks[0] == 0.  faces[(q*dim + d)*nf + idx], nf = (m+1) m^(dim-1) faces per
 * direction; the face between nodes a and a+1 along d (a = 0..m; 0 and m+1 are
 * Dirichlet nodes) has idx  x: a + (m+1)((J-1) + m(K-1)),  y: (I-1) + m(a + (m+1)(K-1)),
 * z: (I-1) + m((J-1) + m a). */
static int g_face_Q = 0;
static const double* g_faces = NULL;

void or_set_faces(int Q, const double* faces)
{
    g_face_Q = Q;
    g_faces = faces;
}

static double face_kappa(int dim, int64_t m, const double* theta, int d, int64_t a, int64_t I,
                         int64_t J, int64_t K)
{
    int64_t nf = (m + 1) * (dim == 3 ? m * m : m);
    int64_t idx;
    if (d == 0) idx = a + (m + 1) * ((J - 1) + m * (K - 1));
    else if (d == 1) idx = (I - 1) + m * (a + (m + 1) * (K - 1));
    else idx = (I - 1) + m * ((J - 1) + m * a);
    double s = 0.0;
    for (int q = 0; q < g_face_Q; ++q) s += theta[q] * g_faces[((int64_t)q * dim + d) * nf + idx];
    return s;
}

/* Edge coefficients of node (I,J,K) in neighbour order -x,+x,-y,+y(,-z,+z).
 * Each is the mean of the cells sharing the edge (AMB-1), summed in the order
 * of AMB-4 -- or, for a face operator, the face coefficients above. */
static void node_kappa(int dim, int64_t m, const int* blocks, const double* theta,
                       int64_t I, int64_t J, int64_t K, double* k)
{
    if (blocks[0] == 0) {
        int64_t Kk = dim == 3 ? K : 1;
        k[0] = face_kappa(dim, m, theta, 0, I - 1, I, J, Kk);
        k[1] = face_kappa(dim, m, theta, 0, I, I, J, Kk);
        k[2] = face_kappa(dim, m, theta, 1, J - 1, I, J, Kk);
        k[3] = face_kappa(dim, m, theta, 1, J, I, J, Kk);
        if (dim == 3) {
            k[4] = face_kappa(dim, m, theta, 2, K - 1, I, J, K);
            k[5] = face_kappa(dim, m, theta, 2, K, I, J, K);
        }
        return;
    }
    if (dim == 2) {
        double c00 = cell_theta(2, m, blocks, theta, I - 1, J - 1, 0);
        double c10 = cell_theta(2, m, blocks, theta, I, J - 1, 0);
        double c01 = cell_theta(2, m, blocks, theta, I - 1, J, 0);
        double c11 = cell_theta(2, m, blocks, theta, I, J, 0);
        k[0] = 0.5 * (c00 + c01);
        k[1] = 0.5 * (c10 + c11);
        k[2] = 0.5 * (c00 + c10);
        k[3] = 0.5 * (c01 + c11);
    } else {
        double c[2][2][2];
        for (int dz = 0; dz < 2; ++dz)
            for (int dy = 0; dy < 2; ++dy)
                for (int dx = 0; dx < 2; ++dx)
                    c[dx][dy][dz] = cell_theta(3, m, blocks, theta, I - 1 + dx, J - 1 + dy, K - 1 + dz);
        k[0] = 0.25 * ((c[0][0][0] + c[0][1][0]) + (c[0][0][1] + c[0][1][1]));
        k[1] = 0.25 * ((c[1][0][0] + c[1][1][0]) + (c[1][0][1] + c[1][1][1]));
        k[2] = 0.25 * ((c[0][0][0] + c[1][0][0]) + (c[0][0][1] + c[1][0][1]));
        k[3] = 0.25 * ((c[0][1][0] + c[1][1][0]) + (c[0][1][1] + c[1][1][1]));
        k[4] = 0.25 * ((c[0][0][0] + c[1][0][0]) + (c[0][1][0] + c[1][1][0]));
        k[5] = 0.25 * ((c[0][0][1] + c[1][0][1]) + (c[0][1][1] + c[1][1][1]));
    }
}

/* neighbour values of node (I,J,K) in order -x,+x,-y,+y(,-z,+z); 0 outside. */
static void node_nbrs(int dim, int64_t m, const double* x, int64_t I, int64_t J, int64_t K,
                      double* v)
{
    int64_t P = (I - 1) + m * (J - 1) + (dim == 3 ? m * m * (K - 1) : 0);
    v[0] = I > 1 ? x[P - 1] : 0.0;
    v[1] = I < m ? x[P + 1] : 0.0;
    v[2] = J > 1 ? x[P - m] : 0.0;
    v[3] = J < m ? x[P + m] : 0.0;
    if (dim == 3) {
        v[4] = K > 1 ? x[P - m * m] : 0.0;
        v[5] = K < m ? x[P + m * m] : 0.0;
    }
}

void or_apply_A(int dim, int64_t m, const int* blocks, const double* theta,
                const double* x, double* y)
{
    double scale = (double)(m + 1) * (double)(m + 1); /* (m+1)^2 = h^-2, AMB-3 */
    int64_t Kmax = dim == 3 ? m : 1;
    for (int64_t K = 1; K <= Kmax; ++K)
        for (int64_t J = 1; J <= m; ++J)
            for (int64_t I = 1; I <= m; ++I) {
                int64_t P = (I - 1) + m * (J - 1) + (dim == 3 ? m * m * (K - 1) : 0);
                double k[6], v[6];
                node_kappa(dim, m, blocks, theta, I, J, K, k);
                node_nbrs(dim, m, x, I, J, K, v);
                double s = 0.0;
                for (int e = 0; e < 2 * dim; ++e) s += k[e] * (x[P] - v[e]);
                y[P] = scale * s;
            }
}

/* Gauss-Seidel update of node P (direct form, AMB-6):
 * y_P <- (h^2 b_P + sum_e kappa_e y_P') / sum_e kappa_e. */
static double gs_value(int dim, int64_t m, const int* blocks, const double* theta,
                       const double* b, const double* y, int64_t I, int64_t J, int64_t K,
                       int64_t P)
{
    double h2 = 1.0 / ((double)(m + 1) * (double)(m + 1));
    double k[6], v[6];
    node_kappa(dim, m, blocks, theta, I, J, K, k);
    node_nbrs(dim, m, y, I, J, K, v);
    double num = h2 * b[P];
    double den = 0.0;
    for (int e = 0; e < 2 * dim; ++e) {
        num += k[e] * v[e];
        den += k[e];
    }
    return num / den;
}

void or_gs_halfsweep(int dim, int64_t m, const int* blocks, const double* theta,
                     const double* b, double* y, int color)
{
    int64_t Kmax = dim == 3 ? m : 1;
    for (int64_t K = 1; K <= Kmax; ++K)
        for (int64_t J = 1; J <= m; ++J)
            for (int64_t I = 1; I <= m; ++I) {
                /* red = (I+J[+K]) even, in full-grid indices (O-2) */
                int64_t par = (I + J + (dim == 3 ? K : 0)) & 1;
                if (par != color) continue;
                int64_t P = (I - 1) + m * (J - 1) + (dim == 3 ? m * m * (K - 1) : 0);
                y[P] = gs_value(dim, m, blocks, theta, b, y, I, J, K, P);
            }
}

static void jacobi_sweep(int dim, int64_t m, const int* blocks, const double* theta,
                         const double* b, double* y, double omega)
{
    int64_t N = dim == 3 ? m * m * m : m * m;
    double* z = (double*)malloc(sizeof(double) * (size_t)N);
    int64_t Kmax = dim == 3 ? m : 1;
    for (int64_t K = 1; K <= Kmax; ++K)
        for (int64_t J = 1; J <= m; ++J)
            for (int64_t I = 1; I <= m; ++I) {
                int64_t P = (I - 1) + m * (J - 1) + (dim == 3 ? m * m * (K - 1) : 0);
                double g = gs_value(dim, m, blocks, theta, b, y, I, J, K, P);
                z[P] = y[P] + omega * (g - y[P]);
            }
    memcpy(y, z, sizeof(double) * (size_t)N);
    free(z);
}

/* lexicographic Gauss-Seidel sweep (node order P ascending, or descending when
 * backward): the ordering SPEC.md:288 uses for its program -- here a comparison smoother
 * (NEXT(3)); same direct-form update as the red-black half-sweep */
static void lex_sweep(int dim, int64_t m, const int* blocks, const double* theta,
                      const double* b, double* y, int backward)
{
    int64_t N = dim == 3 ? m * m * m : m * m;
    for (int64_t t = 0; t < N; ++t) {
        int64_t P = backward ? N - 1 - t : t;
        int64_t I = P % m + 1, J = (P / m) % m + 1, K = dim == 3 ? P / (m * m) + 1 : 1;
        y[P] = gs_value(dim, m, blocks, theta, b, y, I, J, K, P);
    }
}

void or_smooth(int dim, int64_t m, const int* blocks, const double* theta,
               const double* b, double* y, int kind, int sweeps, double omega)
{
    for (int s = 0; s < sweeps; ++s) {
        if (kind == OR_SMOOTH_FWD_LEX || kind == OR_SMOOTH_SYM_LEX) {
            lex_sweep(dim, m, blocks, theta, b, y, 0);
            if (kind == OR_SMOOTH_SYM_LEX) lex_sweep(dim, m, blocks, theta, b, y, 1);
        } else if (kind == OR_SMOOTH_JACOBI) {
            jacobi_sweep(dim, m, blocks, theta, b, y, omega);
        } else {
            /* forward sweep: red then black */
            or_gs_halfsweep(dim, m, blocks, theta, b, y, 0);
            or_gs_halfsweep(dim, m, blocks, theta, b, y, 1);
            if (kind == OR_SMOOTH_SYM_RBGS) {
                /* backward sweep: black then red (symmetric = forward + backward) */
                or_gs_halfsweep(dim, m, blocks, theta, b, y, 1);
                or_gs_halfsweep(dim, m, blocks, theta, b, y, 0);
            }
        }
    }
}

void or_smooth_adjoint(int dim, int64_t m, const int* blocks, const double* theta,
                       const double* b, double* y, int kind, int sweeps, double omega)
{
    for (int s = 0; s < sweeps; ++s) {
        if (kind == OR_SMOOTH_FWD_LEX || kind == OR_SMOOTH_SYM_LEX) {
            if (kind == OR_SMOOTH_SYM_LEX) lex_sweep(dim, m, blocks, theta, b, y, 0);
            lex_sweep(dim, m, blocks, theta, b, y, 1);
        } else if (kind == OR_SMOOTH_JACOBI) {
            jacobi_sweep(dim, m, blocks, theta, b, y, omega);
        } else {
            if (kind == OR_SMOOTH_SYM_RBGS) {     /* R,B,B,R reversed is itself */
                or_gs_halfsweep(dim, m, blocks, theta, b, y, 0);
                or_gs_halfsweep(dim, m, blocks, theta, b, y, 1);
            }
            or_gs_halfsweep(dim, m, blocks, theta, b, y, 1);   /* forward R,B reversed: B,R */
            or_gs_halfsweep(dim, m, blocks, theta, b, y, 0);
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Dense primitives: Cholesky, solves, Neumaier dots (AMB-20). */
/* ------------------------------------------------------------------------ */

int or_cholesky(int n, const double* A, double* L)
{
    memcpy(L, A, sizeof(double) * (size_t)n * (size_t)n);
    for (int k = 0; k < n; ++k) {
        double d = L[k * n + k];
        if (!(d > 0.0)) return k;
        d = sqrt(d);
        L[k * n + k] = d;
        for (int i = k + 1; i < n; ++i) L[i * n + k] /= d;
        for (int j = k + 1; j < n; ++j)
            for (int i = j; i < n; ++i) L[i * n + j] -= L[i * n + k] * L[j * n + k];
    }
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) L[i * n + j] = 0.0;
    return -1;
}

void or_chol_solve(int n, const double* L, const double* b, double* x)
{
    /* forward: L z = b */
    for (int i = 0; i < n; ++i) {
        double s = b[i];
        for (int k = 0; k < i; ++k) s -= L[i * n + k] * x[k];
        x[i] = s / L[i * n + i];
    }
    /* backward: L^T x = z */
    for (int i = n - 1; i >= 0; --i) {
        double s = x[i];
        for (int k = i + 1; k < n; ++k) s -= L[k * n + i] * x[k];
        x[i] = s / L[i * n + i];
    }
}

typedef struct { double s, c; } nsum;
static void nadd(nsum* a, double v)
{
    double t = a->s + v;
    if (fabs(a->s) >= fabs(v)) a->c += (a->s - t) + v;
    else a->c += (v - t) + a->s;
    a->s = t;
}

double or_dot(int64_t N, const double* x, const double* y)
{
    nsum a = {0.0, 0.0};
    for (int64_t i = 0; i < N; ++i) nadd(&a, x[i] * y[i]);
    return a.s + a.c;
}

static double sum_ones(int64_t N, const double* x)
{
    nsum a = {0.0, 0.0};
    for (int64_t i = 0; i < N; ++i) nadd(&a, x[i]);
    return a.s + a.c;
}

/* ------------------------------------------------------------------------ */
/* MGS, offline blocks (eq12c), online assembly (eq12b).   */
/* ------------------------------------------------------------------------ */

int or_mgs_append(int64_t N, int n, double* W, const double* v, double drop_tol)
{
    double* w = W + (int64_t)n * N;
    memcpy(w, v, sizeof(double) * (size_t)N);
    double vnorm = sqrt(or_dot(N, v, v));
    if (!(vnorm > 0.0)) return 1;
    for (int pass = 0; pass < 2; ++pass)
        for (int j = 0; j < n; ++j) {
            const double* wj = W + (int64_t)j * N;
            double c = or_dot(N, wj, w);
            for (int64_t i = 0; i < N; ++i) w[i] -= c * wj[i];
        }
    double wn = sqrt(or_dot(N, w, w));
    if (!(wn >= drop_tol * vnorm)) return 1;
    for (int64_t i = 0; i < N; ++i) w[i] /= wn;
    return 0;
}

static int64_t grid_N(int dim, int64_t m) { return dim == 3 ? m * m * m : m * m; }
static int grid_Q(int dim, const int* blocks)
{
    if (blocks[0] == 0) return g_face_Q;   /* face operator */
    return blocks[0] * blocks[1] * (dim == 3 ? blocks[2] : 1);
}

/* column j of the offline blocks for a basis with leading dimension ldA:
 * (A_{n,q})_{ij} = w_i^T (A_q w_j), i <= j, mirrored; A_q = A(e_q). */
static void offline_column(int dim, int64_t m, const int* blocks, int j, const double* W,
                           double* ANq, int ldA, double* fn)
{
    int64_t N = grid_N(dim, m);
    int Q = grid_Q(dim, blocks);
    double* th = (double*)calloc((size_t)Q, sizeof(double));
    double* Aw = (double*)malloc(sizeof(double) * (size_t)N);
    const double* wj = W + (int64_t)j * N;
    for (int q = 0; q < Q; ++q) {
        memset(th, 0, sizeof(double) * (size_t)Q);
        th[q] = 1.0;
        or_apply_A(dim, m, blocks, th, wj, Aw);
        double* Aq = ANq + (int64_t)q * ldA * ldA;
        for (int i = 0; i <= j; ++i) {
            double v = or_dot(N, W + (int64_t)i * N, Aw);
            Aq[i * ldA + j] = v;
            Aq[j * ldA + i] = v;
        }
    }
    fn[j] = sum_ones(N, wj); /* w_j^T f, f = 1 */
    free(th);
    free(Aw);
}

void or_offline_blocks(int dim, int64_t m, const int* blocks, int n, const double* W,
                       double* ANq, double* fn)
{
    for (int j = 0; j < n; ++j) offline_column(dim, m, blocks, j, W, ANq, n, fn);
}

/* A_n(theta) = sum_q theta_q A_{n,q} (eq12b), leading n x n block of blocks
 * stored with row stride ldA. */
static void online_assemble(int n, int Q, const double* ANq, int ldA, const double* theta,
                            double* An)
{
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int q = 0; q < Q; ++q) s += theta[q] * ANq[(int64_t)q * ldA * ldA + i * ldA + j];
            An[i * n + j] = s;
        }
}

int or_rb_solve(int n, int Q, const double* ANq, const double* fn, const double* mu,
                double* a_n)
{
    double* An = (double*)malloc(sizeof(double) * (size_t)(n * n + 1));
    double* L = (double*)malloc(sizeof(double) * (size_t)(n * n + 1));
    online_assemble(n, Q, ANq, n, mu, An);
    int piv = or_cholesky(n, An, L);
    if (piv < 0) or_chol_solve(n, L, fn, a_n);
    free(An);
    free(L);
    return piv;
}

/* ------------------------------------------------------------------------ */
/* Online solvers.                                                           */
/* ------------------------------------------------------------------------ */

typedef struct {
    int dim; int64_t m; const int* blocks; int64_t N; int Q;
    int n; const double* W; double* L;       /* L: n x n factor of A_n(mu) */
    const double* theta;
    const or_opts* o;
    double* rn; double* e;                   /* n */
    int na;                                  /* active dimension (leading columns of W) */
} solver_ctx;

/* "if the residual norm ratio ||r_k||/||r_{k+1}|| < gamma ... then we
 * increase N by 1" -- capped at the stored dimension (AMB-19). */
int or_adapt_n(double rnorm_k, double rnorm_k1, double gamma, int na, int n_max)
{
    if (gamma > 0.0 && na < n_max && rnorm_k / rnorm_k1 < gamma) return na + 1;
    return na;
}

/* the reduced system of the active dimension na: A_{na} = leading na x na block of
 * A_n(mu), whose Cholesky factor is the leading block of L (nested spaces, AMB-19);
 * e = A_{na}^{-1} rn[0..na), e[na..n) = 0 */
static void solve_active(const solver_ctx* s, const double* rn, double* e)
{
    const int n = s->n, na = s->na;
    for (int i = 0; i < na; ++i) {
        double t = rn[i];
        for (int k = 0; k < i; ++k) t -= s->L[i * n + k] * e[k];
        e[i] = t / s->L[i * n + i];
    }
    for (int i = na - 1; i >= 0; --i) {
        double t = e[i];
        for (int k = i + 1; k < na; ++k) t -= s->L[k * n + i] * e[k];
        e[i] = t / s->L[i * n + i];
    }
    for (int i = na; i < n; ++i) e[i] = 0.0;
}

/* r_n = W^T r (eq5) */
static void project(const solver_ctx* s, const double* r, double* rn)
{
    for (int j = 0; j < s->n; ++j) rn[j] = or_dot(s->N, s->W + (int64_t)j * s->N, r);
}

/* x += W e (eq7):  y0_i = sum_j W_ij e_j (in j order), x_i = x_i + y0_i */
static void prolong_add(const solver_ctx* s, const double* e, double* x)
{
    for (int64_t i = 0; i < s->N; ++i) {
        double acc = 0.0;
        for (int j = 0; j < s->n; ++j) acc += s->W[(int64_t)j * s->N + i] * e[j];
        x[i] = x[i] + acc;
    }
}

static double norm2(int64_t N, const double* v) { return sqrt(or_dot(N, v, v)); }

/* common setup: theta = mu (Q = P), Cholesky of A_n(mu) */
static int setup_reduced(solver_ctx* s, const double* ANq)
{
    if (s->n == 0) return -1;
    double* An = (double*)malloc(sizeof(double) * (size_t)s->n * (size_t)s->n);
    online_assemble(s->n, s->Q, ANq, s->n, s->theta, An);
    int piv = or_cholesky(s->n, An, s->L);
    free(An);
    return piv;
}

int or_rbi(int dim, int64_t m, const int* blocks, int n, const double* W,
           const double* ANq, const double* fn, const double* mu, const double* b_in,
           const or_opts* o, double* x, int* its, double* hist, double* a_n,
           double* true_relres)
{
    solver_ctx s = {dim, m, blocks, grid_N(dim, m), grid_Q(dim, blocks), n, W, NULL, mu, o,
                    NULL, NULL};
    int64_t N = s.N;
    s.na = (o->n_active > 0 && o->n_active < n) ? o->n_active : n;
    s.L = (double*)malloc(sizeof(double) * (size_t)(n * n + 1));
    s.rn = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    s.e = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    double* b = (double*)malloc(sizeof(double) * (size_t)N);
    double* r = (double*)malloc(sizeof(double) * (size_t)N);
    double* Ax = (double*)malloc(sizeof(double) * (size_t)N);
    if (b_in) memcpy(b, b_in, sizeof(double) * (size_t)N);
    else for (int64_t i = 0; i < N; ++i) b[i] = 1.0;
    int status = OR_MAXIT;
    *its = 0;
    if (true_relres) *true_relres = NAN;
    /* Step 0: x = 0 */
    memset(x, 0, sizeof(double) * (size_t)N);
    if (setup_reduced(&s, ANq) >= 0) { status = OR_REDUCED_NOT_SPD; goto done; }
    double bnorm = norm2(N, b);
    if (!isfinite(bnorm)) {   /* AMB-11: NONFINITE (before the b = 0 shortcut below) */
        if (hist) hist[0] = NAN;
        status = OR_NONFINITE;
        goto done;
    }
    for (int it = 0;; ++it) {
        /* Step 2: r = b - A x */
        or_apply_A(dim, m, blocks, mu, x, Ax);
        for (int64_t i = 0; i < N; ++i) r[i] = b[i] - Ax[i];
        double h = bnorm > 0.0 ? norm2(N, r) / bnorm : 0.0;
        if (hist) hist[it] = h;
        *its = it;
        if (true_relres) *true_relres = h;
        if (!isfinite(h)) { status = OR_NONFINITE; break; }
        /* Step 3: stop test (relative, AMB-7) */
        if (h < o->tol) { status = OR_CONVERGED; break; }
        if (it == o->max_iter) { status = OR_MAXIT; break; }
        /* Step 4: r_n = W^T r  (first iteration with b = f: W^T f = f_n, AMB-12) */
        if (n > 0) {
            if (it == 0 && b_in == NULL) memcpy(s.rn, fn, sizeof(double) * (size_t)n);
            else project(&s, r, s.rn);
            /* Step 5: A_n e_n = r_n (active dimension n_active) */
            solve_active(&s, s.rn, s.e);
            if (o->active_n) o->active_n[it] = s.na;
            if (it == 0 && a_n) memcpy(a_n, s.e, sizeof(double) * (size_t)n);
            /* Step 6: x = x + W e_n */
            prolong_add(&s, s.e, x);
        }
        /* Step 7: x = S(A, f, x) */
        or_smooth(dim, m, blocks, mu, b, x, o->smoother, o->sweeps, o->omega);
    }
done:
    free(s.L); free(s.rn); free(s.e); free(b); free(r); free(Ax);
    return status;
}

/* y = RBI(A, r, W, 1) from zero:  y0 = W A_n^{-1} W^T r,
 * y = S(A, r, y0).  If rn_given, W^T r is not recomputed (AMB-12). */
static void rbi_precond(const solver_ctx* s, const double* r, const double* rn_given,
                        double* y, double* e_out)
{
    memset(y, 0, sizeof(double) * (size_t)s->N);
    if (s->o->precond == OR_PRECOND_SYM) {
        /* symmetric two-level RBI (NEXT(3)): y1 = S*(A, r, 0); y2 = y1 + W A_n^{-1} W^T
         * (r - A y1); y = S(A, r, y2) -- M^{-1} is symmetric (S* the adjoint of S) */
        or_smooth_adjoint(s->dim, s->m, s->blocks, s->theta, r, y, s->o->smoother, s->o->sweeps,
                          s->o->omega);
        if (s->n > 0) {
            double* q = (double*)malloc(sizeof(double) * (size_t)s->N);
            or_apply_A(s->dim, s->m, s->blocks, s->theta, y, q);
            for (int64_t i = 0; i < s->N; ++i) q[i] = r[i] - q[i];
            project(s, q, s->rn);
            free(q);
            solve_active(s, s->rn, s->e);
            if (e_out) memcpy(e_out, s->e, sizeof(double) * (size_t)s->n);
            prolong_add(s, s->e, y);
        }
        or_smooth(s->dim, s->m, s->blocks, s->theta, r, y, s->o->smoother, s->o->sweeps, s->o->omega);
        return;
    }
    if (s->n > 0) {
        if (rn_given) memcpy(s->rn, rn_given, sizeof(double) * (size_t)s->n);
        else project(s, r, s->rn);
        solve_active(s, s->rn, s->e);
        if (e_out) memcpy(e_out, s->e, sizeof(double) * (size_t)s->n);
        prolong_add(s, s->e, y);
    }
    or_smooth(s->dim, s->m, s->blocks, s->theta, r, y, s->o->smoother, s->o->sweeps, s->o->omega);
}

int or_rbcg(int dim, int64_t m, const int* blocks, int n, const double* W,
            const double* ANq, const double* fn, const double* mu, const double* b_in,
            const or_opts* o, double* x, int* its, double* hist, double* a_n,
            double* true_relres)
{
    solver_ctx s = {dim, m, blocks, grid_N(dim, m), grid_Q(dim, blocks), n, W, NULL, mu, o,
                    NULL, NULL};
    int64_t N = s.N;
    s.na = (o->n_active > 0 && o->n_active < n) ? o->n_active : n;
    s.L = (double*)malloc(sizeof(double) * (size_t)(n * n + 1));
    s.rn = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    s.e = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    double* f = (double*)malloc(sizeof(double) * (size_t)N);
    double* r = (double*)malloc(sizeof(double) * (size_t)N);
    double* y = (double*)malloc(sizeof(double) * (size_t)N);
    double* p = (double*)malloc(sizeof(double) * (size_t)N);
    double* q = (double*)malloc(sizeof(double) * (size_t)N);
    double* rold = o->beta_rule == OR_BETA_PR ? (double*)malloc(sizeof(double) * (size_t)N) : NULL;
    if (b_in) memcpy(f, b_in, sizeof(double) * (size_t)N);
    else for (int64_t i = 0; i < N; ++i) f[i] = 1.0;
    int status = OR_MAXIT;
    *its = 0;
    if (true_relres) *true_relres = NAN;
    /* Step 0: x_0 = 0, k = 0 */
    memset(x, 0, sizeof(double) * (size_t)N);
    if (setup_reduced(&s, ANq) >= 0) { status = OR_REDUCED_NOT_SPD; goto done; }
    double fnorm = norm2(N, f);
    /* Step 1: r_0 = f - A x_0 = f */
    memcpy(r, f, sizeof(double) * (size_t)N);
    if (hist) hist[0] = fnorm > 0.0 ? 1.0 : 0.0;
    /* AMB-11: NaN / Inf anywhere is NONFINITE -- tested before the f = 0 shortcut,
     * which a NaN norm would otherwise take (!(NaN > 0) holds) */
    if (!isfinite(fnorm)) { status = OR_NONFINITE; goto final; }
    if (!(fnorm > 0.0)) { status = OR_CONVERGED; goto final; }
    /* Step 2: y_0 = RBI(A, r_0, W, 1);  W^T r_0 = W^T f = f_n when b = f */
    if (o->active_n) o->active_n[0] = s.na;
    rbi_precond(&s, r, (b_in == NULL && o->precond != OR_PRECOND_SYM) ? fn : NULL, y, a_n);
    /* Step 3: p_0 = y_0 */
    memcpy(p, y, sizeof(double) * (size_t)N);
    double rho = or_dot(N, r, y);
    if (!(rho > o->delta * norm2(N, y) * norm2(N, r))) {
        status = isfinite(rho) ? OR_PRECOND : OR_NONFINITE;
        goto final;
    }
    for (int k = 0;; ++k) {
        if (k == o->max_iter) { status = OR_MAXIT; *its = k; break; }
        /* Step 5: alpha_k = r_k^T y_k / p_k^T A p_k */
        or_apply_A(dim, m, blocks, mu, p, q);
        double sigma = or_dot(N, p, q);
        if (!(sigma > 0.0)) { status = isfinite(sigma) ? OR_CURVATURE : OR_NONFINITE; *its = k; break; }
        double alpha = rho / sigma;
        /* Step 6-7 */
        for (int64_t i = 0; i < N; ++i) x[i] = x[i] + alpha * p[i];
        if (rold) memcpy(rold, r, sizeof(double) * (size_t)N);   /* r_k, for the PR beta */
        const double rnorm_k = norm2(N, r);
        for (int64_t i = 0; i < N; ++i) r[i] = r[i] - alpha * q[i];
        const double rnorm_k1 = norm2(N, r);
        double h = rnorm_k1 / fnorm;
        if (hist) hist[k + 1] = h;
        *its = k + 1;
        if (!isfinite(h)) { status = OR_NONFINITE; break; }
        /* Step 8 */
        if (h < o->tol) { status = OR_CONVERGED; break; }
        /* adaptive n: grow the space of the next preconditioner */
        s.na = or_adapt_n(rnorm_k, rnorm_k1, o->gamma, s.na, n);
        if (o->active_n) o->active_n[k + 1] = s.na;
        /* Step 9: y_{k+1} = RBI(A, r_{k+1}, W, 1) */
        rbi_precond(&s, r, NULL, y, NULL);
        /* Step 10: beta_k = y_{k+1}^T r_{k+1} / y_k^T r_k */
        double rho_new = or_dot(N, y, r);
        if (!(rho_new > o->delta * norm2(N, y) * norm2(N, r))) {
            status = isfinite(rho_new) ? OR_PRECOND : OR_NONFINITE;
            break;
        }
        /* FR as printed; PR (flexible): beta = y_{k+1}^T (r_{k+1} - r_k) / y_k^T r_k */
        double beta = rold ? (rho_new - or_dot(N, y, rold)) / rho : rho_new / rho;
        /* Step 11: p_{k+1} = y_{k+1} + beta_k p_k */
        for (int64_t i = 0; i < N; ++i) p[i] = y[i] + beta * p[i];
        rho = rho_new;
    }
final:
    if (true_relres) {
        or_apply_A(dim, m, blocks, mu, x, q);
        for (int64_t i = 0; i < N; ++i) q[i] = f[i] - q[i];
        *true_relres = fnorm > 0.0 ? norm2(N, q) / fnorm : 0.0;
    }
done:
    free(s.L); free(s.rn); free(s.e); free(f); free(r); free(y); free(p); free(q); free(rold);
    return status;
}

/* one application of the RBCG preconditioner y = M^{-1} r (either variant), for tests */
int or_precond_apply(int dim, int64_t m, const int* blocks, int n, const double* W,
                     const double* ANq, const double* mu, const or_opts* o, const double* r, double* y)
{
    solver_ctx s = {dim, m, blocks, grid_N(dim, m), grid_Q(dim, blocks), n, W, NULL, mu, o,
                    NULL, NULL};
    s.na = (o->n_active > 0 && o->n_active < n) ? o->n_active : n;
    s.L = (double*)malloc(sizeof(double) * (size_t)(n * n + 1));
    s.rn = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    s.e = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    int st = 0;
    if (setup_reduced(&s, ANq) >= 0) st = -1;
    else rbi_precond(&s, r, NULL, y, NULL);
    free(s.L); free(s.rn); free(s.e);
    return st;
}

int or_cg(int dim, int64_t m, const int* blocks, const double* mu, const double* b_in,
          double tol, int max_iter, double* x, int* its)
{
    int64_t N = grid_N(dim, m);
    double* r = (double*)malloc(sizeof(double) * (size_t)N);
    double* p = (double*)malloc(sizeof(double) * (size_t)N);
    double* q = (double*)malloc(sizeof(double) * (size_t)N);
    for (int64_t i = 0; i < N; ++i) r[i] = b_in ? b_in[i] : 1.0;
    memset(x, 0, sizeof(double) * (size_t)N);
    memcpy(p, r, sizeof(double) * (size_t)N);
    double fnorm = norm2(N, r), rho = or_dot(N, r, r);
    int status = OR_MAXIT;
    *its = 0;
    for (int k = 0; k < max_iter; ++k) {
        or_apply_A(dim, m, blocks, mu, p, q);
        double sigma = or_dot(N, p, q);
        if (!(sigma > 0.0)) { status = OR_CURVATURE; break; }
        double alpha = rho / sigma;
        for (int64_t i = 0; i < N; ++i) x[i] += alpha * p[i];
        for (int64_t i = 0; i < N; ++i) r[i] -= alpha * q[i];
        *its = k + 1;
        double rho_new = or_dot(N, r, r);
        if (sqrt(rho_new) / fnorm < tol) { status = OR_CONVERGED; break; }
        double beta = rho_new / rho;
        for (int64_t i = 0; i < N; ++i) p[i] = r[i] + beta * p[i];
        rho = rho_new;
    }
    free(r); free(p); free(q);
    return status;
}

/* ------------------------------------------------------------------------ */
/* Greedy sampling (algorithm0 / algorithm3) with AMB-13.                    */
/* ------------------------------------------------------------------------ */

/* snapshot solve x(mu) = RBCG(A(mu), f, W_{n}) at tolerance tol (adaptive:
 * PAPER.md:301); n = 0 is the symmetric-GS-preconditioned CG. */
static int snapshot(int dim, int64_t m, const int* blocks, int n, const double* W,
                    const double* ANq_ld, int ldA, const double* fn, const double* mu,
                    double tol, int max_iter, double* x, int* its)
{
    int Q = grid_Q(dim, blocks);
    /* compact leading n x n blocks */
    double* A = (double*)malloc(sizeof(double) * (size_t)(Q * n * n + 1));
    for (int q = 0; q < Q; ++q)
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                A[(int64_t)q * n * n + i * n + j] = ANq_ld[(int64_t)q * ldA * ldA + i * ldA + j];
    or_opts o = {tol, max_iter, OR_SMOOTH_SYM_RBGS, 1, 1.0, 1e-12};
    double trr;
    int st = or_rbcg(dim, m, blocks, n, W, A, fn, mu, NULL, &o, x, its, NULL, NULL, &trr);
    free(A);
    return st;
}

/* affine right-hand sides for the greedy (NEXT(4), AMB-23): f(mu_t) = sum_r phi[t][r] f_r;
 * set by or_set_greedy_rhs before or_greedy / or_basis_from_samples, R = 0 = f = 1 */
static int g_rhs_R = 0;
static const double* g_rhs_phi = NULL;    /* [n_train][R] */
static const double* g_rhs_terms = NULL;  /* [R][N] */
static double* g_rhs_fnr = NULL;          /* [R][n_max] out: f_{N,r} = W^T f_r */

void or_set_greedy_rhs(int R, const double* phi, const double* terms, double* fnr_out)
{
    g_rhs_R = R;
    g_rhs_phi = phi;
    g_rhs_terms = terms;
    g_rhs_fnr = fnr_out;
}

/* snapshot of RBCG (snapshot()) with an explicit right-hand side b */
static int snapshot_b(int dim, int64_t m, const int* blocks, int n, const double* W,
                      const double* ANq_ld, int ldA, const double* fn, const double* mu, const double* b,
                      double tol, int max_iter, double* x, int* its)
{
    int Q = grid_Q(dim, blocks);
    double* A = (double*)malloc(sizeof(double) * (size_t)(Q * n * n + 1));
    for (int q = 0; q < Q; ++q)
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                A[(int64_t)q * n * n + i * n + j] = ANq_ld[(int64_t)q * ldA * ldA + i * ldA + j];
    or_opts o = {tol, max_iter, OR_SMOOTH_SYM_RBGS, 1, 1.0, 1e-12};
    double trr;
    int st = or_rbcg(dim, m, blocks, n, W, A, fn, mu, b, &o, x, its, NULL, NULL, &trr);
    free(A);
    return st;
}

static int greedy_core(int dim, int64_t m, const int* blocks, int n_train,
                       const double* mu_train, int n_max, int adaptive,
                       double snapshot_tol, double drop_tol, double* W, double* ANq,
                       double* fn, int* selected, double* indicator, int* snap_iters,
                       int* n_rejected, int from_list)
{
    int64_t N = grid_N(dim, m);
    int Q = grid_Q(dim, blocks), P = Q;
    double* x = (double*)malloc(sizeof(double) * (size_t)N);
    char* excluded = (char*)calloc((size_t)n_train + 1, 1);
    double* ind = (double*)malloc(sizeof(double) * (size_t)n_train + 8);
    double* AN = (double*)malloc(sizeof(double) * (size_t)n_max * n_max + 8);
    double* L = (double*)malloc(sizeof(double) * (size_t)n_max * n_max + 8);
    double* a = (double*)malloc(sizeof(double) * (size_t)n_max + 8);
    int n = 0, rej = 0, its_first = -1;
    const int R = g_rhs_R;
    double* bsnap = R > 0 ? (double*)malloc(sizeof(double) * (size_t)N) : NULL;
    double* fn_t = R > 0 ? (double*)malloc(sizeof(double) * (size_t)n_max + 8) : NULL;
    /* Step 0/1: mu_1 = Xi_train[0] (AMB-13; Xi_train itself is seeded random) */
    int cand = 0;
    int list_pos = 0;
    while (n < n_max && cand >= 0) {
        const double* mu = mu_train + (int64_t)cand * P;
        if (R > 0) {   /* f(mu_cand) = sum_r phi_r f_r */
            for (int64_t i = 0; i < N; ++i) {
                double v = 0.0;
                for (int r = 0; r < R; ++r) v += g_rhs_phi[(int64_t)cand * R + r] * g_rhs_terms[(int64_t)r * N + i];
                bsnap[i] = v;
            }
        }
        /* Step 3: solve the snapshot (adaptive: RBCG with W_{N-1}) */
        int its = 0, st;
        if (!adaptive || n == 0) {
            /* N = 1 (or plain greedy): the "standard solver" of PAPER.md:291 = SGS-PCG */
            st = snapshot_b(dim, m, blocks, 0, W, ANq, n_max, fn, mu, bsnap, snapshot_tol, 200000, x, &its);
            if (n == 0 && its_first < 0) its_first = its;
        } else {
            /* RBCG with W_{N-1}, guarded (AMB-22): if it has not
             * converged within 2*its_1 + 50 iterations (its_1 = the N = 1 snapshot),
             * fall back to the standard solver. */
            st = snapshot_b(dim, m, blocks, n, W, ANq, n_max, fn, mu, bsnap, snapshot_tol,
                            2 * (its_first > 0 ? its_first : 1000) + 50, x, &its);
            if (st != OR_CONVERGED) {
                st = snapshot_b(dim, m, blocks, 0, W, ANq, n_max, fn, mu, bsnap, snapshot_tol, 200000, x, &its);
                its = -its;   /* reported negative: fallback used */
            }
        }
        (void)st;
        /* Step 4: W_N = MGS(W_{N-1}, x(mu_N)) */
        int rejected = or_mgs_append(N, n, W, x, drop_tol);
        excluded[cand] = 1;
        if (rejected) {
            ++rej;
        } else {
            selected[n] = cand;
            if (snap_iters) snap_iters[n] = its;
            offline_column(dim, m, blocks, n, W, ANq, n_max, fn);
            for (int r = 0; r < R; ++r)   /* f_{N,r}[n] = w_n^T f_r */
                g_rhs_fnr[(int64_t)r * n_max + n] = or_dot(N, W + (int64_t)n * N, g_rhs_terms + (int64_t)r * N);
            ++n;
        }
        if (from_list) {
            ++list_pos;
            cand = list_pos < n_train ? list_pos : -1;
            continue;
        }
        if (n == 0) {
            /* first snapshot rejected: take the next training parameter */
            cand = -1;
            for (int t = 0; t < n_train; ++t) if (!excluded[t]) { cand = t; break; }
            continue;
        }
        /* Step 5: solve A_N(mu) x_N(mu) = f_N(mu) for all mu in Xi_train */
        for (int t = 0; t < n_train; ++t) {
            online_assemble(n, Q, ANq, n_max, mu_train + (int64_t)t * P, AN);
            if (or_cholesky(n, AN, L) >= 0) { ind[t] = -INFINITY; continue; }
            if (R > 0) {   /* f_N(mu_t) = sum_r phi_r(mu_t) f_{N,r} */
                for (int j = 0; j < n; ++j) {
                    double v = 0.0;
                    for (int r = 0; r < R; ++r) v += g_rhs_phi[(int64_t)t * R + r] * g_rhs_fnr[(int64_t)r * n_max + j];
                    fn_t[j] = v;
                }
                or_chol_solve(n, L, fn_t, a);
            } else {
                or_chol_solve(n, L, fn, a);
            }
            double sabs = 0.0;
            for (int j = 0; j < n; ++j) sabs += fabs(a[j]);
            ind[t] = sabs;
        }
        /* Step 6: argmax of the L1 norm, excluding used parameters, lowest index on ties */
        cand = -1;
        double best = -INFINITY;
        for (int t = 0; t < n_train; ++t)
            if (!excluded[t] && ind[t] > best) { best = ind[t]; cand = t; }
        if (indicator) indicator[n - 1] = best;
    }
    if (n_rejected) *n_rejected = rej;
    free(x); free(excluded); free(ind); free(AN); free(L); free(a); free(bsnap); free(fn_t);
    return n;
}

int or_greedy(int dim, int64_t m, const int* blocks, int n_train, const double* mu_train,
              int n_max, int adaptive, double snapshot_tol, double drop_tol,
              double* W_out, double* ANq_out, double* fn_out, int* selected,
              double* indicator, int* snap_iters, int* n_rejected)
{
    return greedy_core(dim, m, blocks, n_train, mu_train, n_max, adaptive, snapshot_tol,
                       drop_tol, W_out, ANq_out, fn_out, selected, indicator, snap_iters,
                       n_rejected, 0);
}

int or_basis_from_samples(int dim, int64_t m, const int* blocks, int count,
                          const double* mus, double snapshot_tol, double drop_tol,
                          double* W_out, double* ANq_out, double* fn_out,
                          int* snap_iters, int* n_rejected)
{
    int* sel = (int*)malloc(sizeof(int) * (size_t)count + 4);
    int n = greedy_core(dim, m, blocks, count, mus, count, 1, snapshot_tol, drop_tol, W_out,
                        ANq_out, fn_out, sel, NULL, snap_iters, n_rejected, 1);
    free(sel);
    return n;
}
