/*
 * oracle.h -- plain, slow, obviously-correct CPU fp64 oracle for the online
 * phase of the reduced-basis iterative solvers of Nguyen & Chen
 * (arXiv:1804.06363, /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * product path under paper_1804_06363_b200/.
 *
 * Conventions:
 *  - grid: dim in {2,3}, m interior nodes per axis, h = 1/(m+1); unknown
 *    P = (I-1) + m(J-1) + m^2(K-1), I,J,K in 1..m; Dirichlet zero outside.
 *  - cell (a,b,c), a in 0..m, block index per axis floor((2a+1)p / (2(m+1))),
 *    q = bx + px*by + px*py*bz; coefficient theta_q (theta = mu, Q = P).
 *  - edge coefficient = cell average (AMB-1/AMB-4), A = (m+1)^2 K, f = 1.
 *  - all vectors of length N = m^dim; W is column-major N x n (ld = N).
 *  - dense small matrices are row-major n x n.
 */
#ifndef RBS_ORACLE_H
#define RBS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_SMOOTH_SYM_RBGS = 0, OR_SMOOTH_FWD_RBGS = 1, OR_SMOOTH_JACOBI = 2,
       OR_SMOOTH_FWD_LEX = 3, OR_SMOOTH_SYM_LEX = 4 };   /* lexicographic GS: comparison only */
enum { OR_PRECOND_POST = 0, OR_PRECOND_SYM = 1 };   /* RBCG preconditioner (NEXT(3)) */
enum { OR_BETA_FR = 0, OR_BETA_PR = 1 };            /* RBCG beta (NEXT(3)) */
enum { OR_CONVERGED = 0, OR_MAXIT = 1, OR_REDUCED_NOT_SPD = 2, OR_CURVATURE = 3,
       OR_PRECOND = 4, OR_NONFINITE = 5 };

typedef struct {
    double tol;        /* relative residual tolerance (AMB-7) */
    int max_iter;      /* AMB-9 */
    int smoother;      /* OR_SMOOTH_* */
    int sweeps;        /* nu */
    double omega;      /* Jacobi damping */
    double delta;      /* PRECOND breakdown threshold (AMB-11) */
    int n_active;      /* active RB dimension (0 = n): the leading columns of W are used */
    double gamma;      /* RBCG adaptive-n rule, 0 = off: grow the active
                          dimension by one when ||r_k|| / ||r_{k+1}|| < gamma */
    int* active_n;     /* optional, max_iter+1 entries: active dimension of the k-th
                          preconditioner application (RBCG) / correction (RBI) */
    int precond;       /* RBCG: OR_PRECOND_POST (the paper's RBI(A, r, W, 1)) or
                          OR_PRECOND_SYM: pre-smoothing with the adjoint sweep, coarse
                          correction, post-smoothing (NEXT(3)) */
    int beta_rule;     /* RBCG: OR_BETA_FR (as printed) or OR_BETA_PR
                          (Polak-Ribiere / flexible: (y_{k+1}^T (r_{k+1} - r_k)) / y_k^T r_k) */
} or_opts;

/* General affine operator (NEXT(4), AMB-23): blocks = {0,0,0} selects face
 * coefficients kappa_e = sum_q theta_q faces[q][d][idx] (layout in oracle.c) set
 * here; the pointer is kept (caller owns it) until the next call. */
void or_set_faces(int Q, const double* faces);

/* (A(theta) x) matrix-free, PAPER.md:98-103 (eq12) with AMB-1..4. */
void or_apply_A(int dim, int64_t m, const int* blocks, const double* theta,
                const double* x, double* y);
/* one red-black Gauss-Seidel half-sweep of colour c on A y = b (AMB-5). */
void or_gs_halfsweep(int dim, int64_t m, const int* blocks, const double* theta,
                     const double* b, double* y, int color);
/* smoother S(A, b, y) in place, PAPER.md:148-153 (eq8). */
void or_smooth(int dim, int64_t m, const int* blocks, const double* theta,
               const double* b, double* y, int kind, int sweeps, double omega);
/* its adjoint (in the A inner product) S*: the elementary sweeps in reverse order, each
 * replaced by its adjoint (a red-black half-sweep and a Jacobi sweep are self-adjoint, a
 * forward lexicographic sweep's adjoint is the backward sweep) -- the pre-smoother of
 * the symmetric two-level preconditioner. */
void or_smooth_adjoint(int dim, int64_t m, const int* blocks, const double* theta,
                       const double* b, double* y, int kind, int sweeps, double omega);

/* adaptive-n rule of PAPER.md:287 (DESIGN.md AMB-19): returns na + 1 when
 * ||r_k|| / ||r_{k+1}|| < gamma (gamma > 0) and na < n_max, else na. */
int or_adapt_n(double rnorm_k, double rnorm_k1, double gamma, int na, int n_max);

/* dense Cholesky A = L L^T (right-looking); returns -1 or failing pivot. */
int or_cholesky(int n, const double* A, double* L);
void or_chol_solve(int n, const double* L, const double* b, double* x);
/* Neumaier-compensated dot product (AMB-20). */
double or_dot(int64_t N, const double* x, const double* y);

/* MGS with one unconditional re-orthogonalisation pass.
 * W column-major with ld = N holding n columns; appends column n on success.
 * returns 0 on success, 1 if rejected (post norm < drop_tol*||v||). */
int or_mgs_append(int64_t N, int n, double* W, const double* v, double drop_tol);

/* offline blocks A_{n,q} = W^T A_q W (i<=j then mirrored) and f_{n,1} = W^T 1
 * (eq12c).  ANq: Q x n x n, fn: n. */
void or_offline_blocks(int dim, int64_t m, const int* blocks, int n, const double* W,
                       double* ANq, double* fn);

/* RBI (algorithm1).  b == NULL means the problem RHS f = 1
 * (then W^T f = fn is taken from the offline block, PAPER.md:171 / AMB-12).
 * hist: max_iter+1 entries (relative residuals), a_n: first reduced coeffs (n).
 * returns status; *its = iterations. */
int or_rbi(int dim, int64_t m, const int* blocks, int n, const double* W,
           const double* ANq, const double* fn, const double* mu, const double* b,
           const or_opts* o, double* x, int* its, double* hist, double* a_n,
           double* true_relres);

/* RBCG (algorithm2); n == 0 is symmetric-GS-PCG. */
int or_rbcg(int dim, int64_t m, const int* blocks, int n, const double* W,
            const double* ANq, const double* fn, const double* mu, const double* b,
            const or_opts* o, double* x, int* its, double* hist, double* a_n,
            double* true_relres);

/* one application y = M^{-1} r of the RBCG preconditioner selected by o->precond
 * (tests of the preconditioner itself); returns 0, or -1 if A_n(mu) is not SPD. */
int or_precond_apply(int dim, int64_t m, const int* blocks, int n, const double* W,
                     const double* ANq, const double* mu, const or_opts* o, const double* r, double* y);

/* plain CG (context only). */
int or_cg(int dim, int64_t m, const int* blocks, const double* mu, const double* b,
          double tol, int max_iter, double* x, int* its);

/* Greedy (algorithm0; adaptive=1: algorithm3).
 * W_out: column-major N x n_max.  ANq_out: Q x n_max x n_max (only the leading
 * n_out x n_out block of each q is meaningful, row stride n_max).
 * snap_iters[k] < 0: the guarded RBCG snapshot did not converge within
 * 2*its_1 + 50 iterations and the SGS-PCG fallback took |snap_iters[k]|
 * iterations (DESIGN.md AMB-22).  returns n_out. */
int or_greedy(int dim, int64_t m, const int* blocks, int n_train, const double* mu_train,
              int n_max, int adaptive, double snapshot_tol, double drop_tol,
              double* W_out, double* ANq_out, double* fn_out, int* selected,
              double* indicator, int* snap_iters, int* n_rejected);

/* Affine right-hand sides for the next or_greedy / or_basis_from_samples (NEXT(4)):
 * snapshots solve with f(mu_t) = sum_r phi[t*R + r] terms[r*N + i]; the offline
 * vectors f_{N,r} = W^T f_r go to fnr_out [R][n_max]; the indicator solves use
 * f_N(mu_t) = sum_r phi_r f_{N,r}.  R = 0 restores f = 1.  Pointers are kept. */
void or_set_greedy_rhs(int R, const double* phi, const double* terms, double* fnr_out);

/* Build a basis from a given sample list (the fine-grid half of the
 * multi-fidelity approach): RBCG snapshots with the growing
 * basis, MGS, incremental offline blocks.  returns n_out. */
int or_basis_from_samples(int dim, int64_t m, const int* blocks, int count,
                          const double* mus, double snapshot_tol, double drop_tol,
                          double* W_out, double* ANq_out, double* fn_out,
                          int* snap_iters, int* n_rejected);

/* Galerkin RB solve for one mu: a_n = A_n(mu)^{-1} f_n. */
int or_rb_solve(int n, int Q, const double* ANq, const double* fn, const double* mu,
                double* a_n);

#ifdef __cplusplus
}
#endif
#endif
