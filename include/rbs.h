/*
 * rbs.h -- C ABI of the B200-native batched reduced-basis (RB) online solver.
 *
 * Method: Nguyen & Chen, "Reduced-basis method for the iterative solution of
 * parametrized SPD linear systems", arXiv:1804.06363.  Citations
 * are PAPER.md line numbers plus the equation / algorithm label.
 *
 * Problem (eq1, 98-103 eq12):  A(mu) x(mu) = f(mu),
 *   A(mu) = sum_q theta_q(mu) A_q,   f(mu) = sum_r phi_r(mu) f_r,
 * with A_q the matrix-free cell-averaged 5-point (2D) / 7-point (3D)
 * diffusion stencils of a piecewise-constant coefficient on a block
 * partition of the unit square / cube (DESIGN.md AMB-1..4), theta_q = mu_q.
 *
 * Conventions for every entry point:
 *  - Status: every call returns rbs_status; nothing aborts, no C++ exception
 *    crosses the ABI.  Details of the last failure: rbs_last_error(ctx).
 *  - Memory: the library allocates NO device memory.  Device buffers are
 *    caller-owned (allocated by PyTorch in the Python binding), sizes are
 *    queried first (rbs_*_size).  Pointers are borrowed for the duration of
 *    the call unless stated otherwise ("retained").
 *  - Streams: work is enqueued on the given cudaStream_t (void*; NULL = legacy
 *    default stream).  Calls that return host results synchronise it.
 *  - Node ordering of N-vectors: lexicographic, x fastest:
 *    P = (I-1) + m(J-1) + m^2(K-1), I,J,K in 1..m (homogeneous Dirichlet).
 *  - Batched vectors at the boundary are query-major [B][N] fp64.  The
 *    internal layout is node-major [N][B_pad] (lane = query); the library
 *    transposes on entry/exit.
 *  - A context is not thread-safe: use one context per host thread.  Several
 *    contexts may share a device (each owns its storage and workspace, e.g.
 *    bench.py's concurrent batch streams); the library keeps no mutable
 *    process-global state (kernel attributes are set once per device under a
 *    lock at rbs_create).
 */
#ifndef RBS_H
#define RBS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RBS_VERSION 1
#define RBS_MAX_BATCH 64     /* queries per rbs_solve_batch call */
#define RBS_MAX_N 64         /* RB dimension n */
#define RBS_MAX_Q 64         /* affine terms */
#define RBS_MAX_R 64         /* right-hand-side terms (rbs_affine_rhs) */

typedef struct rbs_ctx rbs_ctx;

typedef enum {
    RBS_OK = 0,
    RBS_E_ARG = 1,          /* invalid argument (NULL pointer, bad enum, ...) */
    RBS_E_DIM = 2,          /* dimension mismatch / size out of range */
    RBS_E_STATE = 3,        /* call out of order (e.g. solve before basis) */
    RBS_E_NOT_SPD = 4,      /* offline: reduced matrix not SPD */
    RBS_E_CUDA = 5,         /* CUDA runtime error (see rbs_last_error) */
    RBS_E_NOMEM = 6,        /* caller buffer smaller than the queried size */
    RBS_E_UNSUPPORTED = 7   /* valid but not supported by this build */
} rbs_status;

/* per-query termination (a per-query breakdown never fails the call) */
typedef enum {
    RBS_Q_CONVERGED = 0,        /* ||r||/||f|| < tol (eq:relerr) */
    RBS_Q_MAXIT = 1,            /* max_iter reached */
    RBS_Q_REDUCED_NOT_SPD = 2,  /* Cholesky of A_N(mu) hit a pivot <= 0 */
    RBS_Q_CURVATURE = 3,        /* RBCG: p^T A p <= 0 */
    RBS_Q_PRECOND = 4,          /* RBCG: y^T r <= delta ||y|| ||r|| (DESIGN.md AMB-11) */
    RBS_Q_NONFINITE = 5         /* NaN / Inf encountered */
} rbs_qstatus;

enum { RBS_RBI = 0, RBS_RBCG = 1 };
/* smoother S of PAPER.md:148-153 (eq8), "the smoother (Jacobi or Gauss-Seidel)":
 * red-black Gauss-Seidel, symmetric (R,B,R per sweep) or forward (R,B) -- AMB-5/6 --
 * or damped Jacobi y <- y + omega D^-1 (b - A y) (opts.omega; flat kernels, not with
 * mesh slabs) */
enum { RBS_SMOOTH_SYM_RBGS = 0, RBS_SMOOTH_FWD_RBGS = 1, RBS_SMOOTH_JACOBI = 2 };
enum { RBS_MEM_DEVICE = 0, RBS_MEM_HOST = 1 };
/* greedy modes: PLAIN (algorithm0), ADAPTIVE (algorithm3),
 * SAMPLES: adaptive snapshots at the given parameters in list order, no selection -- the
 * fine-grid half of the multi-fidelity approach: select on a coarse grid,
 * then build the fine basis from the selected parameters */
/* SAMPLES_BATCH: the same, the samples solved 8 at a time by RBCG with the symmetric two-level
 * preconditioner on the basis built so far (constant rhs only; DESIGN.md AMB-27) */
enum { RBS_GREEDY_PLAIN = 0, RBS_GREEDY_ADAPTIVE = 1, RBS_GREEDY_SAMPLES = 2, RBS_GREEDY_SAMPLES_BATCH = 3 };

int rbs_version(void);
const char* rbs_status_string(rbs_status s);

/* Create a context bound to CUDA device `cuda_device` (checks sm_100). */
rbs_status rbs_create(int cuda_device, rbs_ctx** out);
void rbs_destroy(rbs_ctx* ctx);
/* Detail of the last failure of a call on ctx ("" if none).  Owned by ctx. */
const char* rbs_last_error(const rbs_ctx* ctx);

/* ---------------------------------------------------------------------------
 * Affine family (eq12).
 *
 * rbs_set_operator_blocks: dim in {2,3}; m[0..dim-1] interior nodes per axis
 * (must be equal: h = 1/(m+1) on every axis; 1 <= m <= 65535; N = m^dim);
 * blocks[0..dim-1] subdomains per axis (1..16).  Q = prod(blocks).  Cell
 * (a,b,c) belongs to block floor((2a+1) p / (2(m+1))) per axis; q = bx +
 * px*by + px*py*bz; A_q = A(e_q).  Invalidates any loaded basis.
 * Errors: RBS_E_ARG / RBS_E_DIM.
 */
rbs_status rbs_set_operator_blocks(rbs_ctx* ctx, int dim, const int64_t m[3], const int blocks[3]);

/* ---------------------------------------------------------------------------
 * General affine operator (NEXT(4); DESIGN.md AMB-23; the paper's Case 1/2,
 * PAPER.md:319-383): A(theta) = (m+1)^2 K(theta), (K x)_P = sum_e kappa_e (x_P - x_P')
 * over the 2*dim faces e of node P (Dirichlet zero outside), with
 *   kappa_e(theta) = sum_q theta_q faces[q][d][idx]   (q ascending),
 * faces_dev: device, row-major [Q][dim][nf], nf = (m+1) m^(dim-1), BORROWED (the
 * caller keeps it alive while the context uses this operator).  The face between
 * nodes a and a+1 (a = 0..m) along axis d has idx
 *   x: a + (m+1)((J-1) + m(K-1)),  y: (I-1) + m(a + (m+1)(K-1)),  z: (I-1) + m((J-1) + m a)
 * (I,J,K in 1..m; K = 1 in 2D).  theta = mu (the caller passes theta as mu to
 * rbs_solve_batch, P = Q).  Runs the flat kernels (no row march).  Invalidates any
 * loaded basis.  Errors: RBS_E_ARG, RBS_E_DIM.
 */
rbs_status rbs_set_operator_faces(rbs_ctx* ctx, int dim, int64_t m, int Q, const double* faces_dev);

/* Affine right-hand sides f(mu_b) = sum_r phi[b][r] f_r for a batch (PAPER.md:98-103,
 * eq12 with R terms): out_dev[b][i] = sum_r phi_host[b*R + r] * terms_dev[r*N + i]
 * (r ascending).  terms_dev [R][N] and out_dev [B][N] are device, caller-owned;
 * out_dev is the rhs_dev of rbs_solve_batch.  Synchronises `stream`.
 * Errors: RBS_E_STATE (no operator), RBS_E_DIM, RBS_E_ARG, RBS_E_CUDA. */
rbs_status rbs_affine_rhs(rbs_ctx* ctx, int B, int R, const double* phi_host, const double* terms_dev,
                          double* out_dev, void* stream);

/* R = 1, f_1 = value * ones(N), phi_1 = 1 (the BASELINE configs use 1.0).  Drops affine
 * rhs terms set by rbs_set_rhs_terms (then the basis must be loaded again). */
rbs_status rbs_set_rhs_constant(rbs_ctx* ctx, double value);

/* Affine right-hand side f(mu) = sum_r phi_r(mu) f_r (eq12; the online
 * f_N(mu) = sum_r phi_r(mu) f_{N,r} of eq12b):
 *  f_dev: R device pointers to vectors of length N (node order of the header), BORROWED
 *  until the next rbs_set_rhs_terms / rbs_set_rhs_constant / operator change.  R = 0
 *  returns to the constant right-hand side.  The next rbs_load_basis (required: the
 *  basis state is invalidated) packs the terms into the basis storage (its size grows by
 *  N8 (round8(R)+4) doubles) and computes the offline f_{N,r} = W^T f_r and the Gram
 *  matrix f_r^T f_s.  rbs_solve_batch with rhs_dev == NULL then forms f(mu_b) on the
 *  device (one pass over the packed terms), f_N(mu) = sum_r phi_r f_{N,r} and
 *  ||f(mu)||^2 = phi^T G phi without any N-length projection.  phi(mu) comes from the
 *  parameter map (rbs_set_param_map; default: all ones).  Not with mesh slabs.
 *  The operator change and rbs_build_greedy* drop the terms.
 *  Errors: RBS_E_STATE (no operator), RBS_E_DIM (R > RBS_MAX_R), RBS_E_ARG (NULL pointer),
 *  RBS_E_UNSUPPORTED (mesh slabs). */
rbs_status rbs_set_rhs_terms(rbs_ctx* ctx, int R, const double* const* f_dev);

/* Parameter map (theta_q(mu), phi_r(mu)), affine in the P parameters:
 *   theta_q(mu) = theta_aff[q][0] + sum_p theta_aff[q][p+1] mu_p   (Q x (P+1), row-major)
 *   phi_r(mu)   = phi_aff[r][0]   + sum_p phi_aff[r][p+1]   mu_p   (R x (P+1), row-major)
 * theta_aff NULL = identity (P == Q); phi_aff NULL = all ones.  Set after rbs_set_rhs_terms
 * (new terms drop phi_aff).  From then on mu_host of rbs_solve_batch is B x P.  A
 * non-affine dependence is written with derived parameters (e.g. Case 2 of PAPER.md
 * Table 1: mu' = (mu_1, mu_2, mu_1 mu_2), DESIGN.md AMB-23).  Copied (not borrowed).
 * Errors: RBS_E_STATE (no operator; phi_aff without terms), RBS_E_DIM (P out of range or
 * identity with P != Q), RBS_E_ARG (non-finite entries). */
rbs_status rbs_set_param_map(rbs_ctx* ctx, int P, const double* theta_aff, const double* phi_aff);

/* Cell-label operator: cell (a,b[,c]) (a,b,c in 0..m, x fastest) carries
 * label cell_label_dev[a + (m+1)(b + (m+1)c)] in 0..Q-1; A(theta) is the cell-averaged
 * stencil with kappa_cell = theta_label(cell) (AMB-1).  Realised as the face operator of
 * rbs_set_operator_faces (DESIGN.md AMB-24): a face's coefficient for term q is the
 * fraction of its 2^(dim-1) cells labelled q, written by a device kernel into
 * faces_storage_dev (caller-owned, RETAINED as the face operator; size from
 * rbs_operator_labels_size = Q dim (m+1) m^(dim-1) doubles).  labels are read once
 * (borrowed for the call).  Synchronises `stream`.  Q <= 255.
 * Errors: RBS_E_ARG (NULL), RBS_E_DIM, RBS_E_NOMEM (storage too small), RBS_E_CUDA. */
rbs_status rbs_operator_labels_size(int dim, int64_t m, int Q, size_t* bytes);
rbs_status rbs_set_operator_labels(rbs_ctx* ctx, int dim, int64_t m, int Q, const uint8_t* cell_label_dev,
                                   void* faces_storage_dev, size_t storage_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Basis W (N x n, orthonormal columns) and offline blocks
 * A_{n,q} = W^T A_q W, f_{n,1} = W^T f_1 (eq12c).
 *
 * rbs_basis_storage_size: device bytes the context needs to keep W (in the
 *   internal node-major padded layout) and the offline blocks.
 * rbs_load_basis: copies W_dev (column-major, leading dimension ldw >= N,
 *   borrowed) into storage_dev (caller-owned, RETAINED until the next
 *   load/destroy).  ANq_host (Q x n x n row-major) / fn_host (n) may be NULL,
 *   then they are computed on the device from W (stencil applications +
 *   projections); otherwise they are copied.  Synchronises `stream`.
 *   1 <= n <= RBS_MAX_N (n = 0 allowed: empty basis, RBCG = SGS-PCG).
 *   Errors: RBS_E_STATE (no operator), RBS_E_DIM, RBS_E_NOMEM, RBS_E_CUDA.
 * rbs_get_offline_blocks: copies the blocks in use to host (Q*n*n, n).
 */
rbs_status rbs_basis_storage_size(const rbs_ctx* ctx, int n, size_t* bytes);
rbs_status rbs_load_basis(rbs_ctx* ctx, int n, const double* W_dev, int64_t ldw,
                          const double* ANq_host, const double* fn_host,
                          void* storage_dev, size_t storage_bytes, void* stream);
rbs_status rbs_get_offline_blocks(const rbs_ctx* ctx, double* ANq_host, double* fn_host);

/* ---------------------------------------------------------------------------
 * Batched online solve (RBI: algorithm1; RBCG: PAPER.md:
 * 260-279 algorithm2) of B queries against the loaded basis.
 */
typedef struct {
    int method;          /* RBS_RBI | RBS_RBCG (default RBCG) */
    double tol;          /* relative residual ||r||/||f|| (default 1e-10, AMB-7) */
    int max_iter;        /* default 20000 (RBCG) -- RBI callers set e.g. 500000 */
    int smoother;        /* RBS_SMOOTH_SYM_RBGS (default) | RBS_SMOOTH_FWD_RBGS (AMB-5/6) |
                            RBS_SMOOTH_JACOBI */
    int sweeps;          /* nu >= 0 (default 1); 0 = no smoothing (Lemma 2 tests) */
    double delta;        /* PRECOND threshold (default 1e-12, AMB-11) */
    int record_history;  /* 1: fill history[B][max_iter+1] */
    int x_location;      /* RBS_MEM_DEVICE (default) | RBS_MEM_HOST for X */
    int graph_chunk;     /* iterations per captured CUDA graph (default 16, even) */
    int profile;         /* 1: launch eagerly (no graph) with CUDA events around every
                            kernel; per-class times via rbs_last_profile (default 0) */
    int n_active;        /* active RB dimension: the leading n_active columns of W are used
                            (0 = all; the iterations-vs-n study).  The
                            reduced solve then uses the leading block of the Cholesky factor
                            (nested spaces, DESIGN.md AMB-19). */
    double gamma;        /* RBCG only, 0 = off: the adaptive-n rule of PAPER.md:287 -- after
                            each x-update, if ||r_k|| / ||r_{k+1}|| < gamma the active
                            dimension grows by one (capped at n) for the next preconditioner
                            application; start value n_active.  Final values: rbs_last_n_active */
    double omega;        /* Jacobi damping, 0 < omega < 2 (default 1); ignored by Gauss-Seidel */
    int precond;         /* RBCG preconditioner (NEXT(3)): RBS_PRECOND_POST
                            (default: the paper's RBI(A, r, W, 1), post-smoothing only) or
                            RBS_PRECOND_SYM: y1 = S*(A, r, 0) (the adjoint sweep: colour
                            sequence reversed), y2 = y1 + W A_n^{-1} W^T (r - A y1),
                            y = S(A, r, y2) -- a symmetric positive definite M^{-1}, so CG's
                            theory holds (DESIGN.md AMB-25).  a_n then reports the first coarse
                            correction.  Flat (non-march) kernels; not with mesh slabs. */
    int beta_rule;       /* RBCG: RBS_BETA_FR (default, beta = y_{k+1}^T r_{k+1} / y_k^T r_k as
                            printed) or RBS_BETA_PR (Polak-Ribiere / flexible:
                            y_{k+1}^T (r_{k+1} - r_k) / y_k^T r_k); flat kernels, not with slabs */
} rbs_solve_opts;
enum { RBS_PRECOND_POST = 0, RBS_PRECOND_SYM = 1 };
enum { RBS_BETA_FR = 0, RBS_BETA_PR = 1 };

void rbs_default_opts(rbs_solve_opts* opts);

/* Device workspace bytes for a batch of B queries with these options. */
rbs_status rbs_solve_workspace_size(const rbs_ctx* ctx, int B, const rbs_solve_opts* opts,
                                    size_t* bytes);

/*
 * rbs_solve_batch:
 *  B         1..RBS_MAX_BATCH queries.
 *  mu_host   B x P host array: theta_q = mu_q (P = Q) or, after rbs_set_param_map,
 *            theta(mu) and phi(mu) of the map.  Values outside the
 *            sampling box are accepted; A(mu) must be SPD for convergence.
 *  rhs_dev   NULL (use f of rbs_set_rhs_terms, else of rbs_set_rhs_constant) or a
 *            B x N device array of per-query right-hand sides (e.g. Lemma-1 tests).
 *  X         B x N output (device, or host when opts->x_location == HOST).
 *  iters, qstatus, relres (last recurrence/true residual ratio), true_relres
 *            (||f - A x||/||f|| recomputed after exit): host arrays of B
 *            (any may be NULL).
 *  a_n       host B x n: reduced coefficients of the first RB correction
 *            (x_hat = W a_n) or NULL.
 *  history   host B x (max_iter+1) relative residuals, NaN-padded; requires
 *            opts->record_history (else ignored; may be NULL).
 *  workspace_dev / workspace_bytes: >= rbs_solve_workspace_size.
 *  Synchronises `stream` before returning.
 *  Errors: RBS_E_STATE (no basis), RBS_E_DIM, RBS_E_ARG, RBS_E_NOMEM, RBS_E_CUDA.
 */
rbs_status rbs_solve_batch(rbs_ctx* ctx, int B, const double* mu_host, const rbs_solve_opts* opts,
                           const double* rhs_dev, double* X, int* iters, int* qstatus,
                           double* relres, double* true_relres, double* a_n, double* history,
                           void* workspace_dev, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Mesh-slab partition of one 3D system.
 * rbs_set_virtual_slabs: split the z-planes 1..m into G slabs (sizes balanced
 *   to within one; slab s owns planes [z0, z1) as paper_1804_06363_b200/dist.py
 *   slab_partition) and run every following rbs_solve_batch slab by slab in
 *   this process: each slab keeps its own batch vectors over its owned planes
 *   plus H ghost planes per side (H = half-sweeps of the smoother), the per-CTA
 *   partial sums of all slabs are combined in a fixed order, and the ghost
 *   planes are refreshed by device copies (r: H planes after the residual pass,
 *   y: 1 plane after the smoother).  G = 1 switches it off.  RBCG only; results
 *   agree with the unpartitioned solve to rounding (the sum order differs).
 *   Errors: RBS_E_STATE (no operator), RBS_E_UNSUPPORTED (2D), RBS_E_DIM (a slab
 *   with fewer than 4 planes).  Invalidates the captured iteration graph.
 */
rbs_status rbs_set_virtual_slabs(rbs_ctx* ctx, int G);

/* Mesh slabs over ranks (one process per GPU, NCCL over NVLink):
 * rbs_nccl_unique_id: write an NCCL unique id (128 bytes) into id_out (rank 0;
 *   the caller distributes it, e.g. with torch.distributed).  Errors: RBS_E_ARG.
 * rbs_dist_init: after rbs_set_operator_blocks (3D), join the communicator as
 *   `rank` of `nranks`; this rank then owns planes [z0, z1) of the slab
 *   partition (balanced to within one plane) and stores `ghost` planes per side
 *   (>= the smoother's half-sweeps; 3 for the default symmetric sweep).  From
 *   then on every N-length buffer of this context is rank-local: the basis
 *   passed to rbs_load_basis is the rows of the STORED planes [g0, g1)
 *   (rbs_local_range), with the offline blocks of the full basis passed on the
 *   host (required); X returned by rbs_solve_batch is [B][owned nodes].  Every
 *   rank calls rbs_solve_batch with the same mu list (collective).  Per RBCG
 *   iteration: grouped ncclSend/ncclRecv of ghost planes with the neighbours
 *   and three ncclAllReduce(sum) of [B]-, [B][n+1]- and [B][2]-sized partials.
 *   Errors: RBS_E_STATE, RBS_E_UNSUPPORTED (2D), RBS_E_DIM (slabs too thin),
 *   RBS_E_CUDA (NCCL failure, detail in rbs_last_error).
 * rbs_local_range: this context's owned [z0, z1) and stored [g0, g1) planes and
 *   the node counts (full grid when not distributed).
 */
rbs_status rbs_nccl_unique_id(void* id_out, size_t bytes);
rbs_status rbs_dist_init(rbs_ctx* ctx, const void* nccl_id, int nranks, int rank, int ghost);
rbs_status rbs_local_range(const rbs_ctx* ctx, int64_t* z0, int64_t* z1, int64_t* g0, int64_t* g1,
                           int64_t* n_stored, int64_t* n_owned);

/* Query sharding over ranks: every rank keeps the full
 * grid and solves its own queries with no collective on the hot path.
 * rbs_comm_init: join an NCCL communicator (id from rbs_nccl_unique_id on one rank,
 *   distributed by the caller) without changing the geometry.  Errors: RBS_E_ARG,
 *   RBS_E_STATE (a mesh-slab context), RBS_E_CUDA (NCCL failure, detail in rbs_last_error).
 * rbs_broadcast_basis: collective; the packed W, the offline blocks A_{n,q} and f_n
 *   (eq12c) go from `root` to every rank by one ncclBroadcast of the
 *   storage prefix that holds them.  root: the basis of dimension n must be loaded
 *   (storage_dev ignored); other ranks: storage_dev (caller-owned, >=
 *   rbs_basis_storage_size(n), RETAINED) becomes their basis storage, the host copies of
 *   the blocks are rebuilt from it, and affine rhs terms (rbs_set_rhs_terms, set on every
 *   rank) get their offline quantities locally.  Synchronises `stream`.
 *   Errors: RBS_E_STATE (no communicator; root without that basis), RBS_E_ARG, RBS_E_DIM,
 *   RBS_E_NOMEM, RBS_E_CUDA (NCCL failure). */
rbs_status rbs_comm_init(rbs_ctx* ctx, const void* nccl_id, int nranks, int rank);
rbs_status rbs_broadcast_basis(rbs_ctx* ctx, int root, int n, void* storage_dev, size_t storage_bytes,
                               void* stream);

/* Active RB dimension of every query at the end of the last rbs_solve_batch
 * (host array of B; n unless opts.n_active / opts.gamma were used). */
rbs_status rbs_last_n_active(const rbs_ctx* ctx, int* n_active_host);

/* Number of kernel launches issued by the last rbs_solve_batch (instrumentation). */
int64_t rbs_last_launch_count(const rbs_ctx* ctx);

/* Kernel classes of the iteration body and their per-class device time (ms,
 * CUDA events on the launching stream) and launch counts, accumulated over the
 * complete iterations of the last rbs_solve_batch run with opts.profile = 1.
 * ms_total / launches: host arrays of RBS_K_NCLASS. */
enum { RBS_K_CGP = 0, RBS_K_ALPHA = 1, RBS_K_PROJ = 2, RBS_K_REDUCE_SOLVE = 3, RBS_K_PROLONG = 4,
       RBS_K_GS = 5, RBS_K_BETA = 6, RBS_K_NCLASS = 7 };
rbs_status rbs_last_profile(const rbs_ctx* ctx, double* ms_total, int64_t* launches);
const char* rbs_kernel_class_name(int k);

/* ---------------------------------------------------------------------------
 * Offline greedy build (algorithm0; adaptive: PAPER.md:294-308
 * algorithm3, snapshots by RBCG with W_{N-1}; DESIGN.md AMB-13).
 *  mu_train_host  n_train x P (host).  mu_1 = mu_train[0].
 *  W_out_dev      column-major N x n_max device array (caller-owned).
 *  ANq_host_out   Q x n_max x n_max (row stride n_max) offline blocks or NULL.
 *  fn_host_out    n_max or NULL.
 *  selected, indicator, snap_iters: host arrays of n_max (may be NULL).
 *  Snapshot solve: RBCG, relative tolerance snapshot_tol; MGS with one
 *  re-orthogonalisation, reject if ||w|| < drop_tol ||x||.
 * The context's basis state is replaced by the built basis (held in
 * workspace_dev, which is RETAINED like storage_dev of rbs_load_basis).
 */
rbs_status rbs_greedy_workspace_size(const rbs_ctx* ctx, int n_train, int n_max, size_t* bytes);
rbs_status rbs_build_greedy(rbs_ctx* ctx, int n_train, const double* mu_train_host, int n_max,
                            int mode, double snapshot_tol, double drop_tol, double* W_out_dev,
                            double* ANq_host_out, double* fn_host_out, int* n_out, int* selected,
                            double* indicator, int* snap_iters, int* n_rejected,
                            void* workspace_dev, size_t workspace_bytes, void* stream);

/* rbs_build_greedy_affine: the same greedy for affine right-hand sides
 * f(mu_t) = sum_r phi_train_host[t*R + r] f_r (terms_dev [R][N], device, borrowed;
 * see rbs_affine_rhs): snapshots solve A(mu) x = f(mu); the offline vectors are
 * f_{N,r} = W^T f_r, returned in fnr_host_out [R][n_max]; the indicator solves use
 * f_N(mu_t) = sum_r phi_r(mu_t) f_{N,r}.  Later solves must pass rhs_dev (the
 * context's constant right-hand side does not describe this problem).  1 <= R <=
 * RBS_MAX_R; other arguments, workspace and errors as rbs_build_greedy. */
rbs_status rbs_build_greedy_affine(rbs_ctx* ctx, int n_train, const double* mu_train_host, int R,
                                   const double* phi_train_host, const double* terms_dev, int n_max,
                                   int mode, double snapshot_tol, double drop_tol, double* W_out_dev,
                                   double* ANq_host_out, double* fnr_host_out, int* n_out, int* selected,
                                   double* indicator, int* snap_iters, int* n_rejected,
                                   void* workspace_dev, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RBS_H */
