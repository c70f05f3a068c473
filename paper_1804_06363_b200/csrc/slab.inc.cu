// slab.inc.cu -- mesh-slab partition of one 3D system,
// included by api.cu.
//
// The z-planes 1..m are split into G slabs (dist.py slab_partition: planes
// balanced to within one).  Slab s owns planes [z0, z1) and stores [g0, g1) =
// the owned planes plus H ghost planes per side (H = the smoother's half-sweep
// count, >= 1).  Every N-length batch vector of a slab is a node-major
// [planes x m^2][Bp] array over the stored planes; W is shared (the slab's rows
// of the full basis are contiguous).  One RBCG iteration:
//   K1 p = y + beta p, sigma partials (owned planes)   -> k_slab_alpha (Step 5)
//   K2 x += alpha p, r -= alpha A p, ||r||^2, W^T r    -> k_reduce_solve (Steps 6-9)
//   halo: r on H planes per side (the smoother's dependency cone)
//   K3 y0 = W e, H half-sweeps on the stored planes, y^T r / y^T y partials
//                                                      -> k_slab_beta (Step 10)
//   halo: y on 1 plane per side (K1 forms p on the first ghost plane)
// Two transports share these passes:
//  * virtual slabs (rbs_set_virtual_slabs): all slabs in one process; the
//    partials of all slabs land in one column range each of the shared partial
//    arrays and are summed in a fixed order; halos are device copies;
//  * ranks (rbs_dist_init): one slab per GPU; before each scalar step the rank's
//    columns are summed (k_reduce_rows) and ncclAllReduce'd over NVLink (three
//    small allreduces per iteration: sigma, [W^T r, ||r||^2], [y^T r, y^T y]),
//    halos are grouped ncclSend/ncclRecv of whole planes with the neighbours.
namespace {

struct Slab {
    Geo g;
    int z0, z1, g0, g1;      // owned [z0, z1), stored [g0, g1) global planes
    int64_t N8;
    int nct, nctf;           // CTAs of the projection / flat passes
    int colP, colF;          // first partial column
    double *X, *R, *P0, *P1, *Y;
    const double* W;
};

struct SlabPlan {
    std::vector<Slab> sl;
    int H = 1, totP = 0, totF = 0;
    SolveLayout L{};         // the shared small arrays (vectors unused)
    double *colP = nullptr, *colF = nullptr;   // ranks: this rank's column sums (allreduced)
    size_t bytes = 0;
};

// slab s of G: the same partition as paper_1804_06363_b200/dist.py slab_partition
void slab_range(int m, int G, int s, int& z0, int& z1) {
    const int base = m / G, extra = m % G;
    const int start = s * base + std::min(s, extra);
    z0 = start + 1;
    z1 = z0 + base + (s < extra ? 1 : 0);
}

SlabPlan slab_plan(const rbs_ctx* c, int B, const rbs_solve_opts* o, void* base) {
    SlabPlan P;
    const Geo& g = c->gglob;
    const int G = c->dist ? 1 : c->nslab, Bp = pow2_batch(B), m = g.m;
    P.H = c->dist ? c->dH : std::max<int>(1, (int)color_seq(o->smoother, o->sweeps).size());
    const int64_t plane = (int64_t)m * m;
    Carve cv(base);
    P.sl.resize(G);
    for (int s = 0; s < G; ++s) {
        Slab& q = P.sl[s];
        if (c->dist) {
            q.z0 = c->dz0; q.z1 = c->dz1; q.g0 = c->dg0; q.g1 = c->dg1;
        } else {
            slab_range(m, G, s, q.z0, q.z1);
            q.g0 = std::max(1, q.z0 - P.H);
            q.g1 = std::min(m + 1, q.z1 + P.H);
        }
        q.g = g;
        q.g.kofs = q.g0 - 1;
        q.g.mz = q.g1 - q.g0;
        q.g.own_lo = q.z0 - q.g0;
        q.g.own_hi = q.z1 - q.g0;
        q.g.N = plane * q.g.mz;
        q.N8 = round_up(q.g.N, 8);
        q.nct = proj_ctas(q.g);
        q.nctf = flat_ctas(q.g);
        q.colP = P.totP;
        q.colF = P.totF;
        P.totP += q.nct;
        P.totF += q.nctf;
        const size_t vec = (size_t)q.N8 * Bp;
        q.X = cv.take<double>(vec);
        q.R = cv.take<double>(vec);
        q.P0 = cv.take<double>(vec);
        q.P1 = cv.take<double>(vec);
        q.Y = cv.take<double>(vec);
        // virtual: rows of the full basis; ranks: the loaded basis is this slab's rows
        q.W = c->Wi ? (c->dist ? c->Wi : c->Wi + (size_t)(q.g0 - 1) * plane * c->ldw) : nullptr;
    }
    // shared small arrays (SolveState); partial arrays sized for all slabs' columns
    const int npad = c->npad;
    SolveLayout& L = P.L;
    L.Xout = o->x_location == RBS_MEM_HOST ? cv.take<double>((size_t)B * g.N) : nullptr;
    L.theta = cv.take<double>((size_t)g.Q * Bp);
    L.fproj = cv.take<double>((size_t)Bp * (npad + 1));
    L.L = cv.take<double>((size_t)Bp * npad * npad + 8);
    L.Ainv = cv.take<double>((size_t)Bp * npad * npad + 8);
    L.E = cv.take<double>((size_t)std::max(npad, 8) * Bp);
    L.a_n = cv.take<double>((size_t)Bp * npad + 8);
    L.partP = cv.take<double>((size_t)Bp * (npad + 1) * P.totP);
    L.partF = cv.take<double>((size_t)Bp * 2 * P.totF);
    L.alpha = cv.take<double>(Bp);
    L.beta = cv.take<double>(Bp);
    L.rho = cv.take<double>(Bp);
    L.rr = cv.take<double>(Bp);
    L.fnorm = cv.take<double>(Bp);
    L.relres = cv.take<double>(Bp);
    L.hist = o->record_history ? cv.take<double>((size_t)Bp * (o->max_iter + 1)) : nullptr;
    L.active = cv.take<int>(Bp);
    L.status = cv.take<int>(Bp);
    L.its = cv.take<int>(Bp);
    L.pivot = cv.take<int>(Bp);
    L.ints = cv.take<int>(8);
    L.na = cv.take<int>(Bp);
    P.colP = cv.take<double>((size_t)Bp * (npad + 1) + 8);
    P.colF = cv.take<double>((size_t)Bp * 2 + 8);
    P.bytes = cv.off + 256;
    return P;
}

}  // namespace

// ---------------------------------------------------------------------------
extern "C" rbs_status rbs_set_virtual_slabs(rbs_ctx* ctx, int G) {
    if (!ctx) return RBS_E_ARG;
    ctx->err.clear();
    if (!ctx->has_op) return fail(ctx, RBS_E_STATE, "set the operator first");
    if (G < 1) return fail(ctx, RBS_E_ARG, "G must be >= 1");
    if (G > 1 && ctx->g.dim != 3) return fail(ctx, RBS_E_UNSUPPORTED, "mesh slabs need a 3D operator");
    if (G > 1 && ctx->g.m / G < 4) return fail(ctx, RBS_E_DIM, "each slab needs >= 4 owned planes");
    ctx->nslab = G;
    if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; ctx->gkey.clear(); }
    return RBS_OK;
}

extern "C" rbs_status rbs_nccl_unique_id(void* id_out, size_t bytes) {
    if (!id_out || bytes < sizeof(ncclUniqueId)) return RBS_E_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return RBS_E_CUDA;
    std::memcpy(id_out, &id, sizeof id);
    return RBS_OK;
}

extern "C" rbs_status rbs_dist_init(rbs_ctx* ctx, const void* nccl_id, int nranks, int rank, int ghost) {
    if (!ctx || !nccl_id) return RBS_E_ARG;
    ctx->err.clear();
    if (!ctx->has_op) return fail(ctx, RBS_E_STATE, "set the operator first");
    const Geo gg = ctx->gglob;
    if (gg.dim != 3) return fail(ctx, RBS_E_UNSUPPORTED, "mesh slabs need a 3D operator");
    if (nranks < 1 || rank < 0 || rank >= nranks || ghost < 1) return fail(ctx, RBS_E_ARG, "bad nranks/rank/ghost");
    if (gg.m / nranks < std::max(4, ghost)) return fail(ctx, RBS_E_DIM, "a slab would own too few planes");
    CK(cudaSetDevice(ctx->device));
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof id);
    if (ctx->comm) { ncclCommDestroy(ctx->comm); ctx->comm = nullptr; }
    ncclResult_t r = ncclCommInitRank(&ctx->comm, nranks, id, rank);
    if (r != ncclSuccess) return fail(ctx, RBS_E_CUDA, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    int z0, z1;
    slab_range(gg.m, nranks, rank, z0, z1);
    ctx->nranks = nranks; ctx->rank = rank; ctx->dH = ghost;
    ctx->dz0 = z0; ctx->dz1 = z1;
    ctx->dg0 = std::max(1, z0 - ghost);
    ctx->dg1 = std::min(gg.m + 1, z1 + ghost);
    // the context's geometry becomes the rank's stored planes: basis rows, vectors
    Geo lg = gg;
    lg.kofs = ctx->dg0 - 1;
    lg.mz = ctx->dg1 - ctx->dg0;
    lg.own_lo = z0 - ctx->dg0;
    lg.own_hi = z1 - ctx->dg0;
    lg.N = (int64_t)gg.m * gg.m * lg.mz;
    ctx->g = lg;
    ctx->N8 = round_up(lg.N, 8);
    ctx->dist = true;
    ctx->nslab = 1;
    ctx->has_basis = false;
    if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; ctx->gkey.clear(); }
    return RBS_OK;
}

// Query sharding: a communicator over the ranks without any change of
// geometry -- every rank keeps the full grid and solves its own queries; the only
// collective is rbs_broadcast_basis (off the hot path).
extern "C" rbs_status rbs_comm_init(rbs_ctx* ctx, const void* nccl_id, int nranks, int rank) {
    if (!ctx || !nccl_id) return RBS_E_ARG;
    ctx->err.clear();
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(ctx, RBS_E_ARG, "bad nranks/rank");
    if (ctx->dist) return fail(ctx, RBS_E_STATE, "context is a mesh slab (rbs_dist_init)");
    CK(cudaSetDevice(ctx->device));
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof id);
    if (ctx->comm) { ncclCommDestroy(ctx->comm); ctx->comm = nullptr; }
    const ncclResult_t r = ncclCommInitRank(&ctx->comm, nranks, id, rank);
    if (r != ncclSuccess) return fail(ctx, RBS_E_CUDA, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    ctx->nranks = nranks;
    ctx->rank = rank;
    ctx->qcomm = true;
    return RBS_OK;
}

// W (packed), the offline blocks A_{n,q} and f_n from `root` to every rank: one
// ncclBroadcast of the storage prefix that holds them (basis_layout: Wi, then ANq, f_n).
// Non-root ranks adopt `storage_dev` as their basis storage and rebuild the host copies;
// affine rhs terms (set on every rank) get their offline quantities locally.
extern "C" rbs_status rbs_broadcast_basis(rbs_ctx* ctx, int root, int n, void* storage_dev,
                                          size_t storage_bytes, void* stream) {
    if (!ctx) return RBS_E_ARG;
    ctx->err.clear();
    if (!ctx->comm || !ctx->qcomm) return fail(ctx, RBS_E_STATE, "no query communicator (rbs_comm_init)");
    if (root < 0 || root >= ctx->nranks) return fail(ctx, RBS_E_ARG, "bad root");
    if (n < 0 || n > RBS_MAX_N) return fail(ctx, RBS_E_DIM, "n out of range");
    const bool is_root = ctx->rank == root;
    if (is_root && (!ctx->has_basis || ctx->n != n)) return fail(ctx, RBS_E_STATE, "root: load the basis (dimension n) first");
    BasisLayout L = basis_layout(ctx, n, is_root ? (void*)ctx->Wi : storage_dev);
    if (!is_root && (!storage_dev || storage_bytes < L.bytes)) return fail(ctx, RBS_E_NOMEM, "storage too small");
    CK(cudaSetDevice(ctx->device));
    const cudaStream_t st = (cudaStream_t)stream;
    const int npad = (int)round_up(n, 8), Q = ctx->g.Q;
    const size_t count = (size_t)(L.ANq - L.Wi) + (size_t)Q * npad * npad + npad;   // doubles
    const ncclResult_t r = ncclBroadcast(L.Wi, L.Wi, count, ncclDouble, root, ctx->comm, st);
    if (r != ncclSuccess) return fail(ctx, RBS_E_CUDA, std::string("ncclBroadcast(basis): ") + ncclGetErrorString(r));
    CK(cudaStreamSynchronize(st));
    if (!is_root) {
        if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; ctx->gkey.clear(); }
        ctx->n = n;
        ctx->npad = npad;
        ctx->ldw = w_ld(npad);
        ctx->Wi = L.Wi;
        ctx->dANq = L.ANq;
        ctx->scratch = L.Z;
        std::vector<double> pad((size_t)Q * npad * npad + npad);
        CK(cudaMemcpy(pad.data(), L.ANq, pad.size() * 8, cudaMemcpyDeviceToHost));
        ctx->hANq.assign((size_t)Q * n * n, 0.0);
        ctx->hfn.assign(n, 0.0);
        for (int q = 0; q < Q; ++q)
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j)
                    ctx->hANq[((size_t)q * n + i) * n + j] = pad[((size_t)q * npad + i) * npad + j];
        for (int j = 0; j < n; ++j) ctx->hfn[j] = pad[(size_t)Q * npad * npad + j];
        if (rbs_status ts = terms_offline(ctx, L, st); ts != RBS_OK) return ts;
        ctx->has_basis = true;
    }
    return RBS_OK;
}

extern "C" rbs_status rbs_local_range(const rbs_ctx* c, int64_t* z0, int64_t* z1, int64_t* g0, int64_t* g1,
                                      int64_t* n_stored, int64_t* n_owned) {
    if (!c) return RBS_E_ARG;
    const Geo& gg = c->gglob;
    const int64_t plane = gg.dim == 3 ? (int64_t)gg.m * gg.m : (int64_t)gg.m;
    const int a0 = c->dist ? c->dz0 : 1, a1 = c->dist ? c->dz1 : gg.m + 1;
    const int b0 = c->dist ? c->dg0 : 1, b1 = c->dist ? c->dg1 : gg.m + 1;
    if (z0) *z0 = a0;
    if (z1) *z1 = a1;
    if (g0) *g0 = b0;
    if (g1) *g1 = b1;
    if (n_stored) *n_stored = (int64_t)(b1 - b0) * plane;
    if (n_owned) *n_owned = (int64_t)(a1 - a0) * plane;
    return RBS_OK;
}

namespace {

rbs_status solve_slabs(rbs_ctx* ctx, int B, const double* mu_host, const rbs_solve_opts* o, double* X,
                       int* iters, int* qstatus, double* relres, double* true_relres, double* a_n,
                       double* history, void* workspace_dev, size_t workspace_bytes, cudaStream_t st) {
    if (o->method != RBS_RBCG) return fail(ctx, RBS_E_UNSUPPORTED, "mesh slabs: RBCG only");
    if (o->profile) return fail(ctx, RBS_E_UNSUPPORTED, "mesh slabs: no profile mode");
    SlabPlan P = slab_plan(ctx, B, o, workspace_dev);
    if (workspace_bytes < slab_plan(ctx, B, o, nullptr).bytes)
        return fail(ctx, RBS_E_NOMEM, "workspace too small");
    for (const Slab& q : P.sl)
        if (q.z1 - q.z0 < P.H) return fail(ctx, RBS_E_DIM, "a slab owns fewer planes than the halo depth");
    const Geo& g = ctx->gglob;
    const bool dist = ctx->dist;
    if (dist && P.H < (int)color_seq(o->smoother, o->sweeps).size())
        return fail(ctx, RBS_E_UNSUPPORTED, "mesh slabs over ranks: more half-sweeps than ghost planes");
    const int Bp = pow2_batch(B), lgB = ilog2(Bp), n = ctx->n, npad = ctx->npad, Q = g.Q;
    const int G = (int)P.sl.size();
    const int64_t plane = (int64_t)g.m * g.m;
    SolveLayout& L = P.L;
    int64_t launches = 0;
    // NCCL calls are enqueued inside lambdas (and inside graph capture): the first
    // failure is kept here and turned into RBS_E_CUDA (with ncclGetErrorString)
    ncclResult_t nres = ncclSuccess;
    std::string nwhere;
    auto nck = [&](ncclResult_t r, const char* what) {
        if (r != ncclSuccess && nres == ncclSuccess) { nres = r; nwhere = what; }
    };
    auto nfail = [&]() {
        return fail(ctx, RBS_E_CUDA, nwhere + ": " + ncclGetErrorString(nres));
    };

    std::vector<double> th((size_t)Q * Bp, 1.0);
    for (int b = 0; b < B; ++b)
        for (int q = 0; q < Q; ++q) th[(size_t)q * Bp + b] = mu_host[(size_t)b * Q + q];
    CK(cudaMemcpyAsync(L.theta, th.data(), th.size() * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(L.ints, 0, 8 * sizeof(int), st));
    int* kcount = L.ints;
    int* done = L.ints + 1;
    unsigned* ticket = (unsigned*)(L.ints + 2);
    CK(cudaMemsetAsync(L.E, 0, (size_t)std::max(npad, 8) * Bp * 8, st));
    CK(cudaMemsetAsync(L.a_n, 0, ((size_t)Bp * npad + 8) * 8, st));
    if (L.hist) CK(cudaMemsetAsync(L.hist, 0xFF, (size_t)Bp * (o->max_iter + 1) * 8, st));
    {
        std::vector<double> fp((size_t)Bp * (npad + 1), 0.0);
        for (int b = 0; b < Bp; ++b) {
            for (int j = 0; j < n; ++j) fp[(size_t)b * (npad + 1) + j] = ctx->fconst * ctx->hfn[j];
            fp[(size_t)b * (npad + 1) + npad] = ctx->fconst * ctx->fconst * (double)g.N;
        }
        CK(cudaMemcpyAsync(L.fproj, fp.data(), fp.size() * 8, cudaMemcpyHostToDevice, st));
    }
    for (Slab& q : P.sl) {
        const int64_t vecN = q.N8 * Bp;
        CK(cudaMemsetAsync(q.X, 0, vecN * 8, st));
        CK(cudaMemsetAsync(q.P0, 0, vecN * 8, st));
        CK(cudaMemsetAsync(q.P1, 0, vecN * 8, st));
        k_fill_batch<<<grid_for(vecN, 256, ctx->num_sms * 8), 256, 0, st>>>(q.R, q.g.N, q.N8, Bp, B, nullptr,
                                                                            ctx->fconst);
        CKL();
        ++launches;
    }
    SolveState S{};
    S.B = B; S.Bp = Bp; S.n = n; S.npad = npad; S.nct = P.totP; S.nctf = P.totF;
    S.maxit = o->max_iter; S.method = 1; S.tol = o->tol; S.delta = o->delta;
    S.ANq = ctx->dANq; S.Q = Q; S.theta = L.theta; S.fproj = L.fproj; S.L = L.L; S.Ainv = L.Ainv; S.E = L.E;
    S.a_n = L.a_n; S.partP = L.partP; S.partF = L.partF; S.alpha = L.alpha; S.beta = L.beta;
    S.rho = L.rho; S.rr = L.rr; S.fnorm = L.fnorm; S.relres = L.relres; S.active = L.active;
    S.status = L.status; S.its = L.its; S.pivot = L.pivot; S.kcount = kcount; S.done = done;
    S.ticket = ticket; S.hist = L.hist;
    set_active_dim(S, L.na, o, n);
    k_setup_reduced<<<Bp, 128, 0, st>>>(S, 0);
    CKL();
    ++launches;

    const std::vector<int> seq = color_seq(o->smoother, o->sweeps);
    const size_t fsm = flat_smem(g, Bp);
    const size_t psm = proj_smem(g, Bp, npad);
    // ---- passes over all slabs --------------------------------------------------
    auto k1 = [&](int it) {   // p = y + beta p, sigma partials; then Step 5
        int c = 0;
        for (Slab& q : P.sl) {
            CGPArgs a{};
            a.g = q.g; a.Bp = Bp; a.lgB = lgB; a.NB = q.g.N * Bp; a.theta = L.theta; a.active = L.active;
            a.beta = L.beta; a.Y = q.Y; a.Pold = (it & 1) ? q.P1 : q.P0; a.Pnew = (it & 1) ? q.P0 : q.P1;
            a.s = S; a.done = done; a.col0 = q.colF; a.ext = 1;
            if (Bp <= 32 && !q.g.faces) {     // stream p_new, then sigma in row segments (kernels.cuh)
                const int64_t nb2 = (int64_t)q.g.N * Bp / 2;
                k_pnew3<<<(unsigned)std::min<int64_t>((nb2 + 255) / 256, (int64_t)ctx->num_sms * 16), 256, 0,
                          st>>>(a.Y, a.Pold, a.Pnew, a.beta, a.active, nb2, Bp, a.done);
                k_sigma3r<4, false><<<q.nctf, kFlat, fsm, st>>>(a);
                ++c;
            } else {
                k_cgp<3><<<q.nctf, kFlat, fsm, st>>>(a);
            }
            ++c;
        }
        if (dist) {   // rank sum of the columns, allreduce over the ranks, Step 5
            SolveState S1 = S;
            S1.partF = P.colF;
            S1.nctf = 1;
            k_reduce_rows<<<Bp, 128, 0, st>>>(L.partF, 2, P.totF, P.colF);
            nck(ncclAllReduce(P.colF, P.colF, (size_t)Bp * 2, ncclDouble, ncclSum, ctx->comm, st),
                "ncclAllReduce(sigma)");
            k_slab_alpha<<<1, 512, 0, st>>>(S1, 1);
            return c + 2;
        }
        k_slab_alpha<<<1, 512, 0, st>>>(S, P.totF);
        return c + 1;
    };
    auto k2 = [&](int it) {   // x, r updates, ||r||^2, W^T r; then Steps 7-9
        int c = 0;
        for (Slab& q : P.sl) {
            ProjArgs a{};
            a.g = q.g; a.Bp = Bp; a.npad = npad; a.nct = P.totP; a.ngroups = (q.g.N + 3) / 4; a.ldw = ctx->ldw;
            a.W = q.W; a.theta = L.theta; a.active = L.active; a.alpha = L.alpha;
            a.P = (it & 1) ? q.P0 : q.P1; a.X = q.X; a.R = q.R; a.V = nullptr; a.vconst = ctx->fconst;
            a.part = L.partP; a.done = done; a.col0 = q.colP;
            const int ch = wtr_smem_bytes(Bp, ctx->ldw, 64) <= (size_t)110 * 1024 ? 64 : 32;
            const size_t wsm = wtr_smem_bytes(Bp, ctx->ldw, ch);
            if (Bp <= 32 && !q.g.faces && wsm <= (size_t)110 * 1024 && npad > 0 && npad <= 64) {
                // the unpartitioned path's pair (§7): x, r updated in row segments on the
                // stored planes (ghost values are refreshed by the r halo), then W^T r and
                // ||r||^2 streamed over the OWNED planes only
                const int lgBs = ilog2(Bp);
                k_xr3r<4, false><<<q.nctf, kFlat, fsm, st>>>(a, lgBs);
                ProjArgs b2 = a;
                const int64_t off = (int64_t)(q.z0 - q.g0) * plane;
                b2.V = q.R + off * Bp;
                b2.W = q.W + off * ctx->ldw;
                b2.g.N = (int64_t)(q.z1 - q.z0) * plane;
                if (ch == 64) {
                    if (Bp == 8) k_wtr<8, 64><<<q.nct, kMT, wsm, st>>>(b2);
                    else if (Bp == 16) k_wtr<16, 64><<<q.nct, kMT, wsm, st>>>(b2);
                    else k_wtr<32, 64><<<q.nct, kMT, wsm, st>>>(b2);
                } else {
                    if (Bp == 8) k_wtr<8, 32><<<q.nct, kMT, wsm, st>>>(b2);
                    else if (Bp == 16) k_wtr<16, 32><<<q.nct, kMT, wsm, st>>>(b2);
                    else k_wtr<32, 32><<<q.nct, kMT, wsm, st>>>(b2);
                }
                ++c;
            } else {
                launch_proj<MODE_CG>(q.g, q.nct, psm, st, a);
            }
            ++c;
        }
        if (dist) {   // rank sum, allreduce of [W^T r, ||r||^2], Steps 7-9
            SolveState S1 = S;
            S1.partP = P.colP;
            S1.nct = 1;
            k_reduce_rows<<<Bp, 128, 0, st>>>(L.partP, npad + 1, P.totP, P.colP);
            nck(ncclAllReduce(P.colP, P.colP, (size_t)Bp * (npad + 1), ncclDouble, ncclSum, ctx->comm, st),
                "ncclAllReduce(W^T r, ||r||^2)");
            k_reduce_solve<<<Bp, kRsThreads, 0, st>>>(S1);
            return c + 2;
        }
        k_reduce_solve<<<Bp, kRsThreads, 0, st>>>(S);
        return c + 1;
    };
    // halo copies: ghost planes of slab s from the owners' stored planes
    auto halo = [&](int which, int depth) {
        int c = 0;
        if (dist) {   // grouped send/recv of whole planes with the neighbouring ranks
            Slab& q = P.sl[0];
            double* v = which == 0 ? q.R : which == 1 ? q.Y : q.X;
            const size_t pe = (size_t)plane * Bp;          // doubles per plane
            nck(ncclGroupStart(), "ncclGroupStart");
            if (ctx->rank > 0) {
                const int d = std::min(depth, q.z0 - q.g0);
                nck(ncclSend(v + (size_t)(q.z0 - q.g0) * pe, d * pe, ncclDouble, ctx->rank - 1, ctx->comm, st),
                    "ncclSend(halo, lower)");
                nck(ncclRecv(v + (size_t)(q.z0 - d - q.g0) * pe, d * pe, ncclDouble, ctx->rank - 1, ctx->comm, st),
                    "ncclRecv(halo, lower)");
            }
            if (ctx->rank + 1 < ctx->nranks) {
                const int d = std::min(depth, q.g1 - q.z1);
                nck(ncclSend(v + (size_t)(q.z1 - d - q.g0) * pe, d * pe, ncclDouble, ctx->rank + 1, ctx->comm, st),
                    "ncclSend(halo, upper)");
                nck(ncclRecv(v + (size_t)(q.z1 - q.g0) * pe, d * pe, ncclDouble, ctx->rank + 1, ctx->comm, st),
                    "ncclRecv(halo, upper)");
            }
            nck(ncclGroupEnd(), "ncclGroupEnd");
            return 0;
        }
        for (int s = 0; s < G; ++s) {
            Slab& q = P.sl[s];
            double* dst = which == 0 ? q.R : which == 1 ? q.Y : q.X;
            const size_t pb = (size_t)plane * Bp * 8;
            if (s > 0) {               // planes [max(g0, z0 - depth), z0) from slab s-1
                const Slab& o2 = P.sl[s - 1];
                const double* src = which == 0 ? o2.R : which == 1 ? o2.Y : o2.X;
                const int a0 = std::max(q.g0, q.z0 - depth), a1 = q.z0;
                if (a1 > a0) {
                    cudaMemcpyAsync((char*)dst + (size_t)(a0 - q.g0) * pb, (const char*)src + (size_t)(a0 - o2.g0) * pb,
                                    (size_t)(a1 - a0) * pb, cudaMemcpyDeviceToDevice, st);
                    ++c;
                }
            }
            if (s + 1 < G) {           // planes [z1, min(g1, z1 + depth)) from slab s+1
                const Slab& o2 = P.sl[s + 1];
                const double* src = which == 0 ? o2.R : which == 1 ? o2.Y : o2.X;
                const int a0 = q.z1, a1 = std::min(q.g1, q.z1 + depth);
                if (a1 > a0) {
                    cudaMemcpyAsync((char*)dst + (size_t)(a0 - q.g0) * pb, (const char*)src + (size_t)(a0 - o2.g0) * pb,
                                    (size_t)(a1 - a0) * pb, cudaMemcpyDeviceToDevice, st);
                    ++c;
                }
            }
        }
        return 0 * c;
    };
    auto k3 = [&](int init) {   // y0 = W e, half-sweeps on the stored planes; then Step 10
        int c = 0;
        for (Slab& q : P.sl) {
            if (npad > 0) {
                ProlongArgs a{};
                a.N = q.g.N; a.Bp = Bp; a.npad = npad; a.ldw = ctx->ldw; a.W = q.W; a.E = L.E;
                a.active = L.active; a.Y = q.Y; a.accumulate = 0; a.done = done;
                a.skip_color = seq.empty() ? -1 : seq[0];   // overwritten unread by the first half-sweep
                a.dim = 3; a.m = q.g.m; a.kofs = q.g.kofs; a.fm = q.g.fm;
                const int pgrid = grid_for(((q.g.N + 7) / 8) * (Bp / 8), 8, ctx->num_sms * 16);
                k_prolong<<<pgrid, kThreads, 0, st>>>(a);
            } else {
                k_fill_batch<<<grid_for(q.N8 * Bp, 256, ctx->num_sms * 8), 256, 0, st>>>(q.Y, q.g.N, q.N8, Bp, 0,
                                                                                         nullptr, 0.0);
            }
            ++c;
            GSArgs a{};
            a.g = q.g; a.Bp = Bp; a.lgB = lgB; a.NB = q.g.N * Bp; a.theta = L.theta; a.active = L.active;
            a.Y = q.Y; a.Rhs = q.R; a.rconst = 0.0; a.init = init; a.s = S; a.done = done;
            a.col0 = q.colF; a.ext = 1;
            std::vector<int> cs = seq;
            if (cs.empty()) cs.push_back(-1);
            for (size_t t = 0; t < cs.size(); ++t) {
                a.color = cs[t];
                const bool l = t + 1 == cs.size();
                if (Bp <= 32 && a.color >= 0 && !q.g.faces) {     // row segments (kernels.cuh)
                    if (l) k_gs3r<true, 4, false><<<q.nctf, kFlat, fsm, st>>>(a);
                    else k_gs3r<false, 4, false><<<q.nctf, kFlat, fsm, st>>>(a);
                } else if (l) k_gs<3, true><<<q.nctf, kFlat, fsm, st>>>(a);
                else k_gs<3, false><<<q.nctf, kFlat, fsm, st>>>(a);
                ++c;
            }
        }
        if (dist) {   // rank sum, allreduce of [y^T r, y^T y], Step 10
            SolveState S1 = S;
            S1.partF = P.colF;
            S1.nctf = 1;
            k_reduce_rows<<<Bp, 128, 0, st>>>(L.partF, 2, P.totF, P.colF);
            nck(ncclAllReduce(P.colF, P.colF, (size_t)Bp * 2, ncclDouble, ncclSum, ctx->comm, st),
                "ncclAllReduce(y^T r, y^T y)");
            k_slab_beta<<<1, 512, 0, st>>>(S1, 1, init);
            return c + 2;
        }
        k_slab_beta<<<1, 512, 0, st>>>(S, P.totF, init);
        return c + 1;
    };

    // ---- RBCG Steps 2-3: y_0 = RBI(A, r_0, W, 1), rho_0 -------------------------
    launches += k3(1);
    halo(1, 1);
    CKL();
    if (nres != ncclSuccess) return nfail();
    int per_iter = 0;
    auto body = [&](int it) {
        int c = k1(it);
        c += k2(it);
        halo(0, P.H);
        c += k3(0);
        halo(1, 1);
        return c;
    };
    const int chunk = o->graph_chunk;
    char keybuf[512];
    snprintf(keybuf, sizeof keybuf, "slab|%d|%d|%p|%d|%d|%d|%d|%d|%d|%.17g|%.17g|%d|%p|%p|%p|%d|%d|%.17g|%d|%.17g"
             "|%d|%p|%p|%p|%p",
             G, (int)dist, workspace_dev, B, Bp, o->smoother, o->sweeps, o->max_iter, chunk, o->tol, o->delta,
             o->record_history, (void*)ctx->Wi, (void*)st, (void*)L.hist, n, npad, ctx->fconst, o->n_active,
             o->gamma, o->x_location, (void*)L.theta, (void*)L.partP, (void*)L.ints, (void*)P.colP);
    const std::string key(keybuf);
    if (!ctx->gexec || ctx->gkey != key) {
        if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; }
        cudaStream_t cap;
        CK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
        cudaGraph_t graph;
        CK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
        cudaStream_t keep = st;
        st = cap;
        for (int it = 0; it < chunk; ++it) per_iter += body(it);
        st = keep;
        const cudaError_t ce = cudaStreamEndCapture(cap, &graph);
        if (nres != ncclSuccess || ce != cudaSuccess) {   // end the capture cleanly before returning
            if (ce == cudaSuccess) cudaGraphDestroy(graph);
            cudaStreamDestroy(cap);
            if (nres != ncclSuccess) return nfail();
            return fail(ctx, RBS_E_CUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(ce));
        }
        CK(cudaGraphInstantiate(&ctx->gexec, graph, 0));
        cudaGraphDestroy(graph);
        cudaStreamDestroy(cap);
        ctx->gkey = key;
        ctx->g_per_chunk = per_iter;
    } else {
        per_iter = ctx->g_per_chunk;
    }
    const int64_t max_launch = (int64_t)o->max_iter / chunk + 3;
    volatile int* hf = ctx->h_flag;
    hf[0] = hf[1] = 0;
    for (int64_t l = 0;; ++l) {
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

    // ---- outputs ----------------------------------------------------------------
    std::vector<int> hs(Bp), hi(Bp), hp(Bp);
    std::vector<double> hrel(Bp), hfn(Bp), tr(Bp, NAN);
    CK(cudaMemcpyAsync(hs.data(), L.status, Bp * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hi.data(), L.its, Bp * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hp.data(), L.pivot, Bp * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hrel.data(), L.relres, Bp * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hfn.data(), L.fnorm, Bp * 8, cudaMemcpyDeviceToHost, st));
    ctx->last_na.assign(Bp, n);
    CK(cudaMemcpyAsync(ctx->last_na.data(), L.na, Bp * 4, cudaMemcpyDeviceToHost, st));
    // true residual ||f - A x|| / ||f||: x halos, then per-slab residual partials
    halo(2, 1);
    for (Slab& q : P.sl) {
        ProjArgs a{};
        a.g = q.g; a.Bp = Bp; a.npad = npad; a.nct = P.totP; a.ngroups = (q.g.N + 3) / 4; a.ldw = ctx->ldw;
        a.W = q.W; a.theta = L.theta; a.active = nullptr; a.alpha = L.alpha; a.X = q.X; a.V = nullptr;
        a.vconst = ctx->fconst; a.part = L.partP; a.done = nullptr; a.col0 = q.colP;
        launch_proj<MODE_RESID>(q.g, q.nct, psm, st, a);
        ++launches;
    }
    k_reduce_rows<<<Bp, 128, 0, st>>>(L.partP, npad + 1, P.totP, L.fproj);
    ++launches;
    if (dist)
        nck(ncclAllReduce(L.fproj, L.fproj, (size_t)Bp * (npad + 1), ncclDouble, ncclSum, ctx->comm, st),
            "ncclAllReduce(true residual)");
    CKL();
    if (nres != ncclSuccess) return nfail();
    {
        std::vector<double> rows((size_t)Bp * (npad + 1));
        CK(cudaMemcpyAsync(rows.data(), L.fproj, rows.size() * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int b = 0; b < Bp; ++b) tr[b] = std::sqrt(rows[(size_t)b * (npad + 1) + npad]) / hfn[b];
    }
    // X: [B][N] (virtual), [B][owned nodes of this rank] (ranks)
    double* xdst = o->x_location == RBS_MEM_HOST ? L.Xout : X;
    const int64_t ldx = dist ? (int64_t)(P.sl[0].z1 - P.sl[0].z0) * plane : g.N;
    for (Slab& q : P.sl) {
        const int64_t nown = (int64_t)(q.z1 - q.z0) * plane;
        k_transpose_out<<<(unsigned)((nown + 31) / 32), 256, 0, st>>>(
            q.X + (size_t)(q.z0 - q.g0) * plane * Bp, nown, Bp, B, xdst + (dist ? 0 : (size_t)(q.z0 - 1) * plane),
            ldx);
        ++launches;
    }
    CKL();
    if (o->x_location == RBS_MEM_HOST)
        CK(cudaMemcpyAsync(X, L.Xout, (size_t)B * ldx * 8, cudaMemcpyDeviceToHost, st));
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

}  // namespace
