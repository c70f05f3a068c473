// greedy.inc.cu -- offline greedy basis construction on the GPU (included by api.cu).
//
// PAPER.md:77-91 (algorithm0) and PAPER.md:294-308 (algorithm3, adaptive:
// snapshot by RBCG with W_{N-1}); DESIGN.md AMB-13:
//   mu_1 = Xi_train[0]; snapshot to relative tolerance snapshot_tol;
//   W_N = MGS(W_{N-1}, x) with one re-orthogonalisation pass, reject if
//   ||w|| < drop_tol ||x|| (then the next-best mu is tried);
//   A_{N,q} extended by one row/column (i <= N, mirrored), f_N by one entry;
//   Step 5: A_N(mu) a = f_N for every training mu (one CTA per mu, reusing
//   k_setup_reduced); Step 6: argmax of sum_n |a_n| over unused mu, lowest
//   index on ties.
// Every N-dependent step runs in the library's kernels; the host only
// sequences the steps and does the argmax over n_train scalars.

namespace rbs {

__global__ void __launch_bounds__(256) k_dot(const double* __restrict__ a, int64_t sa,
                                             const double* __restrict__ b, int64_t sb, int64_t N,
                                             double* __restrict__ part) {
    __shared__ double s[256];
    const int64_t i0 = (N * blockIdx.x) / gridDim.x, i1 = (N * (blockIdx.x + 1)) / gridDim.x;
    double acc = 0.0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += 256) acc = fma(a[i * sa], b[i * sb], acc);
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

__global__ void k_sum_to(const double* __restrict__ part, int cnt, double* __restrict__ out) {
    const double v = warp_sum_row(part, cnt, threadIdx.x & 31);
    if (threadIdx.x == 0) *out = v;
}

// w -= c * W_j  (c on the device)
__global__ void k_mgs_axpy(double* __restrict__ w, const double* __restrict__ Wj, int64_t sW,
                           const double* __restrict__ c, int64_t N) {
    const double cc = *c;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x)
        w[i] = fma(-cc, Wj[i * sW], w[i]);
}

__global__ void k_store_col(const double* __restrict__ w, double wn, double* __restrict__ Wi,
                            int npad, int j, int64_t N) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x)
        Wi[i * npad + j] = w[i] / wn;
}

}  // namespace rbs

namespace {

constexpr int kDotCtas = 296;
constexpr int kSnapBatch = 8;   // fine snapshots solved together (RBS_GREEDY_SAMPLES_BATCH)

struct GreedyLayout {
    double *Wi, *ANq, *Z, *part, *rows, *x, *w, *dpart, *scal, *phi, *xb;
    double *tr_theta, *tr_fproj, *tr_L, *tr_E, *tr_a;
    double *tr_d[6];
    int* tr_i[5];
    void* solve_ws;
    size_t solve_bytes;
    size_t bytes;
};

GreedyLayout greedy_layout(rbs_ctx* c, int nt, int n_max, void* base) {
    const int npad = (int)round_up(n_max, 8);
    Carve cv(base);
    GreedyLayout L{};
    L.Wi = cv.take<double>((size_t)c->N8 * w_ld(npad));
    L.ANq = cv.take<double>((size_t)c->g.Q * npad * npad + 8);
    L.Z = cv.take<double>((size_t)c->N8 * 8);
    L.part = cv.take<double>((size_t)8 * (npad + 1) * proj_ctas(c->g));
    L.rows = cv.take<double>((size_t)8 * (npad + 1));
    L.x = cv.take<double>((size_t)c->N8);
    L.w = cv.take<double>((size_t)c->N8);
    L.xb = cv.take<double>((size_t)kSnapBatch * c->g.N);   // batched fine snapshots (samples mode)
    L.dpart = cv.take<double>(kDotCtas);
    L.scal = cv.take<double>(8);
    L.phi = cv.take<double>(RBS_MAX_R);
    L.tr_theta = cv.take<double>((size_t)c->g.Q * nt);
    L.tr_fproj = cv.take<double>((size_t)nt * (npad + 1));
    L.tr_L = cv.take<double>((size_t)nt * npad * npad + 8);
    L.tr_E = cv.take<double>((size_t)npad * nt + 8);
    L.tr_a = cv.take<double>((size_t)nt * npad + 8);
    for (auto& p : L.tr_d) p = cv.take<double>(nt);
    for (auto& p : L.tr_i) p = cv.take<int>(nt + 8);
    // solve workspace for B = 1 RBCG snapshots with the full padded width
    rbs_ctx tmp = *c;
    tmp.npad = npad;
    tmp.ldw = w_ld(npad);
    rbs_solve_opts o;
    rbs_default_opts(&o);
    L.solve_bytes = solve_layout(&tmp, kSnapBatch, &o, true, nullptr).bytes;   // rhs buffer: affine snapshots
    L.solve_ws = cv.take<char>(L.solve_bytes);
    L.bytes = cv.off + 256;
    return L;
}

}  // namespace

extern "C" {

rbs_status rbs_greedy_workspace_size(const rbs_ctx* c, int n_train, int n_max, size_t* bytes) {
    rbs_ctx* ctx = const_cast<rbs_ctx*>(c);
    if (!ctx || !bytes) return RBS_E_ARG;
    if (!ctx->has_op) return fail(ctx, RBS_E_STATE, "set the operator first");
    if (n_train < 1 || n_max < 1 || n_max > RBS_MAX_N) return fail(ctx, RBS_E_DIM, "bad n_train/n_max");
    *bytes = greedy_layout(ctx, n_train, n_max, nullptr).bytes;
    return RBS_OK;
}

// Greedy core.  R = 0: the constant right-hand side (rbs_set_rhs_constant);
// R > 0: affine right-hand sides f(mu_t) = sum_r phi_train[t][r] f_r (terms_dev
// [R][N]): snapshots solve with that f, the offline vectors are f_{N,r} = W^T f_r
// (fn_out [R][n]) and the indicator solves use f_N(mu_t) = sum_r phi_r(mu_t) f_{N,r}.
static rbs_status greedy_core(rbs_ctx* ctx, int n_train, const double* mu_train, int R,
                              const double* phi_train, const double* terms, int n_max, int mode,
                              double snapshot_tol, double drop_tol, double* W_out,
                              double* ANq_out, double* fn_out, int* n_out, int* selected,
                              double* indicator, int* snap_iters, int* n_rejected,
                              void* workspace, size_t ws_bytes, void* stream) {
    if (!ctx) return RBS_E_ARG;
    ctx->err.clear();
    if (!ctx->has_op) return fail(ctx, RBS_E_STATE, "set the operator first");
    if (n_train < 1 || n_max < 1 || n_max > RBS_MAX_N) return fail(ctx, RBS_E_DIM, "bad n_train/n_max");
    if (!mu_train || !W_out || !n_out || !workspace) return fail(ctx, RBS_E_ARG, "NULL argument");
    if (mode != RBS_GREEDY_PLAIN && mode != RBS_GREEDY_ADAPTIVE && mode != RBS_GREEDY_SAMPLES &&
        mode != RBS_GREEDY_SAMPLES_BATCH)
        return fail(ctx, RBS_E_ARG, "bad mode");
    // multi-fidelity fine half: the given samples in list order, no selection;
    // SAMPLES_BATCH solves them kSnapBatch at a time ("solving the PDE N times on a fine
    // grid"), each batch by RBCG preconditioned with the symmetric two-level RBI on the basis
    // built so far (AMB-27)
    const bool batched = mode == RBS_GREEDY_SAMPLES_BATCH;
    const bool from_list = mode == RBS_GREEDY_SAMPLES || batched;
    if (batched && R > 0) return fail(ctx, RBS_E_UNSUPPORTED, "batched samples: constant right-hand side only");
    // the greedy works in theta space with its own right-hand side: the context's affine
    // rhs terms and parameter map are dropped (set them again before loading a basis)
    ctx->R = 0;
    ctx->fr.clear();
    ctx->T = nullptr;
    ctx->P = 0;
    ctx->Ta.clear();
    ctx->Pa.clear();
    GreedyLayout L = greedy_layout(ctx, n_train, n_max, workspace);
    if (ws_bytes < L.bytes) return fail(ctx, RBS_E_NOMEM, "workspace too small");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    const Geo& g = ctx->g;
    const int Q = g.Q, P = Q, npad = (int)round_up(n_max, 8), nt = n_train, ldw = w_ld(npad);
    const int nct = proj_ctas(g);
    const int vgrid = grid_for(g.N, 256, ctx->num_sms * 8);

    CK(cudaMemsetAsync(L.Wi, 0, (size_t)ctx->N8 * ldw * 8, st));
    CK(cudaMemsetAsync(L.ANq, 0, ((size_t)Q * npad * npad + 8) * 8, st));
    CK(cudaMemsetAsync(L.x, 0, (size_t)ctx->N8 * 8, st));
    CK(cudaMemsetAsync(L.w, 0, (size_t)ctx->N8 * 8, st));
    // the context's basis becomes the growing W (zero columns beyond n)
    if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; ctx->gkey.clear(); }
    ctx->Wi = L.Wi;
    ctx->dANq = L.ANq;
    ctx->npad = npad;
    ctx->ldw = ldw;
    ctx->n = 0;
    ctx->hANq.assign(0, 0.0);
    ctx->hfn.assign(0, 0.0);
    ctx->has_basis = true;

    const int RT = R > 0 ? R : 1;           // right-hand-side terms tracked
    std::vector<double> hA((size_t)Q * npad * npad, 0.0), hf((size_t)RT * npad, 0.0);
    // training parameters theta [Q][nt]
    {
        std::vector<double> th((size_t)Q * nt);
        for (int t = 0; t < nt; ++t)
            for (int q = 0; q < Q; ++q) th[(size_t)q * nt + t] = mu_train[(size_t)t * P + q];
        CK(cudaMemcpyAsync(L.tr_theta, th.data(), th.size() * 8, cudaMemcpyHostToDevice, st));
    }
    std::vector<char> excluded(nt, 0);
    std::vector<double> ind(nt), a_host((size_t)nt * npad);
    rbs_solve_opts so;
    rbs_default_opts(&so);
    so.tol = snapshot_tol;
    so.max_iter = 200000;
    int n = 0, rej = 0, cand = 0, its_first = -1, chunk0 = -1;
    int b_its[kSnapBatch] = {0}, b_qs[kSnapBatch] = {0};
    auto dot = [&](const double* a, int64_t sa, const double* b, int64_t sb, double* out) {
        k_dot<<<kDotCtas, 256, 0, st>>>(a, sa, b, sb, g.N, L.dpart);
        k_sum_to<<<1, 32, 0, st>>>(L.dpart, kDotCtas, out);
    };
    while (n < n_max && cand >= 0) {
        // ---- Step 3: snapshot x(mu_N) = RBCG(A, f, W_{N-1}) -------------------
        ctx->n = mode != RBS_GREEDY_PLAIN ? n : 0;
        ctx->hfn.assign(hf.begin(), hf.begin() + ctx->n);
        ctx->hANq.assign((size_t)Q * ctx->n * ctx->n, 0.0);
        for (int q = 0; q < Q; ++q)
            for (int i = 0; i < ctx->n; ++i)
                for (int j = 0; j < ctx->n; ++j)
                    ctx->hANq[((size_t)q * ctx->n + i) * ctx->n + j] = hA[((size_t)q * npad + i) * npad + j];
        // N = 1 (or plain greedy): SGS-PCG, the standard solver of PAPER.md:291.
        // N >= 2 (adaptive): RBCG with W_{N-1}, guarded (AMB-22): not converged
        // within 2*its_1 + 50 -> fall back to SGS-PCG; its < 0.
        int its = 0, qs = 0;
        const double* xsrc = L.x;
        if (batched) {
            if (chunk0 < 0 || cand >= chunk0 + kSnapBatch) {   // the next batch of samples
                chunk0 = cand;
                const int cb = std::min(kSnapBatch, nt - cand);
                rbs_solve_opts sb = so;
                sb.max_iter = 200000;
                sb.precond = RBS_PRECOND_SYM;
                rbs_status s = rbs_solve_batch(ctx, cb, mu_train + (size_t)cand * P, &sb, nullptr, L.xb,
                                               b_its, b_qs, nullptr, nullptr, nullptr, nullptr, L.solve_ws,
                                               L.solve_bytes, stream);
                if (s != RBS_OK) return s;
            }
            its = b_its[cand - chunk0];
            qs = b_qs[cand - chunk0];
            xsrc = L.xb + (size_t)(cand - chunk0) * g.N;
            if (qs != Q_CONVERGED) {   // fallback: this snapshot alone by SGS-PCG (its reported < 0)
                ctx->n = 0;
                ctx->hfn.clear();
                ctx->hANq.clear();
                rbs_solve_opts s1 = so;
                s1.max_iter = 200000;
                rbs_status s = rbs_solve_batch(ctx, 1, mu_train + (size_t)cand * P, &s1, nullptr, L.x, &its, &qs,
                                               nullptr, nullptr, nullptr, nullptr, L.solve_ws, L.solve_bytes, stream);
                if (s != RBS_OK) return s;
                its = -its;
                xsrc = L.x;
            }
        } else {
            so.max_iter = (ctx->n == 0) ? 200000 : 2 * (its_first > 0 ? its_first : 1000) + 50;
            const double* srhs = nullptr;
            if (R > 0) {   // f(mu_cand) = sum_r phi_r f_r -> L.Z
                CK(cudaMemcpyAsync(L.phi, phi_train + (size_t)cand * R, (size_t)R * 8, cudaMemcpyHostToDevice, st));
                k_affine_rhs<<<grid_for(g.N, 256, ctx->num_sms * 8), 256, 0, st>>>(L.phi, R, terms, g.N, 1, L.Z);
                CKL();
                srhs = L.Z;
            }
            rbs_status s = rbs_solve_batch(ctx, 1, mu_train + (size_t)cand * P, &so, srhs, L.x, &its,
                                           &qs, nullptr, nullptr, nullptr, nullptr, L.solve_ws,
                                           L.solve_bytes, stream);
            if (s != RBS_OK) return s;
            if (ctx->n == 0 && its_first < 0) its_first = its;
            if (qs != Q_CONVERGED && ctx->n > 0) {
                ctx->n = 0;
                ctx->hfn.clear();
                ctx->hANq.clear();
                so.max_iter = 200000;
                s = rbs_solve_batch(ctx, 1, mu_train + (size_t)cand * P, &so, srhs, L.x, &its, &qs,
                                    nullptr, nullptr, nullptr, nullptr, L.solve_ws, L.solve_bytes, stream);
                if (s != RBS_OK) return s;
                its = -its;
            }
            // ---- Step 4: W_N = MGS(W_{N-1}, x) ------------------------------------
        }
        CK(cudaMemcpyAsync(L.w, xsrc, (size_t)g.N * 8, cudaMemcpyDeviceToDevice, st));
        dot(L.w, 1, L.w, 1, L.scal + 0);            // ||x|| (w = x before the MGS passes)
        for (int pass = 0; pass < 2; ++pass)
            for (int j = 0; j < n; ++j) {
                dot(L.Wi + j, ldw, L.w, 1, L.scal + 2);
                k_mgs_axpy<<<vgrid, 256, 0, st>>>(L.w, L.Wi + j, ldw, L.scal + 2, g.N);
            }
        dot(L.w, 1, L.w, 1, L.scal + 1);
        CKL();
        double nrm[2];
        CK(cudaMemcpyAsync(nrm, L.scal, 2 * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const double vnorm = std::sqrt(nrm[0]), wn = std::sqrt(nrm[1]);
        excluded[cand] = 1;
        const bool rejected = !(vnorm > 0.0) || !(wn >= drop_tol * vnorm);
        if (rejected) {
            ++rej;
        } else {
            k_store_col<<<vgrid, 256, 0, st>>>(L.w, wn, L.Wi, ldw, n, g.N);
            CKL();
            // ---- offline column n: (A_{N,q})_{i n} = w_i^T A_q w_n, i <= n --------
            const int j0 = (n / 8) * 8, jj = n - j0;
            for (int q = 0; q < Q; ++q) {
                const int grid = grid_for(g.N * 8, kThreads, ctx->num_sms * 8);
                if (g.dim == 2) k_apply_Aq<2><<<grid, kThreads, 0, st>>>(g, q, L.Wi, ldw, j0, L.Z);
                else k_apply_Aq<3><<<grid, kThreads, 0, st>>>(g, q, L.Wi, ldw, j0, L.Z);
                ProjArgs a{};
                a.g = g; a.Bp = 8; a.npad = npad; a.nct = nct; a.ngroups = (g.N + 3) / 4; a.ldw = ldw;
                a.W = L.Wi; a.V = L.Z; a.part = L.part;
                launch_proj<MODE_PLAIN>(g, nct, proj_smem(g, 8, npad), st, a);
                k_reduce_rows<<<8, 128, 0, st>>>(L.part, npad + 1, nct, L.rows);
                CKL();
                std::vector<double> rows((size_t)8 * (npad + 1));
                CK(cudaMemcpyAsync(rows.data(), L.rows, rows.size() * 8, cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                for (int i = 0; i <= n; ++i) {
                    const double v = rows[(size_t)jj * (npad + 1) + i];
                    hA[((size_t)q * npad + i) * npad + n] = v;
                    hA[((size_t)q * npad + n) * npad + i] = v;
                }
            }
            for (int r = 0; r < RT; ++r) {   // f_{N,r}[n] = w_n^T f_r  (f_1 = 1 for R = 0)
                ProjArgs a{};
                a.g = g; a.Bp = 8; a.npad = npad; a.nct = nct; a.ngroups = (g.N + 3) / 4; a.ldw = ldw;
                a.W = L.Wi; a.part = L.part;
                if (R > 0) {
                    // the projection pass reads [N][8] node-major batches: f_r goes to column 0
                    k_fill_batch<<<grid_for(g.N, 256, ctx->num_sms * 8), 256, 0, st>>>(
                        L.Z, g.N, ctx->N8, 8, 1, terms + (size_t)r * g.N, 0.0);
                    a.V = L.Z;
                } else {
                    a.V = nullptr;
                    a.vconst = 1.0;
                }
                launch_proj<MODE_PLAIN>(g, nct, proj_smem(g, 8, npad), st, a);
                k_reduce_rows<<<1, 128, 0, st>>>(L.part, npad + 1, nct, L.rows);
                CKL();
                double v;
                CK(cudaMemcpyAsync(&v, L.rows + n, 8, cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                hf[(size_t)r * npad + n] = v;
            }
            if (selected) selected[n] = cand;
            if (snap_iters) snap_iters[n] = its;
            ++n;
            CK(cudaMemcpyAsync(L.ANq, hA.data(), hA.size() * 8, cudaMemcpyHostToDevice, st));
        }
        if (from_list) {             // next sample in list order; no indicator solves
            cand = cand + 1 < nt ? cand + 1 : -1;
            continue;
        }
        if (n == 0) {
            cand = -1;
            for (int t = 0; t < nt; ++t)
                if (!excluded[t]) { cand = t; break; }
            continue;
        }
        // ---- Step 5: A_N(mu) a = f_N for all training mu (one CTA each) -------
        {
            std::vector<double> fp((size_t)nt * (npad + 1), 0.0);
            for (int t = 0; t < nt; ++t) {
                for (int j = 0; j < n; ++j) {
                    double v = 0.0;
                    if (R > 0)
                        for (int r = 0; r < R; ++r) v += phi_train[(size_t)t * R + r] * hf[(size_t)r * npad + j];
                    else
                        v = hf[j];
                    fp[(size_t)t * (npad + 1) + j] = v;
                }
                fp[(size_t)t * (npad + 1) + npad] = 1.0;
            }
            CK(cudaMemcpyAsync(L.tr_fproj, fp.data(), fp.size() * 8, cudaMemcpyHostToDevice, st));
            SolveState S{};
            S.B = nt; S.Bp = nt; S.n = n; S.npad = npad; S.maxit = 1; S.method = 1; S.tol = 0.0;
            S.ANq = L.ANq; S.Q = Q; S.theta = L.tr_theta; S.fproj = L.tr_fproj; S.L = L.tr_L;
            S.E = L.tr_E; S.a_n = L.tr_a; S.alpha = L.tr_d[0]; S.beta = L.tr_d[1]; S.rho = L.tr_d[2];
            S.rr = L.tr_d[3]; S.fnorm = L.tr_d[4]; S.relres = L.tr_d[5]; S.active = L.tr_i[0];
            S.status = L.tr_i[1]; S.its = L.tr_i[2]; S.pivot = L.tr_i[3]; S.hist = nullptr;
            k_setup_reduced<<<nt, 128, 0, st>>>(S, 0);
            CKL();
            std::vector<int> piv(nt);
            CK(cudaMemcpyAsync(a_host.data(), L.tr_a, a_host.size() * 8, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(piv.data(), L.tr_i[3], nt * 4, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            // ---- Step 6: argmax_mu sum_n |a_n(mu)| over unused mu --------------
            cand = -1;
            double best = -INFINITY;
            for (int t = 0; t < nt; ++t) {
                double sabs = 0.0;
                for (int j = 0; j < n; ++j) sabs += std::fabs(a_host[(size_t)t * npad + j]);
                ind[t] = piv[t] >= 0 ? -INFINITY : sabs;
                if (!excluded[t] && ind[t] > best) { best = ind[t]; cand = t; }
            }
            if (indicator) indicator[n - 1] = best;
        }
    }
    // ---- outputs -------------------------------------------------------------
    *n_out = n;
    if (n_rejected) *n_rejected = rej;
    if (n > 0) {
        k_unpack_W<<<grid_for(g.N * n, 256, ctx->num_sms * 8), 256, 0, st>>>(L.Wi, g.N, n, ldw, W_out);
        CKL();
    }
    if (ANq_out)
        for (int q = 0; q < Q; ++q)
            for (int i = 0; i < n_max; ++i)
                for (int j = 0; j < n_max; ++j)
                    ANq_out[((size_t)q * n_max + i) * n_max + j] =
                        (i < n && j < n) ? hA[((size_t)q * npad + i) * npad + j] : 0.0;
    if (fn_out)
        for (int r = 0; r < RT; ++r)
            for (int j = 0; j < n_max; ++j) fn_out[(size_t)r * n_max + j] = j < n ? hf[(size_t)r * npad + j] : 0.0;
    // the context keeps the built basis (workspace retained)
    ctx->n = n;
    ctx->hfn.assign(hf.begin(), hf.begin() + n);
    ctx->hANq.assign((size_t)Q * n * n, 0.0);
    for (int q = 0; q < Q; ++q)
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                ctx->hANq[((size_t)q * n + i) * n + j] = hA[((size_t)q * npad + i) * npad + j];
    if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; ctx->gkey.clear(); }
    CK(cudaStreamSynchronize(st));
    return RBS_OK;
}

rbs_status rbs_build_greedy(rbs_ctx* ctx, int n_train, const double* mu_train, int n_max, int mode,
                            double snapshot_tol, double drop_tol, double* W_out,
                            double* ANq_out, double* fn_out, int* n_out, int* selected,
                            double* indicator, int* snap_iters, int* n_rejected,
                            void* workspace, size_t ws_bytes, void* stream) {
    return greedy_core(ctx, n_train, mu_train, 0, nullptr, nullptr, n_max, mode, snapshot_tol, drop_tol,
                       W_out, ANq_out, fn_out, n_out, selected, indicator, snap_iters, n_rejected, workspace,
                       ws_bytes, stream);
}

rbs_status rbs_build_greedy_affine(rbs_ctx* ctx, int n_train, const double* mu_train, int R,
                                   const double* phi_train_host, const double* terms_dev, int n_max,
                                   int mode, double snapshot_tol, double drop_tol, double* W_out,
                                   double* ANq_out, double* fnr_out, int* n_out, int* selected,
                                   double* indicator, int* snap_iters, int* n_rejected,
                                   void* workspace, size_t ws_bytes, void* stream) {
    if (!ctx) return RBS_E_ARG;
    if (R < 1 || R > RBS_MAX_R) return fail(ctx, RBS_E_DIM, "R must be in 1..RBS_MAX_R");
    if (!phi_train_host || !terms_dev) return fail(ctx, RBS_E_ARG, "phi_train/terms is NULL");
    return greedy_core(ctx, n_train, mu_train, R, phi_train_host, terms_dev, n_max, mode, snapshot_tol,
                       drop_tol, W_out, ANq_out, fnr_out, n_out, selected, indicator, snap_iters, n_rejected,
                       workspace, ws_bytes, stream);
}

}  // extern "C"
