"""Thin Python binding of librbs.so (include/rbs.h): argument marshalling only.

Every step of the RB online solve runs in the library's sm_100a kernels.
PyTorch is used for device memory and streams.  There is no CPU fallback: if
librbs.so is missing or cannot be loaded, importing the binding raises.

Functions carry the C names (rbs_create, rbs_set_operator_blocks,
rbs_load_basis, rbs_solve_batch, rbs_build_greedy, ...); `Solver` is a small
convenience wrapper that owns the torch buffers a context needs.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "librbs.so")

RBS_RBI, RBS_RBCG = 0, 1
RBS_SMOOTH_SYM_RBGS, RBS_SMOOTH_FWD_RBGS, RBS_SMOOTH_JACOBI = 0, 1, 2
RBS_MEM_DEVICE, RBS_MEM_HOST = 0, 1
RBS_GREEDY_PLAIN, RBS_GREEDY_ADAPTIVE, RBS_GREEDY_SAMPLES, RBS_GREEDY_SAMPLES_BATCH = 0, 1, 2, 3
RBS_PRECOND_POST, RBS_PRECOND_SYM = 0, 1
RBS_BETA_FR, RBS_BETA_PR = 0, 1
QSTATUS = {0: "CONVERGED", 1: "MAXIT", 2: "REDUCED_NOT_SPD", 3: "CURVATURE", 4: "PRECOND",
           5: "NONFINITE"}


class RbsError(RuntimeError):
    pass


class rbs_solve_opts(C.Structure):
    _fields_ = [("method", C.c_int), ("tol", C.c_double), ("max_iter", C.c_int),
                ("smoother", C.c_int), ("sweeps", C.c_int), ("delta", C.c_double),
                ("record_history", C.c_int), ("x_location", C.c_int), ("graph_chunk", C.c_int),
                ("profile", C.c_int), ("n_active", C.c_int), ("gamma", C.c_double),
                ("omega", C.c_double), ("precond", C.c_int), ("beta_rule", C.c_int)]


_lib = None

_SIGS = {
    "rbs_version": (C.c_int, []),
    "rbs_status_string": (C.c_char_p, [C.c_int]),
    "rbs_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "rbs_destroy": (None, [C.c_void_p]),
    "rbs_last_error": (C.c_char_p, [C.c_void_p]),
    "rbs_last_launch_count": (C.c_int64, [C.c_void_p]),
    "rbs_last_n_active": (C.c_int, [C.c_void_p, C.c_void_p]),
    "rbs_last_profile": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "rbs_kernel_class_name": (C.c_char_p, [C.c_int]),
    "rbs_set_operator_blocks": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int64),
                                          C.POINTER(C.c_int)]),
    "rbs_set_rhs_constant": (C.c_int, [C.c_void_p, C.c_double]),
    "rbs_set_operator_faces": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_int, C.c_void_p]),
    "rbs_affine_rhs": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p]),
    "rbs_set_rhs_terms": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p]),
    "rbs_set_param_map": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    "rbs_operator_labels_size": (C.c_int, [C.c_int, C.c_int64, C.c_int, C.POINTER(C.c_size_t)]),
    "rbs_set_operator_labels": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_int, C.c_void_p, C.c_void_p,
                                          C.c_size_t, C.c_void_p]),
    "rbs_comm_init": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    "rbs_broadcast_basis": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_size_t, C.c_void_p]),
    "rbs_set_virtual_slabs": (C.c_int, [C.c_void_p, C.c_int]),
    "rbs_nccl_unique_id": (C.c_int, [C.c_void_p, C.c_size_t]),
    "rbs_dist_init": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int]),
    "rbs_local_range": (C.c_int, [C.c_void_p] + [C.POINTER(C.c_int64)] * 6),
    "rbs_basis_storage_size": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_size_t)]),
    "rbs_load_basis": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "rbs_get_offline_blocks": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "rbs_default_opts": (None, [C.POINTER(rbs_solve_opts)]),
    "rbs_solve_workspace_size": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(rbs_solve_opts),
                                           C.POINTER(C.c_size_t)]),
    "rbs_solve_batch": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.POINTER(rbs_solve_opts),
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                  C.c_void_p]),
    "rbs_greedy_workspace_size": (C.c_int, [C.c_void_p, C.c_int, C.c_int,
                                            C.POINTER(C.c_size_t)]),
    "rbs_build_greedy": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int,
                                   C.c_double, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.POINTER(C.c_int), C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.POINTER(C.c_int), C.c_void_p, C.c_size_t, C.c_void_p]),
    "rbs_build_greedy_affine": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                          C.c_int, C.c_int, C.c_double, C.c_double, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.POINTER(C.c_int), C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.POINTER(C.c_int), C.c_void_p,
                                          C.c_size_t, C.c_void_p]),
}
EXPORTED = tuple(_SIGS)


def lib():
    """Load librbs.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise RbsError(f"{_SO} not built; run `python -m paper_1804_06363_b200.build`")
        L = C.CDLL(_SO)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(C.c_void_p)
    return C.c_void_p(a.data_ptr())


def _check(ctx, st, what):
    if st != 0:
        detail = lib().rbs_last_error(ctx).decode() if ctx else ""
        raise RbsError(f"{what}: {lib().rbs_status_string(st).decode()} {detail}")


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


# ---- C-named marshalling functions ------------------------------------------
def rbs_create(device: int = 0):
    h = C.c_void_p()
    _check(None, lib().rbs_create(int(device), C.byref(h)), "rbs_create")
    return h


def rbs_destroy(ctx):
    lib().rbs_destroy(ctx)


def rbs_set_operator_blocks(ctx, dim, m, blocks):
    mm = (C.c_int64 * 3)(*([int(m)] * 3))
    bb = (C.c_int * 3)(*(list(blocks) + [1] * (3 - len(blocks))))
    _check(ctx, lib().rbs_set_operator_blocks(ctx, int(dim), mm, bb), "rbs_set_operator_blocks")


def rbs_set_operator_faces(ctx, dim, m, Q, faces_dev):
    _check(ctx, lib().rbs_set_operator_faces(ctx, int(dim), int(m), int(Q), _ptr(faces_dev)),
           "rbs_set_operator_faces")


def rbs_affine_rhs(ctx, B, R, phi_host, terms_dev, out_dev, stream=None):
    _check(ctx, lib().rbs_affine_rhs(ctx, int(B), int(R), _ptr(phi_host), _ptr(terms_dev), _ptr(out_dev),
                                     _stream(stream)), "rbs_affine_rhs")


def rbs_set_rhs_constant(ctx, value):
    _check(ctx, lib().rbs_set_rhs_constant(ctx, float(value)), "rbs_set_rhs_constant")


def rbs_set_rhs_terms(ctx, terms):
    """terms: list of (N,) cuda float64 tensors (borrowed: keep them alive)."""
    R = len(terms)
    arr = (C.c_void_p * max(R, 1))(*[t.data_ptr() for t in terms])
    _check(ctx, lib().rbs_set_rhs_terms(ctx, R, arr if R else None), "rbs_set_rhs_terms")


def rbs_set_param_map(ctx, P, theta_aff=None, phi_aff=None):
    ta = None if theta_aff is None else np.ascontiguousarray(theta_aff, dtype=np.float64)
    pa = None if phi_aff is None else np.ascontiguousarray(phi_aff, dtype=np.float64)
    _check(ctx, lib().rbs_set_param_map(ctx, int(P), _ptr(ta), _ptr(pa)), "rbs_set_param_map")


def rbs_operator_labels_size(dim, m, Q):
    b = C.c_size_t(0)
    _check(None, lib().rbs_operator_labels_size(int(dim), C.c_int64(m), int(Q), C.byref(b)),
           "rbs_operator_labels_size")
    return b.value


def rbs_set_operator_labels(ctx, dim, m, Q, labels_dev, storage, stream=None):
    _check(ctx, lib().rbs_set_operator_labels(ctx, int(dim), C.c_int64(m), int(Q), _ptr(labels_dev),
                                              _ptr(storage), storage.numel(), _stream(stream)),
           "rbs_set_operator_labels")


def rbs_comm_init(ctx, nccl_id: bytes, nranks, rank):
    buf = C.create_string_buffer(nccl_id, 128)
    _check(ctx, lib().rbs_comm_init(ctx, buf, int(nranks), int(rank)), "rbs_comm_init")


def rbs_broadcast_basis(ctx, root, n, storage, stream=None):
    _check(ctx, lib().rbs_broadcast_basis(ctx, int(root), int(n), _ptr(storage),
                                          0 if storage is None else storage.numel(), _stream(stream)),
           "rbs_broadcast_basis")


def rbs_set_virtual_slabs(ctx, G):
    _check(ctx, lib().rbs_set_virtual_slabs(ctx, int(G)), "rbs_set_virtual_slabs")


def rbs_nccl_unique_id():
    buf = (C.c_char * 128)()
    _check(None, lib().rbs_nccl_unique_id(buf, 128), "rbs_nccl_unique_id")
    return bytes(buf)


def rbs_dist_init(ctx, nccl_id: bytes, nranks, rank, ghost=3):
    buf = (C.c_char * 128).from_buffer_copy(nccl_id)
    _check(ctx, lib().rbs_dist_init(ctx, buf, int(nranks), int(rank), int(ghost)), "rbs_dist_init")


def rbs_local_range(ctx):
    v = [C.c_int64() for _ in range(6)]
    _check(ctx, lib().rbs_local_range(ctx, *[C.byref(x) for x in v]), "rbs_local_range")
    return dict(zip(("z0", "z1", "g0", "g1", "n_stored", "n_owned"), (x.value for x in v)))


def rbs_basis_storage_size(ctx, n):
    s = C.c_size_t()
    _check(ctx, lib().rbs_basis_storage_size(ctx, int(n), C.byref(s)), "rbs_basis_storage_size")
    return s.value


def rbs_load_basis(ctx, n, W_dev, ldw, ANq_host, fn_host, storage, stream=None):
    _check(ctx, lib().rbs_load_basis(ctx, int(n), _ptr(W_dev), int(ldw), _ptr(ANq_host),
                                     _ptr(fn_host), _ptr(storage), storage.numel(),
                                     _stream(stream)), "rbs_load_basis")


def rbs_get_offline_blocks(ctx, Q, n):
    A = np.empty((Q, n, n))
    f = np.empty(n)
    _check(ctx, lib().rbs_get_offline_blocks(ctx, _ptr(A), _ptr(f)), "rbs_get_offline_blocks")
    return A, f


def rbs_default_opts(**kw):
    o = rbs_solve_opts()
    lib().rbs_default_opts(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def rbs_solve_workspace_size(ctx, B, opts):
    s = C.c_size_t()
    _check(ctx, lib().rbs_solve_workspace_size(ctx, int(B), C.byref(opts), C.byref(s)),
           "rbs_solve_workspace_size")
    return s.value


def rbs_solve_batch(ctx, B, mu_host, opts, rhs_dev, X, iters, qstatus, relres, true_relres,
                    a_n, history, workspace, stream=None):
    _check(ctx, lib().rbs_solve_batch(ctx, int(B), _ptr(mu_host), C.byref(opts), _ptr(rhs_dev),
                                      _ptr(X), _ptr(iters), _ptr(qstatus), _ptr(relres),
                                      _ptr(true_relres), _ptr(a_n), _ptr(history),
                                      _ptr(workspace), workspace.numel(), _stream(stream)),
           "rbs_solve_batch")


def rbs_last_n_active(ctx, B):
    out = np.zeros(B, dtype=np.int32)
    _check(ctx, lib().rbs_last_n_active(ctx, _ptr(out)), "rbs_last_n_active")
    return out


def rbs_last_launch_count(ctx):
    return int(lib().rbs_last_launch_count(ctx))


RBS_K_NCLASS = 7


def rbs_last_profile(ctx):
    ms = np.zeros(RBS_K_NCLASS)
    cnt = np.zeros(RBS_K_NCLASS, dtype=np.int64)
    _check(ctx, lib().rbs_last_profile(ctx, _ptr(ms), _ptr(cnt)), "rbs_last_profile")
    return {lib().rbs_kernel_class_name(k).decode(): (float(ms[k]), int(cnt[k]))
            for k in range(RBS_K_NCLASS)}


def rbs_kernel_class_name(k):
    return lib().rbs_kernel_class_name(int(k)).decode()


def rbs_greedy_workspace_size(ctx, n_train, n_max):
    s = C.c_size_t()
    _check(ctx, lib().rbs_greedy_workspace_size(ctx, int(n_train), int(n_max), C.byref(s)),
           "rbs_greedy_workspace_size")
    return s.value


def rbs_build_greedy(ctx, mu_train, n_max, mode, snapshot_tol, drop_tol, W_out, workspace,
                     stream=None, phi_train=None, terms_dev=None):
    """phi_train (nt, R) + terms_dev (R, N): affine right-hand sides (rbs_build_greedy_affine);
    the result's fn is then (R, n) = W^T f_r."""
    mu_train = np.ascontiguousarray(mu_train, dtype=np.float64)
    nt, P = mu_train.shape
    R = 0 if phi_train is None else int(np.shape(phi_train)[1])
    ANq = np.zeros((P, n_max, n_max))
    fn = np.zeros((max(R, 1), n_max))
    n_out = C.c_int(0)
    rej = C.c_int(0)
    sel = np.full(n_max, -1, dtype=np.int32)
    ind = np.full(n_max, np.nan)
    its = np.zeros(n_max, dtype=np.int32)
    if R == 0:
        _check(ctx, lib().rbs_build_greedy(ctx, nt, _ptr(mu_train), int(n_max), int(mode),
                                           float(snapshot_tol), float(drop_tol), _ptr(W_out),
                                           _ptr(ANq), _ptr(fn), C.byref(n_out), _ptr(sel), _ptr(ind),
                                           _ptr(its), C.byref(rej), _ptr(workspace),
                                           workspace.numel(), _stream(stream)), "rbs_build_greedy")
    else:
        phi = np.ascontiguousarray(phi_train, dtype=np.float64)
        _check(ctx, lib().rbs_build_greedy_affine(ctx, nt, _ptr(mu_train), R, _ptr(phi), _ptr(terms_dev),
                                                  int(n_max), int(mode), float(snapshot_tol),
                                                  float(drop_tol), _ptr(W_out), _ptr(ANq), _ptr(fn),
                                                  C.byref(n_out), _ptr(sel), _ptr(ind), _ptr(its),
                                                  C.byref(rej), _ptr(workspace), workspace.numel(),
                                                  _stream(stream)), "rbs_build_greedy_affine")
    n = n_out.value
    fn = fn[:, :n].copy()
    return dict(n=n, ANq=ANq[:, :n, :n].copy(), fn=fn[0] if R == 0 else fn, selected=sel[:n].copy(),
                indicator=ind[:n].copy(), snap_iters=its[:n].copy(), n_rejected=rej.value)


# ---- convenience wrapper -----------------------------------------------------
class Solver:
    """Owns a context plus the torch buffers it borrows (storage, workspace)."""

    def __init__(self, dim, m, blocks=None, device=0, rhs_constant=1.0, faces=None):
        """blocks: thermal-block operator; or faces: (Q, dim, (m+1) m^(dim-1)) face
        coefficients of a general affine operator (rbs_set_operator_faces)."""
        import torch
        self.torch = torch
        self.device = torch.device("cuda", device)
        torch.cuda.set_device(self.device)
        self.ctx = rbs_create(device)
        self.dim, self.m = int(dim), int(m)
        self.N = self.m ** self.dim
        if faces is not None:
            f = torch.as_tensor(np.ascontiguousarray(faces), dtype=torch.float64)
            self._faces = f.reshape(f.shape[0], -1).contiguous().to(self.device)   # kept alive (borrowed)
            self.blocks = None
            self.Q = int(self._faces.shape[0])
            rbs_set_operator_faces(self.ctx, dim, m, self.Q, self._faces)
        else:
            self._faces = None
            self.blocks = tuple(blocks)
            self.Q = int(np.prod(self.blocks))
            rbs_set_operator_blocks(self.ctx, dim, m, blocks)
        rbs_set_rhs_constant(self.ctx, rhs_constant)
        self.n = None
        self._storage = None
        self._ws = {}

    def __del__(self):
        try:
            rbs_destroy(self.ctx)
        except Exception:
            pass

    def _bytes(self, nbytes):
        return self.torch.empty(int(nbytes), dtype=self.torch.uint8, device=self.device)

    def affine_rhs(self, phi, terms, stream=None):
        """f(mu_b) = sum_r phi[b, r] terms[r] on the device -> (B, N) tensor for solve_batch(rhs=)."""
        torch = self.torch
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        B, R = phi.shape
        t = terms if torch.is_tensor(terms) else torch.as_tensor(np.ascontiguousarray(terms), dtype=torch.float64)
        t = t.to(self.device).contiguous()
        out = torch.empty((B, self.N), dtype=torch.float64, device=self.device)
        rbs_affine_rhs(self.ctx, B, R, phi, t, out, stream)
        return out

    def set_rhs_terms(self, terms):
        """Affine right-hand side f(mu) = sum_r phi_r(mu) f_r (rbs_set_rhs_terms): terms (R, N)
        array or tensor; the rows are kept on the device (borrowed by the library).  Load
        the basis afterwards."""
        torch = self.torch
        t = terms if torch.is_tensor(terms) else torch.as_tensor(np.ascontiguousarray(terms))
        self._terms = t.to(device=self.device, dtype=torch.float64).contiguous()
        rbs_set_rhs_terms(self.ctx, [self._terms[r] for r in range(self._terms.shape[0])])
        self._ws.clear()
        return self

    def set_param_map(self, P, theta_aff=None, phi_aff=None):
        """theta(mu) = theta_aff [1; mu], phi(mu) = phi_aff [1; mu] (rbs_set_param_map)."""
        rbs_set_param_map(self.ctx, P, theta_aff, phi_aff)
        self.P = int(P)
        return self

    def set_labels(self, labels):
        """Cell-label operator (rbs_set_operator_labels): labels (m+1)^dim uint8, x fastest."""
        torch = self.torch
        lab = torch.as_tensor(np.ascontiguousarray(labels, dtype=np.uint8)).to(self.device)
        Q = int(lab.max().item()) + 1
        self._faces = self._bytes(rbs_operator_labels_size(self.dim, self.m, Q))
        rbs_set_operator_labels(self.ctx, self.dim, self.m, Q, lab, self._faces)
        self.Q, self.blocks, self.n = Q, None, None
        self._ws.clear()
        return self

    def comm_init(self, nccl_id: bytes, nranks, rank):
        """Query sharding: an NCCL communicator over the ranks (rbs_comm_init)."""
        rbs_comm_init(self.ctx, nccl_id, nranks, rank)
        return self

    def broadcast_basis(self, root, n, stream=None):
        """Collective: the basis of `root` to every rank (rbs_broadcast_basis)."""
        if self._storage is None or self.n != n:
            self._storage = self._bytes(rbs_basis_storage_size(self.ctx, n))
        rbs_broadcast_basis(self.ctx, root, n, self._storage, stream)
        self.n = n
        self._ws.clear()
        return self

    def set_slabs(self, G):
        """Mesh-slab mode (3D, RBCG): solve slab by slab with G z-slabs (1 = off)."""
        rbs_set_virtual_slabs(self.ctx, G)
        self._ws.clear()
        return self

    def dist_init(self, nccl_id: bytes, nranks, rank, ghost=3):
        """Mesh slabs over ranks: this context becomes rank's slab (rbs_dist_init)."""
        rbs_dist_init(self.ctx, nccl_id, nranks, rank, ghost)
        r = rbs_local_range(self.ctx)
        self.N = r["n_stored"]
        self.local = r
        self._ws.clear()
        return self

    def load_basis(self, W, ANq=None, fn=None, stream=None):
        """W: (N, n) array (numpy or torch); stored column-major on the device."""
        torch = self.torch
        Wt = torch.as_tensor(np.asarray(W) if not torch.is_tensor(W) else W, dtype=torch.float64)
        n = Wt.shape[1]
        Wc = Wt.t().contiguous().to(self.device)  # (n, N) row-major == (N, n) column-major
        self._storage = self._bytes(rbs_basis_storage_size(self.ctx, n))
        A = None if ANq is None else np.ascontiguousarray(ANq, dtype=np.float64)
        f = None if fn is None else np.ascontiguousarray(fn, dtype=np.float64)
        rbs_load_basis(self.ctx, n, Wc, self.N, A, f, self._storage, stream)
        self.n = n
        self._ws.clear()
        return self

    def offline_blocks(self):
        return rbs_get_offline_blocks(self.ctx, self.Q, self.n)

    def opts(self, **kw):
        return rbs_default_opts(**kw)

    def workspace(self, B, opts):
        key = (B, opts.method, opts.max_iter, opts.record_history, opts.x_location)
        if key not in self._ws:
            self._ws[key] = self._bytes(rbs_solve_workspace_size(self.ctx, B, opts))
        return self._ws[key]

    def solve_batch(self, mu, rhs=None, X=None, stream=None, want_a_n=True, **kw):
        """mu: (B, P) host array.  rhs: optional (B, N) cuda tensor.  Returns dict."""
        torch = self.torch
        o = self.opts(**kw)
        mu = np.ascontiguousarray(mu, dtype=np.float64)
        B = mu.shape[0]
        nx = self.local["n_owned"] if getattr(self, "local", None) else self.N   # ranks: owned nodes
        if X is None:
            if o.x_location == RBS_MEM_HOST:
                X = torch.empty((B, nx), dtype=torch.float64, pin_memory=True)
            else:
                X = torch.empty((B, nx), dtype=torch.float64, device=self.device)
        its = np.zeros(B, dtype=np.int32)
        st = np.zeros(B, dtype=np.int32)
        rel = np.zeros(B)
        trr = np.zeros(B)
        a_n = np.zeros((B, max(self.n or 0, 1))) if want_a_n else None
        hist = np.full((B, o.max_iter + 1), np.nan) if o.record_history else None
        ws = self.workspace(B, o)
        rbs_solve_batch(self.ctx, B, mu, o, rhs, X, its, st, rel, trr, a_n, hist, ws, stream)
        out = dict(X=X, its=its, status=[QSTATUS[int(s)] for s in st], qstatus=st, relres=rel,
                   true_relres=trr, a_n=None if a_n is None else a_n[:, :(self.n or 0)],
                   launches=rbs_last_launch_count(self.ctx), n_active=rbs_last_n_active(self.ctx, B))
        if o.profile:
            out["profile"] = rbs_last_profile(self.ctx)
        if hist is not None:
            out["history"] = [hist[b, :its[b] + 1].copy() for b in range(B)]
        return out

    def build_greedy(self, mu_train, n_max, adaptive=True, snapshot_tol=1e-12, drop_tol=1e-10,
                     stream=None, load=True, phi_train=None, terms=None, samples=False, batched=False):
        """mu_train (nt, P).  Affine right-hand sides: phi_train (nt, R) and terms (R, N).
        samples=True: no selection, adaptive snapshots at mu_train in order (RBS_GREEDY_SAMPLES,
        the fine-grid half of the multi-fidelity approach)."""
        torch = self.torch
        mu_train = np.ascontiguousarray(mu_train, dtype=np.float64)
        Wcol = torch.zeros((n_max, self.N), dtype=torch.float64, device=self.device)
        ws = self._bytes(rbs_greedy_workspace_size(self.ctx, mu_train.shape[0], n_max))
        tdev = None
        if phi_train is not None:
            tdev = terms if torch.is_tensor(terms) else torch.as_tensor(np.ascontiguousarray(terms))
            tdev = tdev.to(device=self.device, dtype=torch.float64).contiguous()
        res = rbs_build_greedy(self.ctx, mu_train, n_max,
                               (RBS_GREEDY_SAMPLES_BATCH if batched else RBS_GREEDY_SAMPLES) if samples else
                               (RBS_GREEDY_ADAPTIVE if adaptive else RBS_GREEDY_PLAIN),
                               snapshot_tol, drop_tol, Wcol, ws, stream, phi_train, tdev)
        n = res["n"]
        res["W"] = Wcol[:n].t()  # (N, n) view of the column-major result
        if load:
            fn1 = res["fn"] if phi_train is None else res["fn"][0]
            self.load_basis(res["W"], res["ANq"], fn1, stream)
        return res
