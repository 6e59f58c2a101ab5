"""ctypes binding of include/pmns.h — argument marshalling only.

Every numeric step runs inside libpmns.so.  Device vectors are torch float64
CUDA tensors in DEVICE ORDER (see pmns.h); the current torch stream is passed
to every call.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpmns.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libpmns.so not built ({LIB_PATH}); run __graft_entry__.build() — there is no CPU fallback")
lib = C.CDLL(LIB_PATH)

STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "ENONPERC", 3: "ESINGULAR", 4: "ENOCONV", 5: "EDIVERGED",
                6: "ENOMEM", 7: "ECUDA", 8: "ENCCL", 9: "ESTATE"}


class PmnsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Problem(C.Structure):
    _fields_ = [("dim", C.c_int32), ("n", C.c_int64 * 3), ("solid", C.POINTER(C.c_uint8)),
                ("h", C.c_double), ("rho", C.c_double), ("mu", C.c_double),
                ("body_force", C.c_double * 3), ("p_in", C.c_double), ("p_out", C.c_double),
                ("periodic", C.c_uint32), ("dt", C.c_double), ("ws_merge_h", C.c_double),
                ("ws_min_cells", C.c_int32), ("dual_layers", C.c_int32), ("mask_band", C.c_int32)]


class Sizes(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("n_c", "n_f", "N", "n_p", "n_iface", "n_coarse", "nx", "ny", "nz",
                                         "dual_unknowns", "mp_bytes", "md_bytes", "coarse_bytes",
                                         "prolong_bytes", "raw_basins", "h2d_bytes", "rank", "world",
                                         "own_lo", "own_hi")]


class MemPlan(C.Structure):
    _fields_ = [("mp_bytes", C.c_int64), ("md_bytes", C.c_int64), ("mp_flops", C.c_double),
                ("md_flops", C.c_double), ("mp_fronts", C.c_int64), ("md_fronts", C.c_int64),
                ("mp_max_pivots", C.c_int64), ("mp_max_boundary", C.c_int64), ("mp_levels", C.c_int64),
                ("krylov_bytes", C.c_int64), ("index_bytes", C.c_int64), ("max_primary_unknowns", C.c_int64),
                ("stencil_runs", C.c_int64)]


class Opts(C.Structure):
    _fields_ = [("newton_tol", C.c_double), ("krylov_tol", C.c_double), ("restart", C.c_int32),
                ("max_krylov", C.c_int32), ("max_newton", C.c_int32), ("variant", C.c_int32)]

VARIANTS = {"gPLMM": 0, "aPLMM_S": 1, "aPLMM_NS": 2}


class Report(C.Structure):
    _fields_ = [("newton_iters", C.c_int32), ("converged", C.c_int32), ("krylov_iters", C.c_int32 * 64),
                ("res_hist", C.c_double * 65), ("b0_norm", C.c_double), ("t_mg_ms", C.c_double),
                ("t_ml_ms", C.c_double), ("t_sol_ms", C.c_double), ("builds", C.c_int32),
                ("total_krylov", C.c_int32), ("kernel_launches", C.c_int64), ("n_steps", C.c_int32),
                ("step_newton", C.c_int32 * 64), ("t_setup_ms", C.c_double), ("bytes_per_iter", C.c_int64),
                ("failed_subdomain", C.c_int32)]

    def as_dict(self):
        n = self.newton_iters
        return dict(newton_iters=n, converged=bool(self.converged),
                    krylov_iters=list(self.krylov_iters[:n]), res_hist=list(self.res_hist[:n + 1]),
                    b0_norm=self.b0_norm, t_mg_ms=self.t_mg_ms, t_ml_ms=self.t_ml_ms, t_sol_ms=self.t_sol_ms,
                    builds=self.builds, total_krylov=self.total_krylov, kernel_launches=self.kernel_launches,
                    n_steps=self.n_steps, step_newton=list(self.step_newton[:self.n_steps]),
                    t_setup_ms=self.t_setup_ms, bytes_per_iter=self.bytes_per_iter,
                    failed_subdomain=self.failed_subdomain)


_vp = C.c_void_p
_SIGS = {
    "pmns_create": (C.c_int, [C.POINTER(Problem), C.c_int32, C.POINTER(_vp)]),
    "pmns_destroy": (None, [_vp]),
    "pmns_last_error": (C.c_char_p, []),
    "pmns_query": (C.c_int, [_vp, C.POINTER(Sizes)]),
    "pmns_memory_plan": (C.c_int, [_vp, C.POINTER(MemPlan)]),
    "pmns_export_layout": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pmns_permute": (C.c_int, [_vp, _vp, _vp, C.c_int32, _vp]),
    "pmns_residual": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "pmns_apply_jacobian": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "pmns_apply_jacobian_fused": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "pmns_apply_jacobian_modified": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "pmns_build_preconditioner": (C.c_int, [_vp, _vp, _vp]),
    "pmns_apply_preconditioner": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "pmns_apply_mg": (C.c_int, [_vp, _vp, _vp, _vp]),
    "pmns_newton_solve": (C.c_int, [_vp, _vp, _vp, C.POINTER(Opts), C.POINTER(Report), _vp]),
    "pmns_solve_steady": (C.c_int, [_vp, _vp, C.POINTER(Opts), C.POINTER(Report), _vp]),
    "pmns_solve_steady_host": (C.c_int, [_vp, _vp, C.POINTER(Opts), C.POINTER(Report)]),
    "pmns_solve_continuation_host": (C.c_int, [_vp, _vp, C.c_int32, C.POINTER(Opts), C.POINTER(Report)]),
    "pmns_solve_transient_host": (C.c_int, [_vp, _vp, C.c_int32, C.POINTER(Opts), C.POINTER(Report)]),
    "pmns_solve_transient": (C.c_int, [_vp, _vp, C.c_int32, C.POINTER(Opts), C.POINTER(Report), _vp]),
    "pmns_coarse_solve": (C.c_int, [_vp, _vp, C.c_int32, C.POINTER(Opts), C.POINTER(Report), _vp]),
    "pmns_solve_continuation": (C.c_int, [_vp, _vp, C.c_int32, C.POINTER(Opts), C.POINTER(Report), _vp]),
    "pmns_profile": (C.c_int, [_vp, C.c_int32]),
    "pmns_profile_query": (C.c_int, [_vp, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                     C.POINTER(C.c_int64)]),
    "pmns_release_cache": (None, []),
    "pmns_comm_unique_id": (C.c_int, [_vp]),
    "pmns_set_comm": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp]),
    "pmns_loopback_create": (_vp, [C.c_int32]),
    "pmns_halo_plan": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _vp]),
    "pmns_loopback_destroy": (None, [_vp]),
    "pmns_set_comm_loopback": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp]),
    "pmns_apply_mp": (C.c_int, [_vp, _vp, _vp, _vp]),
    "pmns_apply_md": (C.c_int, [_vp, _vp, _vp, _vp]),
    "pmns_dgemm": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double, _vp, C.c_int32, C.c_int64,
                             _vp, C.c_int32, C.c_int64, C.c_double, _vp, C.c_int32, C.c_int64, C.c_int32, _vp]),
    "pmns_dense_inverse": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)


def _check(st, ok=(0,)):
    if st not in ok:
        raise PmnsError(st, lib.pmns_last_error().decode())
    return st


def problem_from_config(cfg: dict, image: np.ndarray):
    """Build the C problem struct from a configs/*.json dict and its image."""
    img = np.ascontiguousarray(image, dtype=np.uint8)
    nz, ny, nx = img.shape
    p = Problem()
    p.dim = int(cfg["dim"])
    p.n[0], p.n[1], p.n[2] = nx, ny, nz
    p.solid = img.ctypes.data_as(C.POINTER(C.c_uint8))
    p.h, p.rho, p.mu = float(cfg["h"]), float(cfg["rho"]), float(cfg["mu"])
    bf = list(cfg.get("body_force", [0, 0, 0])) + [0, 0, 0]
    for a in range(3):
        p.body_force[a] = float(bf[a])
    p.p_in, p.p_out = float(cfg.get("p_in") or 0.0), float(cfg.get("p_out") or 0.0)
    per = cfg.get("periodic", [False, False])
    p.periodic = (1 if per[0] else 0) | (2 if per[1] else 0)
    p.dt = float(cfg.get("dt") or 0.0)
    p.ws_merge_h = float(cfg["ws_merge_h"])
    p.ws_min_cells = int(cfg["ws_min_cells"])
    p.dual_layers = int(cfg.get("dual_layers", 1))
    p.mask_band = int(cfg.get("mask_band", 2))
    return p, img


def default_opts(**kw):
    o = Opts(1e-8, 1e-9, 50, 2000, 30, 0)
    for k, v in kw.items():
        if k == "variant" and isinstance(v, str):
            v = VARIANTS[v]
        setattr(o, k, v)
    return o


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    import torch
    if not torch.cuda.is_available():      # host-only contexts: the library answers ESTATE
        return None
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class Solver:
    """One pmns context: image + physical problem, decomposition, device layout."""

    def __init__(self, cfg: dict, image: np.ndarray, device: int = 0):
        self._prob, self._img = problem_from_config(cfg, image)
        h = C.c_void_p()
        _check(lib.pmns_create(C.byref(self._prob), device, C.byref(h)))
        self.h = h
        s = Sizes()
        _check(lib.pmns_query(self.h, C.byref(s)))
        self.sizes = s
        self.N = s.N
        self.nvox = int(np.prod(image.shape))

    def close(self):
        if self.h:
            lib.pmns_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def query(self):
        s = Sizes()
        _check(lib.pmns_query(self.h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in Sizes._fields_}

    def memory_plan(self):
        m = MemPlan()
        _check(lib.pmns_memory_plan(self.h, C.byref(m)))
        return {k: getattr(m, k) for k, _ in MemPlan._fields_}

    def export_layout(self):
        s = self.query()
        perm = np.empty(s["N"], dtype=np.int64)
        lab = np.empty(self.nvox, dtype=np.int32)
        ifc = np.empty(self.nvox, dtype=np.int32)
        dptr = np.empty(s["n_iface"] + 1, dtype=np.int64)
        _check(lib.pmns_export_layout(self.h, perm.ctypes.data, lab.ctypes.data, ifc.ctypes.data,
                                      dptr.ctypes.data, None, None))
        dcells = np.empty(int(dptr[-1]), dtype=np.int64)
        mask = np.empty(s["n_f"], dtype=np.uint8)
        _check(lib.pmns_export_layout(self.h, None, None, None, dptr.ctypes.data, dcells.ctypes.data,
                                      mask.ctypes.data))
        duals = [dcells[dptr[j]:dptr[j + 1]] for j in range(s["n_iface"])]
        return dict(perm=perm, label=lab, iface=ifc, duals=duals, mask=mask.astype(bool))

    def profile(self, enable: bool):
        _check(lib.pmns_profile(self.h, 1 if enable else 0))

    def profile_query(self, kind: int):
        n, ms, by = C.c_int64(), C.c_double(), C.c_int64()
        _check(lib.pmns_profile_query(self.h, kind, C.byref(n), C.byref(ms), C.byref(by)))
        return n.value, ms.value, by.value

    # -- device-vector calls (torch float64 CUDA tensors) ------------------
    def permute(self, src, dst, to_canonical: bool):
        _check(lib.pmns_permute(self.h, _ptr(src), _ptr(dst), 1 if to_canonical else 0, _stream()))

    def residual(self, x, r, u_prev=None):
        _check(lib.pmns_residual(self.h, _ptr(x), _ptr(u_prev), _ptr(r), _stream()))

    def apply_jacobian(self, xk, v, y, b=None):
        """y = J(xk) v, or y = b - J(xk) v when b is given (fused a6/a8 form)."""
        if b is None:
            _check(lib.pmns_apply_jacobian(self.h, _ptr(xk), _ptr(v), _ptr(y), _stream()))
        else:
            _check(lib.pmns_apply_jacobian_fused(self.h, _ptr(xk), _ptr(v), _ptr(b), _ptr(y), _stream()))

    def apply_jacobian_modified(self, w, v, y):
        _check(lib.pmns_apply_jacobian_modified(self.h, _ptr(w), _ptr(v), _ptr(y), _stream()))

    def build_preconditioner(self, x_b=None):
        _check(lib.pmns_build_preconditioner(self.h, _ptr(x_b), _stream()))

    def apply_preconditioner(self, xk, v, z):
        _check(lib.pmns_apply_preconditioner(self.h, _ptr(xk), _ptr(v), _ptr(z), _stream()))

    def set_comm(self, rank, world, uid=None):
        """pmns_set_comm: own a contiguous range of primaries (multi-GPU);
        uid = 128 bytes from comm_unique_id() on rank 0 (None: partition only)."""
        buf = None
        if uid is not None:
            buf = (C.c_uint8 * 128).from_buffer_copy(bytes(uid))
        _check(lib.pmns_set_comm(self.h, int(rank), int(world), C.cast(buf, _vp) if buf is not None else None))

    def halo_plan(self, rank, world):
        """pmns_halo_plan (host-side): {(peer, kind): slots} with kind in
        fwd_recv / fwd_send / rev_send / rev_recv, and the owned ranges."""
        counts = np.zeros(4 * world + 6, dtype=np.int64)
        _check(lib.pmns_halo_plan(self.h, int(rank), int(world), counts.ctypes.data, None))
        slots = np.zeros(max(1, int(counts[:4 * world].sum())), dtype=np.int64)
        _check(lib.pmns_halo_plan(self.h, int(rank), int(world), counts.ctypes.data, slots.ctypes.data))
        out, pos = {}, 0
        for p in range(world):
            for q, kind in enumerate(("fwd_recv", "fwd_send", "rev_send", "rev_recv")):
                n = int(counts[4 * p + q])
                out[(p, kind)] = slots[pos:pos + n].copy()
                pos += n
        r = counts[4 * world:]
        return out, [(int(r[0]), int(r[1])), (int(r[2]), int(r[3])), (int(r[4]), int(r[5]))]

    def set_comm_loopback(self, rank, world, group):
        """pmns_set_comm_loopback: virtual rank `rank` of an in-process loopback
        group (loopback_create(world)); drive each rank from its own thread."""
        _check(lib.pmns_set_comm_loopback(self.h, int(rank), int(world), group))

    def apply_md(self, v, z):
        """pmns_apply_md: z = owned-dual M_d^{-1} v (zeros where no owned dual)."""
        _check(lib.pmns_apply_md(self.h, _ptr(v), _ptr(z), _stream()))

    def apply_mp(self, t, z):
        """pmns_apply_mp: z = owned-primary M_p^{-1} t (zeros elsewhere)."""
        _check(lib.pmns_apply_mp(self.h, _ptr(t), _ptr(z), _stream()))

    def apply_mg(self, v, z):
        _check(lib.pmns_apply_mg(self.h, _ptr(v), _ptr(z), _stream()))

    def newton_solve(self, x, u_prev=None, opts=None):
        rep = Report()
        o = opts or default_opts()
        st = lib.pmns_newton_solve(self.h, _ptr(x), _ptr(u_prev), C.byref(o), C.byref(rep), _stream())
        _check(st, ok=(0, 4))
        return st, rep.as_dict()

    def solve_steady(self, x, opts=None):
        rep = Report()
        o = opts or default_opts()
        st = lib.pmns_solve_steady(self.h, _ptr(x), C.byref(o), C.byref(rep), _stream())
        _check(st, ok=(0, 4))
        return st, rep.as_dict()

    def solve_transient(self, x, n_steps, opts=None):
        rep = Report()
        o = opts or default_opts()
        st = lib.pmns_solve_transient(self.h, _ptr(x), int(n_steps), C.byref(o), C.byref(rep), _stream())
        _check(st, ok=(0, 4))
        return st, rep.as_dict()

    def solve_continuation(self, x, n_incr, opts=None):
        rep = Report()
        o = opts or default_opts()
        st = lib.pmns_solve_continuation(self.h, _ptr(x), int(n_incr), C.byref(o), C.byref(rep), _stream())
        _check(st, ok=(0, 4))
        return st, rep.as_dict()

    def coarse_solve(self, x, n_ramp=2, opts=None):
        """Algorithm 1: coarse-scale steady NS solve; x (device) <- x^."""
        rep = Report()
        o = opts or Opts(0.0, 0.0, 0, 0, 0, 0)
        st = lib.pmns_coarse_solve(self.h, _ptr(x), int(n_ramp), C.byref(o), C.byref(rep), _stream())
        _check(st, ok=(0, 4))
        return st, rep.as_dict()

    def solve_steady_host(self, x_host: np.ndarray, opts=None):
        rep = Report()
        o = opts or default_opts()
        assert x_host.dtype == np.float64 and x_host.flags.c_contiguous and x_host.size == self.N
        st = lib.pmns_solve_steady_host(self.h, x_host.ctypes.data, C.byref(o), C.byref(rep))
        _check(st, ok=(0, 4))
        return st, rep.as_dict()

    def solve_transient_host(self, x_host: np.ndarray, n_steps, opts=None):
        rep = Report()
        o = opts or default_opts()
        assert x_host.dtype == np.float64 and x_host.flags.c_contiguous and x_host.size == self.N
        st = lib.pmns_solve_transient_host(self.h, x_host.ctypes.data, int(n_steps), C.byref(o), C.byref(rep))
        _check(st, ok=(0, 4))
        return st, rep.as_dict()

    def solve_continuation_host(self, x_host: np.ndarray, n_incr, opts=None):
        rep = Report()
        o = opts or default_opts()
        assert x_host.dtype == np.float64 and x_host.flags.c_contiguous and x_host.size == self.N
        st = lib.pmns_solve_continuation_host(self.h, x_host.ctypes.data, int(n_incr), C.byref(o), C.byref(rep))
        _check(st, ok=(0, 4))
        return st, rep.as_dict()


def dgemm(A, B, C, alpha=1.0, beta=0.0, transA=False):
    """pmns_dgemm on contiguous float64 CUDA tensors holding column-major
    matrices as row-major transposes: a column-major r x c matrix is a tensor
    of shape (batch, c, r).  A: (batch, k, m) (or (batch, m, k) with transA,
    the stored k x m matrix), B: (batch, n, k), C: (batch, n, m);
    C = alpha op(A) B + beta C."""
    import torch  # noqa: F401
    bt = A.shape[0]
    if transA:
        k, m = A.shape[-1], A.shape[-2]
        lda = A.shape[-1]
    else:
        k, m = A.shape[-2], A.shape[-1]
        lda = A.shape[-1]
    n = B.shape[-2]
    ldb = B.shape[-1]
    ldc = C.shape[-1]
    _check(lib.pmns_dgemm(1 if transA else 0, m, n, k, alpha, _ptr(A), lda, A.stride(0), _ptr(B), ldb, B.stride(0),
                          beta, _ptr(C), ldc, C.stride(0), bt, _stream()))


def dense_inverse(A):
    """pmns_dense_inverse in place on a square float64 CUDA tensor (its
    row-major storage read as column-major, i.e. this inverts A^T in place,
    which leaves A^{-1} in row-major terms)."""
    n = A.shape[0]
    _check(lib.pmns_dense_inverse(_ptr(A), n, A.stride(0), _stream()))


def release_cache():
    """pmns_release_cache: return cached device blocks and pooled handles."""
    lib.pmns_release_cache()


def loopback_create(world: int):
    """pmns_loopback_create: a group of `world` virtual ranks on one device."""
    g = lib.pmns_loopback_create(int(world))
    if not g:
        raise PmnsError(1, "EINVAL: loopback_create")
    return g


def loopback_destroy(group):
    lib.pmns_loopback_destroy(group)


def comm_unique_id() -> bytes:
    """pmns_comm_unique_id: a fresh NCCL unique id (128 bytes), for rank 0."""
    buf = (C.c_uint8 * 128)()
    _check(lib.pmns_comm_unique_id(C.cast(buf, _vp)))
    return bytes(buf)
