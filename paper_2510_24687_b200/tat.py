"""Thin ctypes binding of libtat (include/tat.h).  Argument marshalling only: every step of
A and A* runs in the sm_100a kernels of libtat.so.  There is no CPU fallback: if the library
is missing or a call fails, an exception is raised.

    plan = Plan(n=512, n_det=512, n_t=1024, batch=16, angles=angles)   # R=c=1, T=2 defaults
    g = plan.forward(f)        # f: float32 CUDA tensor [B, n, n]  -> g [B, n_t, n_det]
    u = plan.adjoint(g)        # A* = omega A^T (L2 adjoint, eqn:innerProducts P:L217-222)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TAT_LIB") or os.path.join(_HERE, "libtat.so")   # TAT_LIB: tuning builds

TAT_OK = 0
STATUS = {0: "TAT_OK", 1: "TAT_ERR_INVALID_ARGUMENT", 2: "TAT_ERR_UNSUPPORTED_GEOMETRY",
          3: "TAT_ERR_OUT_OF_MEMORY", 4: "TAT_ERR_CUDA"}

# every symbol include/tat.h declares
EXPORTS = ("tat_plan_create", "tat_forward", "tat_adjoint", "tat_forward_host",
           "tat_adjoint_host", "tat_plan_destroy", "tat_plan_info", "tat_plan_derive",
           "tat_plan_host_multiplier", "tat_profile_begin", "tat_profile_end",
           "tat_transpose", "tat_forward_scaled", "tat_inverse",
           "tat_residual", "tat_adjoint_step", "tat_nnls", "tat_power_norm",
           "tat_plan_set_quadrature", "tat_plan_set_interpolation", "tat_status_string",
           "tat_last_error", "tat_pair_host", "tat_host_join", "tat_nnls_converge")

QUAD_TRAPEZOID, QUAD_LOWK = 0, 1        # tat_plan_set_quadrature rules (DESIGN reading G25)
INTERP_BILINEAR, INTERP_DEAPOD = 0, 1   # tat_plan_set_interpolation rules (reading G26)


class TatError(RuntimeError):
    def __init__(self, status: int, message: str):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {message}")


class PlanInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("n_det", ctypes.c_int), ("n_t", ctypes.c_int),
                ("batch", ctypes.c_int), ("N", ctypes.c_int), ("J", ctypes.c_int),
                ("M", ctypes.c_int), ("n_ring", ctypes.c_int), ("K", ctypes.c_int),
                ("n_nodes_half", ctypes.c_int),
                ("L", ctypes.c_double), ("T_new", ctypes.c_double), ("dxi", ctypes.c_double),
                ("dlam", ctypes.c_double), ("omega", ctypes.c_double), ("dt", ctypes.c_double),
                ("h", ctypes.c_double), ("wJ", ctypes.c_double),
                ("workspace_bytes", ctypes.c_size_t), ("table_bytes", ctypes.c_size_t),
                ("launches_forward", ctypes.c_int), ("launches_adjoint", ctypes.c_int),
                ("n_targets", ctypes.c_int), ("generation", ctypes.c_uint)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libtat.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libtat.so not found at {path}; run __graft_entry__.build() "
                          "or python -m paper_2510_24687_b200.build_lib")
    lib = ctypes.CDLL(path)
    vp, i, d, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_size_t
    dp = ctypes.POINTER(ctypes.c_double)
    ip = ctypes.POINTER(ctypes.c_int)
    lib.tat_plan_create.argtypes = [ctypes.POINTER(vp), i, i, i, d, d, d, i, dp]
    lib.tat_forward.argtypes = [vp, vp, vp, vp]
    lib.tat_adjoint.argtypes = [vp, vp, vp, vp]
    lib.tat_forward_host.argtypes = [vp, vp, vp, vp]
    lib.tat_adjoint_host.argtypes = [vp, vp, vp, vp]
    lib.tat_plan_destroy.argtypes = [vp]
    lib.tat_plan_destroy.restype = None
    lib.tat_plan_info.argtypes = [vp, ctypes.POINTER(PlanInfo), ip]
    lib.tat_plan_derive.argtypes = [i, i, i, d, d, d, i, dp, ctypes.POINTER(PlanInfo), ip]
    lib.tat_plan_host_multiplier.argtypes = [i, i, i, d, d, d, dp, ctypes.POINTER(ctypes.c_float), sz]
    lib.tat_profile_begin.argtypes = [vp, i]
    lib.tat_profile_end.argtypes = [vp, ctypes.POINTER(ctypes.c_float), ip, ip]
    f32 = ctypes.c_float
    lib.tat_transpose.argtypes = [vp, vp, vp, vp]
    lib.tat_plan_set_quadrature.argtypes = [vp, i]
    lib.tat_plan_set_interpolation.argtypes = [vp, i]
    lib.tat_inverse.argtypes = [vp, vp, vp, d, vp]
    lib.tat_forward_scaled.argtypes = [vp, vp, vp, f32, vp]
    lib.tat_residual.argtypes = [vp, vp, vp, vp, vp]
    lib.tat_adjoint_step.argtypes = [vp, vp, vp, f32, i, vp, vp]
    lib.tat_nnls.argtypes = [vp, vp, vp, vp, f32, i, i, vp, vp]
    lib.tat_power_norm.argtypes = [vp, i, ctypes.c_ulonglong, dp, vp]
    lib.tat_pair_host.argtypes = [vp, vp, vp, vp, vp]
    lib.tat_host_join.argtypes = [vp, vp]
    lib.tat_nnls_converge.argtypes = [vp, vp, vp, vp, f32, i, i, d, i, vp, ip, vp]
    lib.tat_status_string.argtypes = [i]
    lib.tat_status_string.restype = ctypes.c_char_p
    lib.tat_last_error.argtypes = []
    lib.tat_last_error.restype = ctypes.c_char_p
    for name in ("tat_plan_create", "tat_forward", "tat_adjoint", "tat_forward_host",
                 "tat_adjoint_host", "tat_plan_info", "tat_plan_derive",
                 "tat_plan_host_multiplier", "tat_profile_begin", "tat_profile_end",
                 "tat_transpose", "tat_forward_scaled", "tat_inverse",
                 "tat_residual", "tat_adjoint_step", "tat_nnls", "tat_power_norm",
                 "tat_plan_set_quadrature", "tat_plan_set_interpolation", "tat_pair_host",
                 "tat_host_join", "tat_nnls_converge"):
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _check(status: int):
    if status != TAT_OK:
        raise TatError(status, load_library().tat_last_error().decode())


def _angles(angles, n_det):
    a = np.ascontiguousarray(np.asarray(angles, dtype=np.float64))
    if a.shape != (n_det,):
        raise ValueError(f"angles must have shape ({n_det},)")
    return a


def derive(n, n_det, n_t, R=1.0, c=1.0, T=2.0, batch=1, angles=None):
    """Host-only constants (tat_plan_derive).  Returns (info dict, ring indices, status)."""
    lib = load_library()
    a = _angles(angles, n_det)
    info = PlanInfo()
    ring = np.zeros(n_det, dtype=np.int32)
    st = lib.tat_plan_derive(n, n_det, n_t, R, c, T, batch,
                             a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                             ctypes.byref(info), ring.ctypes.data_as(ctypes.POINTER(ctypes.c_int)))
    return info.as_dict(), ring, st


def host_multiplier(n, n_det, n_t, R=1.0, c=1.0, T=2.0, angles=None):
    """The float32 multiplier table m'[k][j] the plan uploads (host-only)."""
    info, _, st = derive(n, n_det, n_t, R, c, T, 1, angles)
    if st not in (TAT_OK, 2):
        _check(st)
    out = np.zeros((info["K"] + 1, info["J"] + 1), dtype=np.float32)
    lib = load_library()
    a = _angles(angles, n_det)
    _check(lib.tat_plan_host_multiplier(n, n_det, n_t, R, c, T,
                                        a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                        out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), out.size))
    return out


class Plan:
    """A tat_plan: device tables + workspace for one geometry and batch size."""

    def __init__(self, n, n_det, n_t, R=1.0, c=1.0, T=2.0, batch=1, angles=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("libtat needs a CUDA device (no CPU fallback)")
        self._lib = load_library()
        torch.cuda.current_device()          # make sure a context exists on this thread
        a = _angles(angles, n_det)
        h = ctypes.c_void_p()
        _check(self._lib.tat_plan_create(ctypes.byref(h), n, n_det, n_t, R, c, T, batch,
                                         a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        self._h = h
        self.n, self.n_det, self.n_t, self.batch = n, n_det, n_t, batch
        self.quadrature = "trapezoid"
        self.interpolation = "bilinear"
        self.info = self._info()

    def _info(self):
        info = PlanInfo()
        ring = np.zeros(self.n_det, dtype=np.int32)
        _check(self._lib.tat_plan_info(self._h, ctypes.byref(info),
                                       ring.ctypes.data_as(ctypes.POINTER(ctypes.c_int))))
        d = info.as_dict()
        d["ring"] = ring
        return d

    @property
    def omega(self) -> float:
        return self.info["omega"]

    def _stream(self, stream):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream()
        return ctypes.c_void_p(s.cuda_stream)

    def _chk(self, t, shape, name):
        import torch
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
                and tuple(t.shape) == shape):
            raise ValueError(f"{name} must be a contiguous float32 CUDA tensor of shape {shape}")
        if t.data_ptr() % 16:
            raise ValueError(f"{name} must be 16-byte aligned (include/tat.h)")

    def forward(self, f, out=None, stream=None):
        """g = A f on the current (or given) torch stream; no host synchronisation."""
        import torch
        self._chk(f, (self.batch, self.n, self.n), "f")
        g = out if out is not None else torch.empty((self.batch, self.n_t, self.n_det),
                                                    device=f.device, dtype=torch.float32)
        self._chk(g, (self.batch, self.n_t, self.n_det), "g")
        _check(self._lib.tat_forward(self._h, ctypes.c_void_p(f.data_ptr()),
                                     ctypes.c_void_p(g.data_ptr()), self._stream(stream)))
        return g

    def adjoint(self, g, out=None, stream=None):
        """f = A* g (= omega A^T g) on the current (or given) torch stream."""
        import torch
        self._chk(g, (self.batch, self.n_t, self.n_det), "g")
        f = out if out is not None else torch.empty((self.batch, self.n, self.n),
                                                    device=g.device, dtype=torch.float32)
        self._chk(f, (self.batch, self.n, self.n), "f")
        _check(self._lib.tat_adjoint(self._h, ctypes.c_void_p(g.data_ptr()),
                                     ctypes.c_void_p(f.data_ptr()), self._stream(stream)))
        return f

    def set_quadrature(self, rule):
        """"trapezoid" (default, reading G9) or "lowk" (reading G25: the trapezoid plus its
        Euler-Maclaurin endpoint term at lambda = 0 for the k = 0 harmonic)."""
        code = {"trapezoid": QUAD_TRAPEZOID, "lowk": QUAD_LOWK}.get(rule, rule)
        _check(self._lib.tat_plan_set_quadrature(self._h, int(code)))
        self.quadrature = {QUAD_TRAPEZOID: "trapezoid", QUAD_LOWK: "lowk"}[int(code)]

    def set_interpolation(self, rule):
        """"bilinear" (default, the paper's) or "deapod" (reading G26: f pre-divided by the
        bilinear window K(x), A_D = A diag(1/K))."""
        code = {"bilinear": INTERP_BILINEAR, "deapod": INTERP_DEAPOD}.get(rule, rule)
        _check(self._lib.tat_plan_set_interpolation(self._h, int(code)))
        self.interpolation = {INTERP_BILINEAR: "bilinear", INTERP_DEAPOD: "deapod"}[int(code)]

    def transpose(self, g, out=None, stream=None):
        """f = A^T g (Euclidean transpose, = A* g / omega): the backward of A."""
        import torch
        self._chk(g, (self.batch, self.n_t, self.n_det), "g")
        f = out if out is not None else torch.empty((self.batch, self.n, self.n),
                                                    device=g.device, dtype=torch.float32)
        self._chk(f, (self.batch, self.n, self.n), "f")
        _check(self._lib.tat_transpose(self._h, ctypes.c_void_p(g.data_ptr()),
                                       ctypes.c_void_p(f.data_ptr()), self._stream(stream)))
        return f

    def forward_scaled(self, f, alpha: float, out=None, stream=None):
        """g = alpha A f (alpha = omega: the backward of A*)."""
        import torch
        self._chk(f, (self.batch, self.n, self.n), "f")
        g = out if out is not None else torch.empty((self.batch, self.n_t, self.n_det),
                                                    device=f.device, dtype=torch.float32)
        self._chk(g, (self.batch, self.n_t, self.n_det), "g")
        _check(self._lib.tat_forward_scaled(self._h, ctypes.c_void_p(f.data_ptr()),
                                            ctypes.c_void_p(g.data_ptr()), float(alpha),
                                            self._stream(stream)))
        return g

    def inverse(self, g, r0: float = 0.95, out=None, stream=None):
        """f = A^{-1} g (Algorithm 3, approximate universal backprojection), support |x| <= r0."""
        import torch
        self._chk(g, (self.batch, self.n_t, self.n_det), "g")
        f = out if out is not None else torch.empty((self.batch, self.n, self.n),
                                                    device=g.device, dtype=torch.float32)
        self._chk(f, (self.batch, self.n, self.n), "f")
        _check(self._lib.tat_inverse(self._h, ctypes.c_void_p(g.data_ptr()),
                                     ctypes.c_void_p(f.data_ptr()), float(r0), self._stream(stream)))
        return f

    def A(self, f):
        """Differentiable A (torch.autograd): backward = A^T."""
        return _ForwardFn.apply(f, self)

    def Astar(self, g):
        """Differentiable A* (torch.autograd): backward = omega A."""
        return _AdjointFn.apply(g, self)

    # ---- iterative driver (NNLS / projected Landweber, §4.2)
    def residual(self, f, g_obs, out=None, stream=None):
        """r = A f - g_obs (fused into the last forward kernel)."""
        import torch
        self._chk(f, (self.batch, self.n, self.n), "f")
        self._chk(g_obs, (self.batch, self.n_t, self.n_det), "g_obs")
        r = out if out is not None else torch.empty_like(g_obs)
        self._chk(r, (self.batch, self.n_t, self.n_det), "r")
        _check(self._lib.tat_residual(self._h, ctypes.c_void_p(f.data_ptr()),
                                      ctypes.c_void_p(g_obs.data_ptr()),
                                      ctypes.c_void_p(r.data_ptr()), self._stream(stream)))
        return r

    def _roi(self, roi):
        if roi is None:
            return ctypes.c_void_p(None)
        self._chk(roi, (self.n, self.n), "roi")
        return ctypes.c_void_p(roi.data_ptr())

    def adjoint_step(self, r, f, lam: float, nonneg: bool = True, roi=None, stream=None):
        """f <- Pi max(0, f - lam A* r) in place (fused into the last adjoint kernel)."""
        self._chk(r, (self.batch, self.n_t, self.n_det), "r")
        self._chk(f, (self.batch, self.n, self.n), "f")
        _check(self._lib.tat_adjoint_step(self._h, ctypes.c_void_p(r.data_ptr()),
                                          ctypes.c_void_p(f.data_ptr()), float(lam), int(nonneg),
                                          self._roi(roi), self._stream(stream)))
        return f

    def nnls(self, g_obs, f, lam: float, iters: int, nonneg: bool = True, roi=None, r_work=None,
             stream=None):
        """`iters` NNLS iterations in place on f (start value in f); enqueue-only."""
        import torch
        self._chk(g_obs, (self.batch, self.n_t, self.n_det), "g_obs")
        self._chk(f, (self.batch, self.n, self.n), "f")
        r = r_work if r_work is not None else torch.empty_like(g_obs)
        self._chk(r, (self.batch, self.n_t, self.n_det), "r_work")
        _check(self._lib.tat_nnls(self._h, ctypes.c_void_p(g_obs.data_ptr()),
                                  ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(r.data_ptr()),
                                  float(lam), int(iters), int(nonneg), self._roi(roi),
                                  self._stream(stream)))
        return f

    def nnls_converge(self, g_obs, f, lam: float, max_iters: int, rel_tol: float = 3e-3,
                      check_every: int = 1, nonneg: bool = True, roi=None, r_work=None, stream=None):
        """NNLS with the paper's stopping rule (synchronous).  Returns the
        per-image iteration counts (negative: not converged within max_iters)."""
        import torch
        self._chk(g_obs, (self.batch, self.n_t, self.n_det), "g_obs")
        self._chk(f, (self.batch, self.n, self.n), "f")
        r = r_work if r_work is not None else torch.empty_like(g_obs)
        self._chk(r, (self.batch, self.n_t, self.n_det), "r_work")
        it = np.zeros(self.batch, dtype=np.int32)
        _check(self._lib.tat_nnls_converge(self._h, ctypes.c_void_p(g_obs.data_ptr()),
                                           ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(r.data_ptr()),
                                           float(lam), int(max_iters), int(check_every), float(rel_tol),
                                           int(nonneg), self._roi(roi),
                                           it.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                           self._stream(stream)))
        return it

    def pair_host(self, f_host: np.ndarray, u_host: np.ndarray, g_host=None, stream=None):
        """Pipelined g = A f, u = A* g from / to host buffers (tat_pair_host); enqueue-only,
        results valid after join_host(stream) and a synchronisation of that stream."""
        assert f_host.dtype == np.float32 and f_host.flags.c_contiguous and f_host.shape == (self.batch, self.n, self.n)
        assert u_host.dtype == np.float32 and u_host.flags.c_contiguous and u_host.shape == (self.batch, self.n, self.n)
        gp = None
        if g_host is not None:
            assert g_host.dtype == np.float32 and g_host.flags.c_contiguous
            assert g_host.shape == (self.batch, self.n_t, self.n_det)
            gp = g_host.ctypes.data
        _check(self._lib.tat_pair_host(self._h, ctypes.c_void_p(f_host.ctypes.data), ctypes.c_void_p(gp),
                                       ctypes.c_void_p(u_host.ctypes.data), self._stream(stream)))

    def join_host(self, stream=None):
        """Make the stream wait for every copy tat_pair_host has enqueued (tat_host_join)."""
        _check(self._lib.tat_host_join(self._h, self._stream(stream)))

    def power_norm(self, iters: int = 20, seed: int = 0, stream=None) -> float:
        """Largest eigenvalue of A*A by power iteration (synchronous setup call)."""
        out = ctypes.c_double()
        _check(self._lib.tat_power_norm(self._h, int(iters), ctypes.c_ulonglong(seed),
                                        ctypes.byref(out), self._stream(stream)))
        return out.value

    def forward_host(self, f_host: np.ndarray, g_host: np.ndarray, stream=None):
        """Host-buffer variant (H2D + A + D2H on the stream); caller synchronises."""
        assert f_host.dtype == np.float32 and f_host.flags.c_contiguous
        assert g_host.dtype == np.float32 and g_host.flags.c_contiguous
        _check(self._lib.tat_forward_host(self._h, ctypes.c_void_p(f_host.ctypes.data),
                                          ctypes.c_void_p(g_host.ctypes.data), self._stream(stream)))

    def adjoint_host(self, g_host: np.ndarray, f_host: np.ndarray, stream=None):
        assert f_host.dtype == np.float32 and f_host.flags.c_contiguous
        assert g_host.dtype == np.float32 and g_host.flags.c_contiguous
        _check(self._lib.tat_adjoint_host(self._h, ctypes.c_void_p(g_host.ctypes.data),
                                          ctypes.c_void_p(f_host.ctypes.data), self._stream(stream)))

    def profile_begin(self, max_calls: int):
        _check(self._lib.tat_profile_begin(self._h, max_calls))

    def profile_end(self):
        """(stage_ms[11] summed, n_forward, n_adjoint); stages K1..K5, K5T, K4T, K3T, K2Ta,
        K2Tb, K1T."""
        ms = (ctypes.c_float * 11)()
        nf, na = ctypes.c_int(), ctypes.c_int()
        _check(self._lib.tat_profile_end(self._h, ms, ctypes.byref(nf), ctypes.byref(na)))
        return list(ms), nf.value, na.value

    def close(self):
        if getattr(self, "_h", None):
            self._lib.tat_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- torch.autograd wrappers: every pass runs in libtat's kernels
def _autograd_fns():
    import torch

    class ForwardFn(torch.autograd.Function):
        @staticmethod
        def forward(ctx, f, plan):
            ctx.plan = plan
            return plan.forward(f.contiguous())

        @staticmethod
        def backward(ctx, grad_g):
            return ctx.plan.transpose(grad_g.contiguous()), None

    class AdjointFn(torch.autograd.Function):
        @staticmethod
        def forward(ctx, g, plan):
            ctx.plan = plan
            return plan.adjoint(g.contiguous())

        @staticmethod
        def backward(ctx, grad_f):
            return ctx.plan.forward_scaled(grad_f.contiguous(), ctx.plan.omega), None

    return ForwardFn, AdjointFn


class _Lazy:
    def __init__(self, idx):
        self.idx = idx

    def apply(self, *args):
        global _FNS
        if _FNS is None:
            _FNS = _autograd_fns()
        return _FNS[self.idx].apply(*args)


_FNS = None
_ForwardFn = _Lazy(0)
_AdjointFn = _Lazy(1)
