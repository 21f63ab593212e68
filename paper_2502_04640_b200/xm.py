"""Thin ctypes binding of libxm (include/xm.h).  Argument marshalling only:
every step of the path runs in the CUDA library; there is no CPU fallback —
importing this module fails loudly when libxm.so is missing.

Arrays may be numpy arrays (host) or torch tensors (host or CUDA); outputs are
numpy arrays unless a torch tensor is passed in ``out``.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libxm.so")

XM_OK, XM_UNCERTIFIED, XM_NOT_CONVERGED = 0, 2, 3
STATUS_NAMES = {0: "OK", 2: "UNCERTIFIED", 3: "NOT_CONVERGED", -1: "EINVAL", -2: "EDISCONNECTED",
                -3: "ENOMEM", -4: "ECUDA", -5: "ENCCL", -6: "ERETRACT", -7: "EESCAPE",
                -8: "EINFEASIBLE", -9: "EDEGENERATE", -10: "ESTATE"}


class XMError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS_NAMES.get(code, str(code))


class Options(ctypes.Structure):
    _fields_ = [("grad_tol", ctypes.c_double), ("delta0_coef", ctypes.c_double),
                ("delta_max_mult", ctypes.c_double), ("rho_prime", ctypes.c_double),
                ("tcg_kappa", ctypes.c_double), ("tcg_theta", ctypes.c_double),
                ("eig_tol", ctypes.c_double), ("cert_tol", ctypes.c_double),
                ("scale_floor", ctypes.c_double), ("tcg_max_inner", ctypes.c_int32),
                ("max_outer", ctypes.c_int32), ("rank_cap", ctypes.c_int32),
                ("lanczos_max", ctypes.c_int32), ("refresh_every", ctypes.c_int32),
                ("profile", ctypes.c_int32), ("cert_cholesky", ctypes.c_int32),
                ("spmm_kernel", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("scale_reg", ctypes.c_double), ("implicit_q", ctypes.c_int32)]


class SolveInfo(ctypes.Structure):
    _fields_ = [("f", ctypes.c_double), ("grad_norm", ctypes.c_double),
                ("lambda_min", ctypes.c_double), ("normQ", ctypes.c_double),
                ("s_min", ctypes.c_double), ("r", ctypes.c_int32), ("certified", ctypes.c_int32),
                ("converged", ctypes.c_int32), ("escapes", ctypes.c_int32),
                ("outer_iters", ctypes.c_int64), ("hvps", ctypes.c_int64),
                ("spmms", ctypes.c_int64), ("lanczos_steps", ctypes.c_int64)]


class Certificate(ctypes.Structure):
    _fields_ = [("lambda_min", ctypes.c_double), ("lambda_lower", ctypes.c_double),
                ("rho_dual", ctypes.c_double),
                ("rho_hat", ctypes.c_double), ("rho_lower", ctypes.c_double),
                ("eta", ctypes.c_double), ("eta_E", ctypes.c_double),
                ("rho_lower_rigorous", ctypes.c_double), ("eta_rigorous", ctypes.c_double),
                ("kkt_resid", ctypes.c_double), ("grad_norm", ctypes.c_double),
                ("trace_X", ctypes.c_double), ("normQ", ctypes.c_double),
                ("lanczos_steps", ctypes.c_int32), ("certified", ctypes.c_int32),
                ("method", ctypes.c_int32), ("lower_rigorous", ctypes.c_int32)]


class BatchResult(ctypes.Structure):
    _fields_ = [("f", ctypes.c_double), ("grad_norm", ctypes.c_double),
                ("lambda_min", ctypes.c_double), ("normQ", ctypes.c_double),
                ("r", ctypes.c_int32), ("certified", ctypes.c_int32), ("status", ctypes.c_int32),
                ("hvps", ctypes.c_int32), ("outer_iters", ctypes.c_int32),
                ("lanczos_steps", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [("kernel_launches", ctypes.c_int64), ("spmm_calls", ctypes.c_int64),
                ("spmm_rows", ctypes.c_int64), ("spmm_ms", ctypes.c_double),
                ("spmm_timed", ctypes.c_int64), ("spmm_alg_bytes", ctypes.c_double), ("ms_build", ctypes.c_double),
                ("ms_solve", ctypes.c_double), ("ms_certify", ctypes.c_double),
                ("ms_round", ctypes.c_double), ("n_dup", ctypes.c_int64), ("E", ctypes.c_int64),
                ("nnzb_S", ctypes.c_int64), ("q_bytes", ctypes.c_int64)]


def _to_dict(s: ctypes.Structure) -> dict:
    return {k: getattr(s, k) for k, _ in s._fields_}


_P = ctypes.c_void_p
_SIGS = {
    "xm_default_options": (None, [_P]),
    "xm_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "xm_last_error": (ctypes.c_char_p, [_P]),
    "xm_create": (ctypes.c_int, [ctypes.POINTER(_P), ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P, _P]),
    "xm_destroy": (None, [_P]),
    "xm_nccl_unique_id": (ctypes.c_int, [_P]),
    "xm_shard_rows": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _P, _P, _P]),
    "xm_build_Q": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, _P, _P, _P, _P]),
    "xm_solve": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_double, _P]),
    "xm_certify": (ctypes.c_int, [_P, _P, _P]),
    "xm_round_recover": (ctypes.c_int, [_P, _P, _P, _P, _P, _P]),
    "xm_edge_residuals": (ctypes.c_int, [_P, _P]),
    "xm_xm2": (ctypes.c_int, [_P, ctypes.c_double, _P, _P, _P]),
    "xm_get_S_pattern": (ctypes.c_int, [_P, _P, _P, _P]),
    "xm_get_Q_rows": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, _P]),
    "xm_set_Q": (ctypes.c_int, [_P, ctypes.c_int32, _P]),
    "xm_spmm": (ctypes.c_int, [_P, _P, _P, ctypes.c_int32]),
    "xm_grad": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_int32]),
    "xm_hvp": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_int32]),
    "xm_tcg": (ctypes.c_int, [_P, _P, ctypes.c_int32, ctypes.c_double, ctypes.c_int32, _P, _P, _P, _P]),
    "xm_project": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_int32]),
    "xm_solve_batch": (ctypes.c_int, [_P, ctypes.c_int32, ctypes.c_int32, _P, ctypes.c_int64, _P,
                                      ctypes.c_int32, _P, _P]),
    "xm_retract": (ctypes.c_int, [_P, _P, _P, _P, ctypes.c_int32]),
    "xm_get_factor": (ctypes.c_int, [_P, _P, _P]),
    "xm_set_factor": (ctypes.c_int, [_P, _P, ctypes.c_int32]),
    "xm_get_stats": (ctypes.c_int, [_P, _P]),
    "xm_reset_stats": (ctypes.c_int, [_P]),
    "xm_set_profile": (ctypes.c_int, [_P, ctypes.c_int32]),
}

_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libxm.so not built ({path}); run `python -m paper_2502_04640_b200.build`")
    lib = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def default_options(**overrides) -> Options:
    o = Options()
    load_library().xm_default_options(ctypes.byref(o))
    for k, v in overrides.items():
        if not hasattr(o, k):
            raise KeyError(k)
        setattr(o, k, v)
    return o


def shard_rows(N: int, world: int, rank: int):
    """(f0, f1, nfpr): frames [f0, f1) of `rank` (area-balanced, 32-frame
    aligned bands of the lower triangle), nfpr = the largest band
    (xm_shard_rows; host-only, no GPU needed)."""
    f0, f1, nf = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    st = load_library().xm_shard_rows(int(N), int(world), int(rank), ctypes.byref(f0),
                                      ctypes.byref(f1), ctypes.byref(nf))
    if st != 0:
        raise XMError(st, "xm_shard_rows")
    return f0.value, f1.value, nf.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = load_library().xm_nccl_unique_id(buf)
    if st != 0:
        raise XMError(st, "ncclGetUniqueId")
    return buf.raw


LOOPBACK_MAGIC = b"XM-LOOPBACK"


def loopback_id(token: str) -> bytes:
    """128-byte id selecting the in-process loopback group (include/xm.h
    XM_LOOPBACK_MAGIC): `world` Contexts created with it, one host thread each,
    run the world > 1 path on one GPU without NCCL."""
    raw = LOOPBACK_MAGIC + b"\0" + token.encode()
    if len(raw) > 128:
        raise ValueError("token too long")
    return raw.ljust(128, b"\0")


# --------------------------------------------------------------- marshalling
def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _in_ptr(x, dtype, keep: list):
    """Pointer to caller data (numpy → host pointer, torch → its data_ptr)."""
    if x is None:
        return None
    if _is_torch(x):
        import torch
        tdt = {np.float64: torch.float64, np.int32: torch.int32}[dtype]
        if x.dtype != tdt or not x.is_contiguous():
            x = x.to(tdt).contiguous()
        keep.append(x)
        return ctypes.c_void_p(x.data_ptr())
    a = np.ascontiguousarray(x, dtype=dtype)
    keep.append(a)
    return ctypes.c_void_p(a.ctypes.data)


def _out_arr(out, shape, dtype):
    if out is not None:
        return out, ctypes.c_void_p(out.data_ptr() if _is_torch(out) else out.ctypes.data)
    a = np.empty(shape, dtype=dtype)
    return a, ctypes.c_void_p(a.ctypes.data)


class Context:
    """One libxm context (one process per GPU)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1,
                 nccl_id: Optional[bytes] = None, options: Optional[Options] = None,
                 stream: Optional[int] = None, **opt_overrides):
        self.lib = load_library()
        self.h = ctypes.c_void_p()
        opts = options if options is not None else default_options(**opt_overrides)
        idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id else None
        st = self.lib.xm_create(ctypes.byref(self.h), device, rank, world, idbuf,
                                ctypes.byref(opts), ctypes.c_void_p(stream) if stream else None)
        self._check(st, "xm_create")
        self.options = opts
        self.N = self.M = self.n = 0
        self.E_user = 0
        self.r = 0

    # ------------------------------------------------------------------
    def _check(self, st: int, what: str, ok=(0,)):
        if st in ok:
            return st
        detail = ""
        if self.h:
            d = self.lib.xm_last_error(self.h)
            detail = d.decode() if d else ""
        raise XMError(st, f"{what}: {detail or self.lib.xm_strerror(st).decode()}")

    def close(self):
        if self.h:
            self.lib.xm_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ------------------------------------------------------------------ path
    def build_Q(self, N, M, frame, landmark, pts, w=None):
        keep = []
        E = int(frame.shape[0])
        st = self.lib.xm_build_Q(self.h, int(N), int(M), E, _in_ptr(frame, np.int32, keep),
                                 _in_ptr(landmark, np.int32, keep), _in_ptr(pts, np.float64, keep),
                                 _in_ptr(w, np.float64, keep))
        self._check(st, "xm_build_Q")
        self.N, self.M, self.n = int(N), int(M), 3 * int(N)
        self.E_user = E

    def solve(self, r0: int = 3, tol: float = 0.0):
        info = SolveInfo()
        st = self.lib.xm_solve(self.h, int(r0), float(tol), ctypes.byref(info))
        self._check(st, "xm_solve", ok=(0, 2, 3))
        self.r = info.r
        return st, _to_dict(info)

    def certify(self, want_vector: bool = False, out=None):
        c = Certificate()
        vec, vp = (None, None)
        if want_vector:
            vec, vp = _out_arr(out, (self.n,), np.float64)
        st = self.lib.xm_certify(self.h, ctypes.byref(c), vp)
        self._check(st, "xm_certify")
        d = _to_dict(c)
        if want_vector:
            d["v"] = vec
        return d

    def round_recover(self):
        R = np.empty((self.N, 3, 3))
        s = np.empty(self.N)
        t = np.empty((self.N, 3))
        p = np.empty((max(self.M, 1), 3))
        nf = ctypes.c_int32()
        st = self.lib.xm_round_recover(self.h, R.ctypes.data, s.ctypes.data, t.ctypes.data,
                                       p.ctypes.data, ctypes.byref(nf))
        self._check(st, "xm_round_recover")
        return dict(R=R, s=s, t=t, p=p[: self.M], n_flipped=int(nf.value))

    def edge_residuals(self):
        """Eq. (3) summand per measurement of the last build input (xm.h)."""
        res = np.empty(max(self.E_user, 1))
        self._check(self.lib.xm_edge_residuals(self.h, res.ctypes.data), "xm_edge_residuals")
        return res[: self.E_user]

    def xm2(self, drop_fraction: float = 0.1):
        """XM² step (xm.h): drop, restore, rebuild Q.  Returns (keep mask over
        the original input, n_dropped, n_restored); solve / certify / round again."""
        keep = np.zeros(max(self.E_user, 1), dtype=np.uint8)
        nd, nr = ctypes.c_int64(), ctypes.c_int64()
        self._check(self.lib.xm_xm2(self.h, float(drop_fraction), keep.ctypes.data, ctypes.byref(nd),
                                    ctypes.byref(nr)), "xm_xm2")
        return keep[: self.E_user].astype(bool), int(nd.value), int(nr.value)

    def round_recover_into(self, R, s, t, p):
        """Same as round_recover, writing into caller buffers (torch tensors on
        the device or pinned host, or numpy arrays)."""
        def ptr(x):
            return ctypes.c_void_p(x.data_ptr() if _is_torch(x) else x.ctypes.data)
        nf = ctypes.c_int32()
        st = self.lib.xm_round_recover(self.h, ptr(R), ptr(s), ptr(t), ptr(p), ctypes.byref(nf))
        self._check(st, "xm_round_recover")
        return int(nf.value)

    # ------------------------------------------------------------------ hooks
    def S_pattern(self):
        nnzb = ctypes.c_int64()
        self._check(self.lib.xm_get_S_pattern(self.h, None, None, ctypes.byref(nnzb)), "xm_get_S_pattern")
        rowptr = np.empty(self.N + 1, dtype=np.int64)
        colidx = np.empty(max(nnzb.value, 1), dtype=np.int32)
        self._check(self.lib.xm_get_S_pattern(self.h, rowptr.ctypes.data, colidx.ctypes.data,
                                              ctypes.byref(nnzb)), "xm_get_S_pattern")
        return rowptr, colidx[: nnzb.value]

    def Q_rows(self, row0: int, nrows: int, out=None):
        arr, p = _out_arr(out, (nrows, self.n), np.float64)
        self._check(self.lib.xm_get_Q_rows(self.h, int(row0), int(nrows), p), "xm_get_Q_rows")
        return arr

    def set_Q(self, Q):
        keep = []
        n = int(Q.shape[0])
        self._check(self.lib.xm_set_Q(self.h, n // 3, _in_ptr(Q, np.float64, keep)), "xm_set_Q")
        self.N, self.M, self.n = n // 3, 0, n

    def _vec_op(self, fn, name, args, r, out=None):
        keep = []
        ptrs = [_in_ptr(a, np.float64, keep) for a in args]
        arr, p = _out_arr(out, (self.n, r), np.float64)
        self._check(fn(self.h, *ptrs, p, int(r)), name)
        return arr

    def spmm(self, V, out=None):
        r = int(V.shape[1])
        return self._vec_op(self.lib.xm_spmm, "xm_spmm", [V], r, out)

    def grad(self, Y, out=None):
        r = int(Y.shape[1])
        keep = []
        arr, p = _out_arr(out, (self.n, r), np.float64)
        f = ctypes.c_double()
        self._check(self.lib.xm_grad(self.h, _in_ptr(Y, np.float64, keep), p, ctypes.byref(f), r), "xm_grad")
        return arr, f.value

    def hvp(self, Y, V, out=None):
        keep = []
        r = int(Y.shape[1])
        arr, p = _out_arr(out, (self.n, r), np.float64)
        self._check(self.lib.xm_hvp(self.h, _in_ptr(Y, np.float64, keep), _in_ptr(V, np.float64, keep),
                                    p, r), "xm_hvp")
        return arr

    def solve_batch(self, Q, Y0, shared_Q: bool = False):
        """B small instances at once (xm_solve_batch, NEXT-4).  Q: (B, n, n) or,
        with shared_Q, one (n, n); Y0: (B, n, r0).  Returns (Y (B, n, 8), results
        as a list of dicts)."""
        Q = np.ascontiguousarray(Q, dtype=np.float64)
        Y0 = np.ascontiguousarray(Y0, dtype=np.float64)
        B, n, r0 = Y0.shape
        Yo = np.empty((B, n, 8))
        res = (BatchResult * B)()
        stride = 0 if shared_Q else n * n
        self._check(self.lib.xm_solve_batch(self.h, B, n // 3, Q.ctypes.data, stride, Y0.ctypes.data, r0,
                                            Yo.ctypes.data, ctypes.cast(res, ctypes.c_void_p)),
                    "xm_solve_batch")
        return Yo, [_to_dict(r) for r in res]

    TCG_STOP = {1: "negcurv", 2: "exceeded", 3: "converged", 4: "maxinner"}
    TCG_PATHS = {"auto": 0, "persist_sym": 1, "persist": 2, "fused": 3, "three_kernel": 4}

    def tcg(self, Y, Delta, path="auto"):
        """One tCG solve at Y (xm_tcg): returns (eta, Heta, n_hvp, stop)."""
        keep = []
        r = int(Y.shape[1])
        eta = np.empty((self.n, r))
        Heta = np.empty((self.n, r))
        nh, st = ctypes.c_int32(), ctypes.c_int32()
        self._check(self.lib.xm_tcg(self.h, _in_ptr(Y, np.float64, keep), r, float(Delta),
                                    self.TCG_PATHS[path], eta.ctypes.data, Heta.ctypes.data,
                                    ctypes.byref(nh), ctypes.byref(st)), "xm_tcg")
        return eta, Heta, nh.value, self.TCG_STOP.get(st.value, str(st.value))

    def project(self, Y, W, out=None):
        return self._vec_op(self.lib.xm_project, "xm_project", [Y, W], int(Y.shape[1]), out)

    def retract(self, Y, V, out=None):
        return self._vec_op(self.lib.xm_retract, "xm_retract", [Y, V], int(Y.shape[1]), out)

    def get_factor(self):
        r = ctypes.c_int32()
        self._check(self.lib.xm_get_factor(self.h, None, ctypes.byref(r)), "xm_get_factor")
        Y = np.empty((self.n, r.value))
        self._check(self.lib.xm_get_factor(self.h, Y.ctypes.data, ctypes.byref(r)), "xm_get_factor")
        return Y

    def set_factor(self, Y):
        keep = []
        self._check(self.lib.xm_set_factor(self.h, _in_ptr(Y, np.float64, keep), int(Y.shape[1])),
                    "xm_set_factor")

    def stats(self) -> dict:
        s = Stats()
        self._check(self.lib.xm_get_stats(self.h, ctypes.byref(s)), "xm_get_stats")
        return _to_dict(s)

    def reset_stats(self):
        self._check(self.lib.xm_reset_stats(self.h), "xm_reset_stats")

    def set_profile(self, on: bool):
        self._check(self.lib.xm_set_profile(self.h, int(bool(on))), "xm_set_profile")


def solve_scene(scene, device: int = 0, r0: int = 3, tol: float = 0.0, **opts):
    """Convenience: build Q → solve → certify → round/recover on one GPU."""
    with Context(device=device, **opts) as ctx:
        ctx.build_Q(scene.N, scene.M, scene.frame, scene.landmark, scene.pts, scene.w)
        st, info = ctx.solve(r0, tol)
        cert = ctx.certify()
        sol = ctx.round_recover()
        return st, info, cert, sol
