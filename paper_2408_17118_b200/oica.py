"""Thin ctypes binding of liboica.so (include/oica.h).  Argument marshalling only.

Every step of the hot path runs in liboica's CUDA kernels; this module only converts torch
tensors / numpy arrays to pointers and status codes to exceptions.  There is no fallback:
if liboica.so is missing or the device is not sm_100a, calls raise OicaError.

Device memory comes from torch (`torch.empty(..., device="cuda")`), streams from
`torch.cuda.Stream`, and multi-process setup from `torch.distributed` (only to broadcast the
NCCL unique id).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# OICA_LIB selects another build of the library (the -DOICA_EXPERIMENTS timing build,
# paper_2408_17118_b200/build.py --experiments); bench.py refuses to run with it set
LIB_PATH = os.environ.get("OICA_LIB") or os.path.join(_HERE, "liboica.so")

OK = 0
STATUS = ["OK", "INVALID_ARGUMENT", "DIMENSION_MISMATCH", "RANK_DEFICIENT", "ALL_CANDIDATES_DEGENERATE",
          "DOMAIN", "STATE", "UNSUPPORTED_DEVICE", "OUT_OF_MEMORY", "CUDA", "NCCL", "NONFINITE"]

PREC_AUTO, PREC_FP32, PREC_TC, PREC_TC_SPLIT = 0, 1, 2, 3
SHARD_L, SHARD_M, SHARD_HYBRID = 0, 1, 2
INCLUDE_UNCONVERGED, STOP_ON_GAUSSIANITY, RAW_ARGMAX, REDUCE_X, EAGER, NO_PERSISTENT = 0x1, 0x2, 0x4, 0x8, 0x10, 0x20
MAX_CLUSTERS = 8


class OicaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.name = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        super().__init__(f"OICA_ERR_{self.name}: {msg}")


class Config(C.Structure):
    _fields_ = [("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32), ("shard_mode", C.c_int32),
                ("precision", C.c_int32), ("reserved", C.c_int32), ("stream", C.c_void_p),
                ("nccl_unique_id", C.c_void_p)]


_P = C.POINTER


class Result(C.Structure):
    _fields_ = [("W", _P(C.c_double)), ("alpha", _P(C.c_double)), ("upsilon", _P(C.c_double)),
                ("index", _P(C.c_int64)), ("iters", _P(C.c_int32)), ("n_iter", _P(C.c_int32)),
                ("cluster_size", _P(C.c_int32)), ("n_converged", _P(C.c_int32)), ("n_unconverged", _P(C.c_int32)),
                ("n_degenerate", _P(C.c_int32)), ("sum_active", _P(C.c_int64)), ("gaussian_flag", _P(C.c_uint8)),
                ("near_tie", _P(C.c_uint8)), ("n_extracted", C.c_int32), ("stopped", C.c_int32),
                ("dim", _P(C.c_int32)), ("objective", _P(C.c_double))]


class Stats(C.Structure):
    _fields_ = [("kernel_launches", C.c_int64), ("step_launches", C.c_int64), ("step_ms", C.c_double),
                ("step_flops", C.c_double), ("iterations", C.c_int64), ("sum_active", C.c_int64),
                ("precision", C.c_int32), ("slots", C.c_int32), ("step_issued_flops", C.c_double),
                ("fine_rows", C.c_int64), ("tail_iterations", C.c_int64), ("exchange_ms", C.c_double),
                ("exchange_calls", C.c_int64), ("graph_iterations", C.c_int64), ("graph_ms", C.c_double),
                ("graph_flops", C.c_double)]


class IterationRecord(C.Structure):
    _fields_ = [("component", C.c_int32), ("iteration", C.c_int32), ("L_act", C.c_int32), ("fine_rows", C.c_int32),
                ("step_ms", C.c_double), ("flops", C.c_double)]


class ClusterRecord(C.Structure):
    _fields_ = [("upsilon", C.c_double), ("alpha", C.c_double), ("q", C.c_int64), ("size", C.c_int64),
                ("iters", C.c_int32), ("valid", C.c_int32), ("objective", C.c_double)]


# every symbol include/oica.h declares (checked by tests/test_abi.py)
SIGNATURES = {
    "oica_create": (C.c_int, [_P(Config), _P(C.c_void_p)]),
    "oica_destroy": (C.c_int, [C.c_void_p]),
    "oica_status_string": (C.c_char_p, [C.c_int]),
    "oica_last_error": (C.c_char_p, [C.c_void_p]),
    "oica_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "oica_whiten": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_void_p,
                              C.c_int64, _P(C.c_double), _P(C.c_double), _P(C.c_double)]),
    "oica_set_data": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64]),
    "oica_set_data_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64]),
    "oica_init_candidates": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int64]),
    "oica_distribute_data": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                       C.c_int64, C.c_int32]),
    "oica_extract_components": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_double, C.c_uint32,
                                          _P(C.c_double), C.c_int32, _P(Result)]),
    "oica_fixed_point_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "oica_fixed_point_step_mixed": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, _P(C.c_uint8), C.c_void_p,
                                              C.c_void_p]),
    "oica_draw_candidates": (C.c_int, [C.c_void_p, C.c_int32, _P(C.c_double), C.c_int32, C.c_void_p]),
    "oica_get_candidates": (C.c_int, [C.c_void_p, _P(C.c_double), _P(C.c_double), _P(C.c_int32), _P(C.c_uint8),
                                      _P(C.c_int64), _P(C.c_int64)]),
    "oica_get_stats": (C.c_int, [C.c_void_p, _P(Stats)]),
    "oica_get_iteration_log": (C.c_int, [C.c_void_p, _P(IterationRecord), C.c_int64, _P(C.c_int64)]),
    "oica_reset_stats": (C.c_int, [C.c_void_p]),
    "oica_synchronize": (C.c_int, [C.c_void_p]),
    "oica_merge_records": (C.c_int, [_P(ClusterRecord), _P(C.c_double), C.c_int32, C.c_int32, _P(C.c_int32),
                                     _P(C.c_int64), _P(C.c_uint8)]),
    "oica_complement_basis": (C.c_int, [_P(C.c_double), C.c_int32, C.c_int32, _P(C.c_double)]),
    "oica_slot_plan": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, _P(C.c_int64), _P(C.c_int32)]),
    "oica_split_parts": (C.c_int, [C.c_int32, C.c_int32, _P(C.c_int32)]),
    "oica_deflate_basis": (C.c_int, [_P(C.c_double), C.c_int32, C.c_int32, _P(C.c_double), _P(C.c_double)]),
}

_lib = None


def lib():
    """Load liboica.so (raises if it was not built: there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OicaError(9, f"{LIB_PATH} not found; run `python -m paper_2408_17118_b200.build`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int, ctx=None):
    if status != OK:
        msg = lib().oica_last_error(ctx).decode() if ctx else lib().oica_status_string(status).decode()
        raise OicaError(status, msg)


def _dptr(t) -> int:
    """Device pointer of a CUDA torch tensor (contiguity checked by the caller)."""
    if not t.is_cuda:
        raise OicaError(1, "expected a CUDA tensor")
    return t.data_ptr()


def _ready(t):
    """The library's stream does not order itself after torch's: make the caller's pending work on
    this tensor (e.g. an asynchronous host-to-device copy) complete before the library reads it."""
    import torch
    torch.cuda.current_stream(t.device).synchronize()


def _np_ptr(a, ctype):
    return a.ctypes.data_as(_P(ctype)) if a is not None else None


def _point_to_torch_nccl():
    """liboica dlopens libnccl.so.2; prefer the copy torch ships (same process, same version)."""
    if os.environ.get("OICA_NCCL_LIB"):
        return
    try:
        import nvidia.nccl
        for d in nvidia.nccl.__path__:
            p = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(p):
                os.environ["OICA_NCCL_LIB"] = p
                return
    except Exception:
        pass


def nccl_unique_id() -> bytes:
    _point_to_torch_nccl()
    buf = C.create_string_buffer(128)
    _check(lib().oica_nccl_unique_id(buf))
    return buf.raw


def merge_records(records, W):
    """Host-only selection merge (oica_merge_records): records = list of dicts, W = n x N."""
    n = len(records)
    arr = (ClusterRecord * max(n, 1))()
    for k, r in enumerate(records):
        arr[k] = ClusterRecord(r["upsilon"], r["alpha"], r["q"], r["size"], r.get("iters", 0), r.get("valid", 1),
                               r.get("objective", r["alpha"] + 3.0))
    W = np.ascontiguousarray(W, dtype=np.float64)
    win, size, tie = C.c_int32(-1), C.c_int64(0), C.c_uint8(0)
    st = lib().oica_merge_records(arr, _np_ptr(W, C.c_double), n, W.shape[1] if W.ndim == 2 else 1,
                                  C.byref(win), C.byref(size), C.byref(tie))
    return dict(status=st, winner=win.value, size=size.value, near_tie=bool(tie.value))


def complement_basis(W, N):
    """Host-only (oica_complement_basis): orthonormal basis (N-k x N) of the complement of W's rows."""
    W = np.ascontiguousarray(np.asarray(W, dtype=np.float64).reshape(-1, N))
    k = W.shape[0]
    G = np.zeros((N - k, N))
    _check(lib().oica_complement_basis(_np_ptr(W, C.c_double) if k else None, k, N, _np_ptr(G, C.c_double)))
    return G


def slot_plan(M_global, M_local=None, precision=PREC_TC):
    """Host-only (oica_slot_plan): (slot_len, S_local) of the step kernels' split-M slots."""
    ln, S = C.c_int64(), C.c_int32()
    _check(lib().oica_slot_plan(precision, M_global, M_global if M_local is None else M_local, C.byref(ln),
                                C.byref(S)))
    return ln.value, S.value


def split_parts(L_global: int, S: int) -> int:
    """Host-only (oica_split_parts): CTAs sharing each slot's chunks for L_global active runs."""
    P = C.c_int32()
    _check(lib().oica_split_parts(L_global, S, C.byref(P)))
    return P.value


def deflate_basis(G, b):
    """Host-only (oica_deflate_basis): basis of the complement of w = G^T b inside span(G)."""
    G = np.ascontiguousarray(G, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    d, N = G.shape
    out = np.zeros((d - 1, N))
    _check(lib().oica_deflate_basis(_np_ptr(G, C.c_double), d, N, _np_ptr(b, C.c_double), _np_ptr(out, C.c_double)))
    return out


@dataclass
class Extraction:
    W: np.ndarray
    alpha: np.ndarray
    upsilon: np.ndarray
    index: np.ndarray
    iters: np.ndarray
    n_iter: np.ndarray
    cluster_size: np.ndarray
    n_converged: np.ndarray
    n_unconverged: np.ndarray
    n_degenerate: np.ndarray
    sum_active: np.ndarray
    gaussian_flag: np.ndarray
    near_tie: np.ndarray
    n_extracted: int
    stopped: bool
    dim: np.ndarray = None
    objective: np.ndarray = None   # sum y^4 / M at the accepted w (oica_result.objective)


class Context:
    """One liboica context (one device, one rank)."""

    def __init__(self, device: int = 0, precision: int = PREC_AUTO, rank: int = 0, world: int = 1,
                 shard_mode: int = SHARD_L, stream=None, nccl_id: Optional[bytes] = None):
        if world > 1 or nccl_id is not None:
            _point_to_torch_nccl()
        self._idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        cfg = Config(device, rank, world, shard_mode, precision, 0,
                     C.c_void_p(stream.cuda_stream if stream is not None else 0),
                     C.cast(self._idbuf, C.c_void_p) if self._idbuf is not None else None)
        h = C.c_void_p()
        _check(lib().oica_create(C.byref(cfg), C.byref(h)))
        self.h = h
        self.N = self.M = None
        self._keep = None

    def close(self):
        if getattr(self, "h", None):
            lib().oica_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _c(self, st):
        _check(st, self.h)

    # -- boundary
    def whiten(self, X, Xw_out, eig_floor: float = 1e-12):
        N, M = X.shape
        _ready(X)
        mean = np.zeros(N)
        V = np.zeros((N, N))
        eig = np.zeros(N)
        self._c(lib().oica_whiten(self.h, _dptr(X), N, M, X.stride(0), eig_floor, _dptr(Xw_out), Xw_out.stride(0),
                                  _np_ptr(mean, C.c_double), _np_ptr(V, C.c_double), _np_ptr(eig, C.c_double)))
        return mean, V, eig

    def set_data(self, Xw, M_global: Optional[int] = None):
        """Bind device fp32 N x M_local whitened data (borrowed: the tensor is kept alive here)."""
        if Xw.dtype.__str__() != "torch.float32" or Xw.stride(1) != 1:
            raise OicaError(1, "Xw must be an fp32 row-major CUDA tensor")
        N, M = Xw.shape
        self._keep = Xw
        _ready(Xw)
        self._c(lib().oica_set_data(self.h, _dptr(Xw), N, M, Xw.stride(0), M if M_global is None else M_global))
        self.N, self.M = N, M

    def set_data_host(self, Xw: np.ndarray, M_global: Optional[int] = None):
        Xw = np.ascontiguousarray(Xw, dtype=np.float32) if not (isinstance(Xw, np.ndarray) and Xw.dtype == np.float32
                                                                 and Xw.flags.c_contiguous) else Xw
        N, M = Xw.shape
        self._c(lib().oica_set_data_host(self.h, Xw.ctypes.data, N, M, M, M if M_global is None else M_global))
        self.N, self.M = N, M

    def set_data_host_ptr(self, ptr: int, N: int, M: int, ld: int, M_global: Optional[int] = None):
        """Host fp32 buffer by address (pinned torch tensor: tensor.data_ptr()).  The copy is only
        enqueued: a pinned buffer must stay valid and unchanged until the next extract /
        synchronize / set_data* call returns (include/oica.h)."""
        self._c(lib().oica_set_data_host(self.h, ptr, N, M, ld, M if M_global is None else M_global))
        self.N, self.M = N, M

    def distribute_data(self, X_root, N: int, M_global: int, X_out, root: int = 0):
        """C3: root's device fp32 N x M_global whitened data -> X_out on every rank (replicated for
        L-shard / hybrid, this rank's column block for M-shard).  X_root may be None off root."""
        _ready(X_out if X_root is None else X_root)
        self._c(lib().oica_distribute_data(self.h, _dptr(X_root) if X_root is not None else None, N, M_global,
                                           X_root.stride(0) if X_root is not None else M_global, _dptr(X_out),
                                           X_out.stride(0), root))

    def init_candidates(self, seed: int, L: int):
        self._c(lib().oica_init_candidates(self.h, seed & 0xFFFFFFFFFFFFFFFF, L))

    # -- hot path
    def extract(self, N_out: int, max_iter: int = 200, tol: float = 1e-10, flags: int = 0,
                W_prefix: Optional[np.ndarray] = None) -> Extraction:
        N = self.N
        k = 0 if W_prefix is None else int(np.asarray(W_prefix).reshape(-1, N).shape[0])
        Wp = None if W_prefix is None else np.ascontiguousarray(np.asarray(W_prefix, dtype=np.float64).reshape(k, N))
        a = dict(W=np.zeros((N_out, N)), alpha=np.zeros(N_out), upsilon=np.zeros(N_out),
                 index=np.full(N_out, -1, dtype=np.int64), iters=np.zeros(N_out, np.int32),
                 n_iter=np.zeros(N_out, np.int32), cluster_size=np.zeros(N_out, np.int32),
                 n_converged=np.zeros(N_out, np.int32), n_unconverged=np.zeros(N_out, np.int32),
                 n_degenerate=np.zeros(N_out, np.int32), sum_active=np.zeros(N_out, np.int64),
                 gaussian_flag=np.zeros(N_out, np.uint8), near_tie=np.zeros(N_out, np.uint8),
                 dim=np.zeros(N_out, np.int32), objective=np.zeros(N_out))
        if Wp is not None:
            a["W"][:k] = Wp
        ct = dict(W=C.c_double, alpha=C.c_double, upsilon=C.c_double, index=C.c_int64, iters=C.c_int32,
                  n_iter=C.c_int32, cluster_size=C.c_int32, n_converged=C.c_int32, n_unconverged=C.c_int32,
                  n_degenerate=C.c_int32, sum_active=C.c_int64, gaussian_flag=C.c_uint8, near_tie=C.c_uint8,
                  dim=C.c_int32, objective=C.c_double)
        res = Result(**{f: _np_ptr(a[f], ct[f]) for f in ct}, n_extracted=0, stopped=0)
        self._c(lib().oica_extract_components(self.h, N_out, max_iter, tol, flags,
                                              _np_ptr(Wp, C.c_double), k, C.byref(res)))
        n = res.n_extracted
        return Extraction(W=a["W"][:n].copy(), **{f: a[f] for f in ct if f != "W"}, n_extracted=n,
                          stopped=bool(res.stopped))

    # -- test / bench entry points
    def fixed_point_step(self, W, G_out, s4_out, fine: Optional[np.ndarray] = None):
        """One contraction; `fine` (host uint8 per row, fine rows last): per-row precision."""
        L = W.shape[0]
        _ready(W)
        if fine is None:
            self._c(lib().oica_fixed_point_step(self.h, _dptr(W), L, _dptr(G_out), _dptr(s4_out)))
        else:
            f = np.ascontiguousarray(fine, dtype=np.uint8)
            self._c(lib().oica_fixed_point_step_mixed(self.h, _dptr(W), L, _np_ptr(f, C.c_uint8), _dptr(G_out),
                                                      _dptr(s4_out)))

    def draw_candidates(self, i: int, W_acc: Optional[np.ndarray], W_out):
        k = 0 if W_acc is None else W_acc.shape[0]
        Wa = None if W_acc is None else np.ascontiguousarray(W_acc, dtype=np.float64)
        self._c(lib().oica_draw_candidates(self.h, i, _np_ptr(Wa, C.c_double), k, _dptr(W_out)))

    def candidates(self):
        Ll, base = C.c_int64(), C.c_int64()
        self._c(lib().oica_get_candidates(self.h, None, None, None, None, C.byref(Ll), C.byref(base)))
        n = Ll.value
        W = np.zeros((n, self.N))
        alpha = np.zeros(n)
        iters = np.zeros(n, np.int32)
        state = np.zeros(n, np.uint8)
        self._c(lib().oica_get_candidates(self.h, _np_ptr(W, C.c_double), _np_ptr(alpha, C.c_double),
                                          _np_ptr(iters, C.c_int32), _np_ptr(state, C.c_uint8), None, None))
        return dict(W=W, alpha=alpha, iters=iters, state=state, id_base=base.value)

    def iteration_log(self) -> list:
        """Per-iteration records of the last extract call (component, iteration, L_act, fine_rows,
        step_ms, flops)."""
        n = C.c_int64()
        self._c(lib().oica_get_iteration_log(self.h, None, 0, C.byref(n)))
        buf = (IterationRecord * max(1, n.value))()
        self._c(lib().oica_get_iteration_log(self.h, buf, n.value, C.byref(n)))
        return [{f: getattr(buf[k], f) for f, _ in IterationRecord._fields_} for k in range(n.value)]

    def stats(self) -> dict:
        s = Stats()
        self._c(lib().oica_get_stats(self.h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in Stats._fields_}

    def reset_stats(self):
        self._c(lib().oica_reset_stats(self.h))

    def synchronize(self):
        self._c(lib().oica_synchronize(self.h))
