"""B200-native exhaustive FCNN-surrogate sweep (arxiv 2306.14011 hot path).

Thin ctypes binding over ``libsurrogate.so`` (C ABI in ``include/surrogate.h``):
argument marshalling only — every step of the path (decode, normalisation,
MLP layers, top-k, merges) runs in the CUDA kernels of ``csrc/``.  PyTorch is
used for device memory and streams.  There is no CPU fallback: if the shared
library is missing or the device is not sm_100 the calls raise.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .build import LIB_PATH, build_library  # noqa: F401

PREC = {"bf16": 0, "fp32": 1, "tf32": 2, "fp16": 3, "fp32_3xtf32": 4}
K_MAX = 1024
EXPORTS = [
    "surrogate_create", "surrogate_destroy", "surrogate_last_error", "surrogate_load_weights",
    "surrogate_predict", "surrogate_sweep", "surrogate_sweep_host", "surrogate_eval_range",
    "surrogate_merge_topk", "surrogate_sweep_records", "surrogate_decode_range", "surrogate_space_size",
    "surrogate_sweep_operands",
    "surrogate_kernel_timing", "surrogate_kernel_timing_get", "surrogate_last_launches",
    "surrogate_selftest_umma", "surrogate_table_bytes", "surrogate_debug_trace", "surrogate_reset_cache",
    "surrogate_arith", "surrogate_train",
]


class SurrogateError(RuntimeError):
    pass


class _Space(ctypes.Structure):
    _fields_ = [("num_params", ctypes.c_uint32), ("radix", ctypes.POINTER(ctypes.c_uint32)),
                ("values", ctypes.POINTER(ctypes.c_double)), ("begin", ctypes.c_uint64),
                ("end", ctypes.c_uint64)]


class _Model(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_uint32), ("widths", ctypes.POINTER(ctypes.c_uint32)),
                ("W", ctypes.POINTER(ctypes.POINTER(ctypes.c_double))),
                ("b", ctypes.POINTER(ctypes.POINTER(ctypes.c_double))),
                ("x_shift", ctypes.POINTER(ctypes.c_double)), ("x_scale", ctypes.POINTER(ctypes.c_double)),
                ("y_mean", ctypes.c_double), ("y_scale", ctypes.c_double),
                ("num_const_features", ctypes.c_uint32), ("const_features", ctypes.POINTER(ctypes.c_double)),
                ("ensemble", ctypes.c_uint32), ("precision", ctypes.c_int)]


_LIB = None


def lib() -> ctypes.CDLL:
    """Load the in-tree CUDA library; raise loudly when it is absent."""
    global _LIB
    if _LIB is None:
        path = os.environ.get("SURR_LIB", LIB_PATH)  # development A/B of two in-tree builds
        if not os.path.exists(path):
            raise SurrogateError(f"{path} not built (run __graft_entry__.build()); no CPU fallback exists")
        L = ctypes.CDLL(path)
        vp, u32, u64, i32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
        L.surrogate_create.argtypes = [i32, ctypes.POINTER(vp)]
        L.surrogate_destroy.argtypes = [vp]
        L.surrogate_destroy.restype = None
        L.surrogate_last_error.argtypes = [vp]
        L.surrogate_last_error.restype = ctypes.c_char_p
        L.surrogate_load_weights.argtypes = [vp, ctypes.POINTER(_Model)]
        L.surrogate_predict.argtypes = [vp, vp, u64, vp, vp]
        L.surrogate_sweep.argtypes = [vp, ctypes.POINTER(_Space), u32, vp, vp, ctypes.POINTER(u32), vp]
        L.surrogate_sweep_host.argtypes = [vp, ctypes.POINTER(_Space), u32, vp, vp, ctypes.POINTER(u32), vp]
        L.surrogate_eval_range.argtypes = [vp, ctypes.POINTER(_Space), vp, vp]
        if hasattr(L, "surrogate_sweep_operands"):  # (absent from round-1 builds used for A/B)
            L.surrogate_sweep_operands.argtypes = [vp, ctypes.POINTER(_Space), u64, vp, vp]
        L.surrogate_merge_topk.argtypes = [vp, vp, u32, u32, u32, vp, vp, vp, vp]
        L.surrogate_sweep_records.argtypes = [vp, ctypes.POINTER(_Space), u32, vp, vp]
        L.surrogate_decode_range.argtypes = [vp, ctypes.POINTER(_Space), u64, u64, vp, vp]
        L.surrogate_space_size.argtypes = [ctypes.POINTER(_Space), ctypes.POINTER(u64)]
        L.surrogate_kernel_timing.argtypes = [vp, i32]
        L.surrogate_kernel_timing_get.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(u32)]
        L.surrogate_last_launches.argtypes = [vp]
        L.surrogate_last_launches.restype = u32
        L.surrogate_selftest_umma.argtypes = [i32, i32, u32, u32, vp, vp, vp]
        L.surrogate_debug_trace.argtypes = [vp, vp, u32]
        L.surrogate_reset_cache.argtypes = [vp]
        L.surrogate_arith.argtypes = [vp, ctypes.POINTER(u32), ctypes.POINTER(u32), ctypes.POINTER(ctypes.c_double)]
        L.surrogate_train.argtypes = [vp, vp, u32, vp, vp, vp, vp, u64, vp, ctypes.POINTER(_TrainHyper), vp, vp, vp]
        L.surrogate_table_bytes.argtypes = [vp]
        L.surrogate_table_bytes.restype = u32
        for name in EXPORTS:
            if not hasattr(L, name):
                continue
            fn = getattr(L, name)
            if fn.restype is ctypes.c_int and name not in ("surrogate_last_launches",):
                fn.restype = ctypes.c_int
        _LIB = L
    return _LIB


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _check(rc: int, handle=None):
    if rc != 0:
        msg = lib().surrogate_last_error(handle).decode(errors="replace")
        raise SurrogateError(f"status {rc}: {msg}")


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class SpaceDesc:
    """Host-side search-space descriptor (value lists in Table order)."""

    def __init__(self, value_lists, begin: int = 0, end: int = 0):
        self.radix = np.ascontiguousarray([len(v) for v in value_lists], dtype=np.uint32)
        self.values = np.ascontiguousarray(np.concatenate([np.asarray(v, np.float64) for v in value_lists]))
        self.c = _Space(len(value_lists), _ptr(self.radix, ctypes.c_uint32), _ptr(self.values, ctypes.c_double),
                        int(begin), int(end))


def space_size(value_lists) -> int:
    d = SpaceDesc(value_lists)
    out = ctypes.c_uint64()
    _check(lib().surrogate_space_size(ctypes.byref(d.c), ctypes.byref(out)))
    return out.value


class Surrogate:
    """One handle on one CUDA device (surrogate_create / surrogate_destroy)."""

    def __init__(self, device: int = 0):
        self.device = int(device)
        h = ctypes.c_void_p()
        _check(lib().surrogate_create(self.device, ctypes.byref(h)))
        self.h = h
        self.precision = None
        self.P = None

    def close(self):
        if self.h:
            lib().surrogate_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- model
    def load(self, model: dict, precision: str = "bf16"):
        """surrogate_load_weights from the model record of workloads.load_model."""
        widths = np.ascontiguousarray(model["widths"], dtype=np.uint32)
        members = model["members"]
        L = len(widths) - 1
        keep = []
        Wp = (ctypes.POINTER(ctypes.c_double) * (L * len(members)))()
        bp = (ctypes.POINTER(ctypes.c_double) * (L * len(members)))()
        for e, m in enumerate(members):
            for l in range(L):
                w = np.ascontiguousarray(m["W"][l], dtype=np.float64)
                b = np.ascontiguousarray(m["b"][l], dtype=np.float64)
                keep += [w, b]
                Wp[e * L + l] = _ptr(w, ctypes.c_double)
                bp[e * L + l] = _ptr(b, ctypes.c_double)
        xs = np.ascontiguousarray(model["x_shift"], dtype=np.float64)
        xc = np.ascontiguousarray(model["x_scale"], dtype=np.float64)
        cf = np.ascontiguousarray(model.get("const_features", np.zeros(0)), dtype=np.float64)
        cfp = _ptr(cf, ctypes.c_double) if cf.size else ctypes.POINTER(ctypes.c_double)()
        mc = _Model(L, _ptr(widths, ctypes.c_uint32), Wp, bp, _ptr(xs, ctypes.c_double),
                    _ptr(xc, ctypes.c_double), float(model["y_mean"]), float(model["y_scale"]),
                    int(cf.size), cfp, len(members), PREC[precision])
        _check(lib().surrogate_load_weights(self.h, ctypes.byref(mc)), self.h)
        self.precision = precision
        # identity of the loaded model (weights, scalers, device features,
        # precision, ensemble size): part of every campaign checkpoint fingerprint
        import hashlib
        dg = hashlib.sha256(f"{precision}|{len(members)}|{list(map(int, widths))}|".encode())
        for a in keep + [xs, xc, cf, np.array([model["y_mean"], model["y_scale"]], np.float64)]:
            dg.update(np.ascontiguousarray(a).tobytes())
        self.model_digest = dg.hexdigest()
        self.P = int(widths[0]) - int(cf.size)
        return self

    # ---------------------------------------------------------------- calls
    def sweep(self, value_lists, k: int, begin: int = 0, end: int = 0, stream=None):
        """Top-k (idx int64 tensor, t float32 tensor, count) on the device."""
        import torch
        d = SpaceDesc(value_lists, begin, end)
        idx = torch.empty(k, dtype=torch.int64, device=f"cuda:{self.device}")
        t = torch.empty(k, dtype=torch.float32, device=f"cuda:{self.device}")
        cnt = ctypes.c_uint32()
        _check(lib().surrogate_sweep(self.h, ctypes.byref(d.c), k, ctypes.c_void_p(idx.data_ptr()),
                                     ctypes.c_void_p(t.data_ptr()), ctypes.byref(cnt), _stream_ptr(stream)), self.h)
        return idx, t, cnt.value

    def sweep_into(self, desc: SpaceDesc, k: int, idx, t, stream=None) -> int:
        """Allocation-free sweep into caller tensors (bench inner loop)."""
        cnt = ctypes.c_uint32()
        _check(lib().surrogate_sweep(self.h, ctypes.byref(desc.c), k, ctypes.c_void_p(idx.data_ptr()),
                                     ctypes.c_void_p(t.data_ptr()), ctypes.byref(cnt), _stream_ptr(stream)), self.h)
        return cnt.value

    def sweep_host(self, value_lists, k: int, begin: int = 0, end: int = 0, stream=None, desc=None,
                   out=None):
        """End-to-end call with host outputs (numpy uint64 idx, float32 t, count)."""
        d = desc if desc is not None else SpaceDesc(value_lists, begin, end)
        if out is None:
            out = (np.empty(k, np.uint64), np.empty(k, np.float32))
        idx, t = out
        cnt = ctypes.c_uint32()
        _check(lib().surrogate_sweep_host(self.h, ctypes.byref(d.c), k, idx.ctypes.data_as(ctypes.c_void_p),
                                          t.ctypes.data_as(ctypes.c_void_p), ctypes.byref(cnt),
                                          _stream_ptr(stream)), self.h)
        return idx, t, cnt.value

    def sweep_records(self, value_lists, k: int, begin: int = 0, end: int = 0, stream=None):
        """Top-k as surr_record rows (int64 tensor [k, 2]: idx, key | pad << 32)."""
        import torch
        d = SpaceDesc(value_lists, begin, end)
        recs = torch.empty((k, 2), dtype=torch.int64, device=f"cuda:{self.device}")
        _check(lib().surrogate_sweep_records(self.h, ctypes.byref(d.c), k, ctypes.c_void_p(recs.data_ptr()),
                                             _stream_ptr(stream)), self.h)
        return recs

    def merge_topk(self, recs, lists: int, k_in: int, k: int, stream=None):
        """Merge `lists` sorted record lists (tensor [lists*k_in, 2]) into (idx, t, recs)."""
        import torch
        dev = f"cuda:{self.device}"
        idx = torch.empty(k, dtype=torch.int64, device=dev)
        t = torch.empty(k, dtype=torch.float32, device=dev)
        out = torch.empty((k, 2), dtype=torch.int64, device=dev)
        _check(lib().surrogate_merge_topk(self.h, ctypes.c_void_p(recs.data_ptr()), lists, k_in, k,
                                          ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(t.data_ptr()),
                                          ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)), self.h)
        return idx, t, out

    def sweep_records_into(self, desc: SpaceDesc, k: int, recs, stream=None) -> int:
        _check(lib().surrogate_sweep_records(self.h, ctypes.byref(desc.c), k, ctypes.c_void_p(recs.data_ptr()),
                                             _stream_ptr(stream)), self.h)
        return self.last_launches()

    def merge_topk_into(self, recs, lists: int, k_in: int, k: int, idx, t, stream=None):
        _check(lib().surrogate_merge_topk(self.h, ctypes.c_void_p(recs.data_ptr()), lists, k_in, k,
                                          ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(t.data_ptr()),
                                          None, _stream_ptr(stream)), self.h)

    def reset_cache(self):
        """Drop the cached value table (next sweep rebuilds + uploads it)."""
        _check(lib().surrogate_reset_cache(self.h), self.h)

    def arith(self):
        """(mma kind, passes, issued tensor FLOPs per config and member) of the
        loaded model's kernel: ("f16" | "tf32", 1 | 3, float)."""
        kind, passes, fl = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_double()
        _check(lib().surrogate_arith(self.h, ctypes.byref(kind), ctypes.byref(passes), ctypes.byref(fl)), self.h)
        return ("f16" if kind.value == 0 else "tf32"), int(passes.value), float(fl.value)

    def lut_bytes(self) -> int:
        """Bytes of the value table uploaded by the last sweep (the per-step H2D)."""
        return int(lib().surrogate_table_bytes(self.h))

    def eval_range(self, value_lists, begin: int, end: int, stream=None):
        """t(I) for every I in [begin, end) from the fused kernel (dense mode)."""
        import torch
        d = SpaceDesc(value_lists, begin, end)
        t = torch.empty(end - begin, dtype=torch.float32, device=f"cuda:{self.device}")
        _check(lib().surrogate_eval_range(self.h, ctypes.byref(d.c), ctypes.c_void_p(t.data_ptr()),
                                          _stream_ptr(stream)), self.h)
        return t

    def sweep_operands(self, value_lists, begin: int, end: int, stride: int = 1, stream=None):
        """Layer-1 operand rows the fused sweep kernel built for I = begin + q stride
        in [begin, end): int32 [n, 16] device tensor (8 hi column pairs, 8 lo pairs;
        parity hook of the decoder and the value table)."""
        import torch
        d = SpaceDesc(value_lists, begin, end)
        n = (end - begin + stride - 1) // stride
        out = torch.empty((n, 16), dtype=torch.int32, device=f"cuda:{self.device}")
        _check(lib().surrogate_sweep_operands(self.h, ctypes.byref(d.c), stride, ctypes.c_void_p(out.data_ptr()),
                                              _stream_ptr(stream)), self.h)
        return out

    def predict(self, x, stream=None):
        """Explicit batch: x float32 [n, P] device tensor of raw values -> t [n]."""
        import torch
        x = x.contiguous()
        if x.dtype != torch.float32 or x.dim() != 2 or x.shape[1] != self.P:
            raise ValueError(f"x must be float32 [n, {self.P}]")
        t = torch.empty(x.shape[0], dtype=torch.float32, device=x.device)
        _check(lib().surrogate_predict(self.h, ctypes.c_void_p(x.data_ptr()), x.shape[0],
                                       ctypes.c_void_p(t.data_ptr()), _stream_ptr(stream)), self.h)
        return t

    def decode_range(self, value_lists, first: int, n: int, stream=None):
        import torch
        d = SpaceDesc(value_lists)
        out = torch.empty((n, len(value_lists)), dtype=torch.uint8, device=f"cuda:{self.device}")
        _check(lib().surrogate_decode_range(self.h, ctypes.byref(d.c), first, n, ctypes.c_void_p(out.data_ptr()),
                                            _stream_ptr(stream)), self.h)
        return out

    def debug_trace(self, buf):
        """Record CTA 0's pipeline timeline into a device int64 tensor (None: off)."""
        _check(lib().surrogate_debug_trace(self.h, ctypes.c_void_p(buf.data_ptr()) if buf is not None else None,
                                           0 if buf is None else buf.numel()), self.h)

    def kernel_timing(self, enable: bool):
        _check(lib().surrogate_kernel_timing(self.h, 1 if enable else 0), self.h)

    def kernel_timing_get(self):
        ms = ctypes.c_double()
        n = ctypes.c_uint32()
        _check(lib().surrogate_kernel_timing_get(self.h, ctypes.byref(ms), ctypes.byref(n)), self.h)
        return ms.value, n.value

    def last_launches(self) -> int:
        return int(lib().surrogate_last_launches(self.h))


def selftest_umma(precision: str, A: np.ndarray, B: np.ndarray, device: int = 0) -> np.ndarray:
    """D = A[128 x K] @ B[K x N] through one tcgen05 UMMA chain (test hook)."""
    A = np.ascontiguousarray(A, np.float32)
    B = np.ascontiguousarray(B, np.float32)
    assert A.shape[0] == 128 and A.shape[1] == B.shape[0]
    D = np.empty((128, B.shape[1]), np.float32)
    rc = lib().surrogate_selftest_umma(device, PREC[precision], B.shape[1], A.shape[1],
                                       A.ctypes.data_as(ctypes.c_void_p), B.ctypes.data_as(ctypes.c_void_p),
                                       D.ctypes.data_as(ctypes.c_void_p))
    _check(rc)
    return D


class _TrainHyper(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("lr0", ctypes.c_double), ("eps", ctypes.c_double), ("tol", ctypes.c_double),
                ("batch_size", ctypes.c_uint32), ("max_epochs", ctypes.c_uint32),
                ("n_iter_no_change", ctypes.c_uint32)]


# the paper's Table "Hyperparameter" + scikit-learn's n_iter_no_change
TRAIN_HYPER = dict(alpha=1e-4, beta1=0.95, beta2=0.90, lr0=0.0009, eps=1e-9, tol=1e-6, batch_size=200,
                   max_epochs=200, n_iter_no_change=10)


def train_ensemble(members, X, y, perms=None, hyper=None, device: int = 0):
    """GPU training of E F-H-H-1 nets at once (surrogate_train, one cluster per
    member): members = [(W, b), ...] with W, b lists of 3 float64 arrays
    (fan_in x fan_out, initial values); X [n, F] / y [n] standardised; perms
    [E, max_epochs, n] uint32 epoch orders or None.  Returns, per member,
    (W, b, loss_history, stop_reason in {"max_epochs", "tol_converged"})."""
    h = dict(TRAIN_HYPER)
    if hyper:
        h.update(hyper)
    E = len(members)
    Ws = [[np.ascontiguousarray(w, np.float64).copy() for w in m[0]] for m in members]
    bs = [[np.ascontiguousarray(v, np.float64).reshape(-1).copy() for v in m[1]] for m in members]
    if E == 0 or any(len(w) != 3 or len(v) != 3 for w, v in zip(Ws, bs)):
        raise ValueError("one or more F-H-H-1 nets")
    X = np.ascontiguousarray(X, np.float64)
    y = np.ascontiguousarray(y, np.float64).reshape(-1)
    n = X.shape[0]
    W0 = Ws[0]
    widths = np.ascontiguousarray([W0[0].shape[0], W0[0].shape[1], W0[1].shape[1], W0[2].shape[1]], np.uint32)
    if perms is not None:
        perms = np.ascontiguousarray(perms, np.uint32)
        if perms.shape != (E, h["max_epochs"], n):
            raise ValueError(f"perms must be [{E}, {h['max_epochs']}, {n}]")
    hp = _TrainHyper(h["alpha"], h["beta1"], h["beta2"], h["lr0"], h["eps"], h["tol"], int(h["batch_size"]),
                     int(h["max_epochs"]), int(h["n_iter_no_change"]))
    Wp = (ctypes.c_void_p * (3 * E))(*[w.ctypes.data for m in Ws for w in m])
    bp = (ctypes.c_void_p * (3 * E))(*[v.ctypes.data for m in bs for v in m])
    hist = np.zeros((E, h["max_epochs"]), np.float64)
    ep = np.zeros(E, np.uint32)
    reason = np.zeros(E, np.uint32)
    s = Surrogate(device)
    _check(lib().surrogate_train(s.h, widths.ctypes.data, E, ctypes.cast(Wp, ctypes.c_void_p),
                                 ctypes.cast(bp, ctypes.c_void_p), X.ctypes.data, y.ctypes.data, n,
                                 None if perms is None else perms.ctypes.data, ctypes.byref(hp),
                                 hist.ctypes.data, ep.ctypes.data, reason.ctypes.data), s.h)
    return [(Ws[e], bs[e], hist[e, :ep[e]].tolist(), "tol_converged" if reason[e] == 1 else "max_epochs")
            for e in range(E)]


def train(W, b, X, y, perms=None, hyper=None, device: int = 0):
    """One member: train_ensemble([(W, b)], ...) with perms [max_epochs, n]."""
    return train_ensemble([(W, b)], X, y, None if perms is None else np.asarray(perms)[None], hyper, device)[0]


def key_to_float(keys: np.ndarray) -> np.ndarray:
    """Inverse of the kernels' order-preserving float -> uint32 key (for records)."""
    k = np.asarray(keys, np.uint32)
    u = np.where(k & 0x80000000, k & 0x7FFFFFFF, ~k).astype(np.uint32)
    return u.view(np.float32)
