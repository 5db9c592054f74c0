"""Tensor plumbing between the Python API and the C ABI.

PyTorch is used for device memory and streams only; all arithmetic of the
path runs in libloki_b200.so.  Inputs may be numpy arrays / CPU tensors (the
reference's calling convention -- copied to the current CUDA device, results
copied back) or CUDA tensors (kept on device, results returned on device).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ShapeError, UnsupportedShapeError

_F32 = torch.float32


def current_device() -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.LibraryMissing("no CUDA device: libloki_b200 has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_of(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class _NoGuard:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


_NO_GUARD = _NoGuard()


def on_device(device):
    """The library launches on the CURRENT device: make it the tensors' device for the call
    (a no-op context when it already is, so the steady-state path pays nothing)."""
    if device.index is None or torch.cuda.current_device() == device.index:
        return _NO_GUARD
    return torch.cuda.device(device)


def as_device(x, dtype=_F32, device=None, keep_dtype=False, rows_only=False):
    """-> (contiguous CUDA tensor, came_from_host).  rows_only: a CUDA tensor whose last dim is
    contiguous is kept as the (possibly strided) view it is -- cache views are never copied."""
    if isinstance(x, torch.Tensor) and x.is_cuda:
        t = x
        if not keep_dtype and t.dtype != dtype:
            t = t.to(dtype)
        if rows_only and t.dim() >= 1 and t.stride(-1) == 1:
            return t, False
        return t.contiguous(), False
    dev = device or current_device()
    if isinstance(x, torch.Tensor):
        t = x
        if not keep_dtype and t.dtype != dtype:
            t = t.to(dtype)
        return t.contiguous().to(dev, non_blocking=False), True
    a = np.asarray(x)
    if not keep_dtype or a.dtype.kind != "f":
        a = a.astype(torch_to_np(dtype), copy=False)
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev), True


def torch_to_np(dt):
    return {torch.float32: np.float32, torch.float64: np.float64, torch.int64: np.int64,
            torch.int32: np.int32}[dt]


def back(t, host: bool):
    if host:
        return t.detach().cpu().numpy()
    return t


def cache_dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return _lib.DTYPE_F32
    if t.dtype == torch.bfloat16:
        return _lib.DTYPE_BF16
    raise UnsupportedShapeError(f"cache dtype {t.dtype} (float32 or bfloat16 only)")


def row_capacity(K: torch.Tensor) -> int:
    """Rows per (b, KV head) of the buffer behind a [B, Hkv, S, D] cache view.

    A prefix view [:, :, :S] of a [B, Hkv, cap, D] buffer (KvCache.storage sliced to its
    length) is addressed as the buffer itself -- S_cap = cap -- so the kernels see one
    packed row space and nothing is copied; otherwise S_cap = S."""
    B, Hkv, S, D = K.shape
    ss = K.stride(2)
    if ss < D:
        return S
    outer = K.stride(1) if Hkv > 1 else (K.stride(0) if B > 1 else 0)
    if outer <= S * ss or outer % ss:
        return S
    cap = outer // ss
    if Hkv > 1 and B > 1 and K.stride(0) != Hkv * K.stride(1):
        return S
    need = K.storage_offset() + (B * Hkv * cap - 1) * ss + D  # elements the packed view touches
    if need * K.element_size() > K.untyped_storage().nbytes():
        return S
    return cap


def geom_of(K: torch.Tensor, Hq: int) -> _lib.KvGeom:
    """Geometry of a [B, Hkv, S, D] cache view (D contiguous), S_cap = row_capacity(K)."""
    if K.dim() != 4 or K.stride(3) != 1:
        raise ShapeError(f"cache must be a [B, Hkv, S, D] view with contiguous rows, got {tuple(K.shape)}")
    B, Hkv, _, D = K.shape
    cap = row_capacity(K)
    sh = K.stride(1) if Hkv > 1 else cap * K.stride(2)
    sb = K.stride(0) if B > 1 else Hkv * sh
    return _lib.KvGeom(B, Hq, Hkv, D, cap, cache_dtype_code(K), sb, sh, K.stride(2))


@dataclass
class DecodeOutputs:
    out: torch.Tensor | None
    idx: torch.Tensor | None
    approx: torch.Tensor | None
    weights: torch.Tensor | None


class DecodeCall:
    """A prepared loki_decode invocation: the argument block is built once,
    so `run()` is a single C call (CUDA-graph capturable, no allocation)."""

    def __init__(self, q_hat, K, V, lens, S_max, d, *, k_f=0.0, k_fixed=0, select_mode=_lib.SELECT_TOPK,
                 ext_scores=None, ext_idx=None, idx_stride=0, out=None, idx_out=None, approx_out=None,
                 weights_out=None, Hq=None, cluster=0):
        ref = K if K is not None else ext_scores
        self.device = ref.device
        self.lib = _lib.lib_for(self.device)
        if K is not None:
            g = geom_of(K, Hq if Hq is not None else q_hat.shape[1])
        else:  # ranking externally supplied scores: [B, Hq, S_cap]
            B, Hq_, S_cap = ext_scores.shape
            g = _lib.KvGeom(B, Hq_, Hq_ if Hq is None else Hq, 1, S_cap, _lib.DTYPE_F32, 0, 0, 1)
        self.keep = [q_hat, K, V, lens, ext_scores, ext_idx, out, idx_out, approx_out, weights_out]
        a = _lib.DecodeArgs()
        a.q_hat = _lib.ptr(q_hat)
        a.K = _lib.ptr(K)
        a.V = _lib.ptr(V)
        a.g = g
        a.lens = _lib.ptr(lens)
        a.S_max = int(S_max)
        a.d = int(d)
        a.k_f = float(k_f)
        a.k_fixed = int(k_fixed)
        a.select_mode = int(select_mode)
        a.ext_scores = _lib.ptr(ext_scores)
        a.ext_idx = _lib.ptr(ext_idx)
        a.idx_stride = int(idx_stride)
        a.out = _lib.ptr(out)
        a.idx_out = _lib.ptr(idx_out)
        a.approx_out = _lib.ptr(approx_out)
        a.weights_out = _lib.ptr(weights_out)
        a.cluster_override = int(cluster)
        nbytes = ctypes.c_size_t(0)
        _lib.check(self.lib.loki_decode_workspace_bytes(ctypes.byref(a), ctypes.byref(nbytes)))
        self.workspace = None
        if nbytes.value:
            self.workspace = torch.zeros(nbytes.value, dtype=torch.uint8, device=self.device)
            a.workspace = self.workspace.data_ptr()
            a.workspace_bytes = nbytes.value
        self.args = a
        self._argp = ctypes.byref(a)
        self.outputs = DecodeOutputs(out, idx_out, approx_out, weights_out)

    def plan(self):
        c, r, s = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_size_t()
        _lib.check(self.lib.loki_decode_plan(self._argp, ctypes.byref(c), ctypes.byref(r), ctypes.byref(s)))
        return {"ctas_per_unit": c.value, "rows_per_cta": r.value, "smem_bytes": s.value}

    def run(self, stream=None):
        with on_device(self.device):
            _lib.check(self.lib.loki_decode(self._argp, stream if stream is not None else stream_of(self.device)))
        return self.outputs

    def run_phase(self, launches: int, stream=None):
        """Phase timing only (loki_decode_phase): 1 = the A launch (approx scores + top-k), 2 = the B launch
        (exact attention over the selection A left in the workspace), 3 = both."""
        with on_device(self.device):
            _lib.check(self.lib.loki_decode_phase(self._argp, int(launches),
                                                  stream if stream is not None else stream_of(self.device)))
        return self.outputs


def lens_tensor(lens, B, device):
    if isinstance(lens, torch.Tensor):
        t = lens.to(device=device, dtype=torch.int32)
        host = lens.detach().cpu().tolist() if lens.device.type == "cpu" else None
    else:
        vals = [int(x) for x in (lens if np.ndim(lens) else [lens] * B)]
        t = torch.tensor(vals, dtype=torch.int32, device=device)
        host = vals
    return t.contiguous(), host


def inv_freq_host(head_dim: int, base: float) -> np.ndarray:
    """base ** (-(2 i) / D) in fp64, identical to rope.py:34 / :66."""
    return base ** (-np.arange(head_dim // 2, dtype=np.float64) * 2.0 / head_dim)


_INV_FREQ_CACHE = {}


def inv_freq_device(head_dim: int, base: float, device) -> torch.Tensor:
    key = (head_dim, float(base), str(device))
    t = _INV_FREQ_CACHE.get(key)
    if t is None:
        t = torch.from_numpy(inv_freq_host(head_dim, base)).to(device)
        _INV_FREQ_CACHE[key] = t
    return t


def isqrt_scale(D: int) -> float:
    return 1.0 / math.sqrt(D)
