"""L1 primitives on the GPU -- mirrors lokiattn/linalg.py:76-138.

softmax_row and topk_indices run in libloki_b200 (sm_100a); the index
canonicalisation is host-side validation logic, as in the reference.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _core, _lib
from .errors import BudgetError, ShapeError


def _as_vector(scores):
    """1-D view, accepting 1xN / Nx1 (linalg.py:27-34)."""
    t, host = _core.as_device(scores, torch.float32)
    if t.dim() == 2 and 1 in t.shape:
        t = t.reshape(-1)
    if t.dim() != 1:
        raise ShapeError(f"scores must be 1-D, got shape={tuple(t.shape)}")
    return t, host


def softmax_row(scores):
    """Numerically stable softmax of one score vector (linalg.py:76-92).

    Max-subtraction, exp and the normaliser run in fp64 on the device; the
    result is fp32 (fp64 input gets an fp64-typed copy of that result).
    """
    is_f64 = (isinstance(scores, np.ndarray) and scores.dtype == np.float64) or \
        (isinstance(scores, torch.Tensor) and scores.dtype == torch.float64)
    t, host = _core.as_device(scores, torch.float32)
    if t.dim() == 2 and 1 in t.shape:
        t = t.reshape(-1)
    if t.dim() != 1 or t.numel() == 0:
        raise ShapeError(f"softmax_row expects a nonempty vector, got shape={tuple(t.shape)}")
    out = softmax_rows(t.reshape(1, -1)).reshape(-1)
    if is_f64:
        out = out.double()
    return _core.back(out, host)


def softmax_rows(x: torch.Tensor) -> torch.Tensor:
    """Row-wise softmax_row over a [R, n] CUDA tensor (batched extension)."""
    x = x.contiguous()
    if x.dim() != 2 or x.shape[1] == 0:
        raise ShapeError(f"softmax_rows expects a nonempty [R, n] matrix, got {tuple(x.shape)}")
    out = torch.empty_like(x, dtype=torch.float32)
    lib = _lib.lib_for(x.device)
    _lib.check(lib.loki_softmax_rows(x.data_ptr(), x.shape[0], x.shape[1], x.shape[1], out.data_ptr(),
                                     _core.stream_of(x.device)))
    return out


def topk_indices(scores, k):
    """Indices of the k largest scores, ascending; ties at the threshold go to
    the lower index (linalg.py:95-118).  k == n returns arange(n)."""
    s, host = _as_vector(scores)
    n = s.numel()
    if not 1 <= k <= n:
        raise BudgetError(f"k={k} outside [1, {n}]")
    idx = topk_rows(s.reshape(1, 1, n), k)
    out = idx.reshape(-1).to(torch.int64)
    return _core.back(out, host)


def topk_rows(scores: torch.Tensor, k, lens=None) -> torch.Tensor:
    """Batched topk_indices over [B, H, S] CUDA scores -> int32 [B, H, k_max].

    Each row uses its batch's length (lens[b], default S) and k (an int, or a
    per-batch sequence); entries past a row's k are left as -1.
    """
    scores = scores.contiguous()
    B, H, S = scores.shape
    lens_t, lens_h = _core.lens_tensor(S if lens is None else lens, B, scores.device)
    if np.ndim(k) == 0:
        k_fixed, kmax = int(k), int(k)
    else:
        raise ShapeError("per-row k is expressed through lens with a shared k_fixed")
    S_max = max(lens_h) if lens_h is not None else S
    idx = torch.full((B, H, kmax), -1, dtype=torch.int32, device=scores.device)
    call = _core.DecodeCall(None, None, None, lens_t, S_max, 1, k_fixed=k_fixed, select_mode=_lib.SELECT_TOPK,
                            ext_scores=scores, idx_stride=kmax, idx_out=idx)
    call.run()
    return idx


def canonicalize_indices(indices, n):
    """Validate against row count n, return ascending (linalg.py:121-138).

    Duplicates -> ShapeError, out of range -> IndexError.
    """
    t, host = _core.as_device(indices, torch.int64)
    t = t.reshape(-1)
    if t.numel() == 0:
        return _core.back(t, host)
    ascending = bool((t[1:] > t[:-1]).all()) if t.numel() > 1 else True
    if not ascending:
        t = torch.sort(t).values
        if bool((t[1:] == t[:-1]).any()):
            raise ShapeError("duplicate indices")
    if int(t[0]) < 0 or int(t[-1]) >= n:
        raise IndexError(f"index outside [0, {n})")
    return _core.back(t, host)
