"""Gather-aware kernels on the GPU -- mirrors lokiattn/kernels.py:76-308.

Same names, argument meaning and errors as the reference; the arithmetic is
the sm_100a code in libloki_b200.so.  TileSpec is accepted for API
compatibility: tiling on the GPU is chosen by the launch planner, and results
are deterministic for a fixed shape (fixed-order reductions).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _core, _lib
from .errors import BudgetError, ShapeError
from .linalg import canonicalize_indices


@dataclass(frozen=True)
class TileSpec:
    """Tile sizes of the reference's CPU kernels (kernels.py:76-88); validated, not used."""

    tile_m: int = 8
    tile_n: int = 256

    def __post_init__(self):
        if self.tile_m < 1 or self.tile_n < 1:
            raise ShapeError(f"tile sizes must be >= 1, got {self}")


DEFAULT_TILES = TileSpec()

_MAX_GROUP = 8  # query rows per fused launch (one KV head, up to 8 query heads)


def _query_block(q_hat):
    q, host = _core.as_device(q_hat, torch.float32)
    if q.dim() == 1:
        return q.reshape(1, -1), True, host
    if q.dim() == 2:
        return q, False, host
    raise ShapeError(f"query must be 1-D or 2-D, got ndim={q.dim()}")


def _matrix(K, device):
    t, _ = _core.as_device(K, torch.float32, device=device, keep_dtype=True)
    if t.dtype not in (torch.float32, torch.bfloat16):
        t = t.float()
    return t


def sliced_score_kernel(q_hat, K_hat, d, tiles: TileSpec = DEFAULT_TILES):
    """out[j] = sum_{t<d} q[t] K[j, t]  (kernels.py:223-241); an m x D query
    block yields m x S scores.  Reads only the leading d columns of K."""
    q, squeeze, host = _query_block(q_hat)
    K = _matrix(K_hat, q.device)
    if K.dim() != 2 or K.shape[1] != q.shape[1]:
        raise ShapeError(f"key shape {tuple(K.shape)} does not match query dim {q.shape[1]}")
    if not 1 <= d <= K.shape[1]:
        raise BudgetError(f"d={d} outside [1, {K.shape[1]}]")
    m, S = q.shape[0], K.shape[0]
    out = torch.empty((m, S), dtype=torch.float32, device=q.device)
    if S > 0:
        K4 = K.unsqueeze(0).unsqueeze(0)
        lens, _ = _core.lens_tensor(S, 1, q.device)
        for i0 in range(0, m, _MAX_GROUP):
            qb = q[i0:i0 + _MAX_GROUP].contiguous()
            mb = qb.shape[0]
            ob = out[i0:i0 + mb]
            call = _core.DecodeCall(qb.reshape(1, mb, -1), K4, None, lens, S, d, select_mode=_lib.SELECT_NONE,
                                    approx_out=ob, Hq=mb)
            call.run()
    res = out[0] if squeeze else out
    return _core.back(res, host)


def gathered_score_kernel(q_hat, K_hat, indices, tiles: TileSpec = DEFAULT_TILES):
    """out[j] = q . K[indices[j]] over the full width (kernels.py:244-261).
    Indices are canonicalised (ascending; duplicates ShapeError, range IndexError)."""
    q, squeeze, host = _query_block(q_hat)
    K = _matrix(K_hat, q.device)
    if K.dim() != 2 or K.shape[1] != q.shape[1]:
        raise ShapeError(f"key shape {tuple(K.shape)} does not match query dim {q.shape[1]}")
    idx = canonicalize_indices(_core.as_device(indices, torch.int64, device=q.device)[0], K.shape[0])
    m, n = q.shape[0], idx.numel()
    out = torch.empty((m, n), dtype=torch.float32, device=q.device)
    if n:
        lib = _lib.lib_for(q.device)
        _lib.check(lib.loki_gathered_scores(q.data_ptr(), m, K.data_ptr(), K.stride(0), _core.cache_dtype_code(K),
                                            K.shape[1], idx.data_ptr(), n, out.data_ptr(),
                                            _core.stream_of(q.device)))
    res = out[0] if squeeze else out
    return _core.back(res, host)


def _weighted_sum(w, V, idx, device):
    D = V.shape[1]
    n = w.numel()
    lib = _lib.lib_for(device)
    nbytes = lib.loki_weighted_sum_workspace(n, D)
    partial = torch.empty(nbytes // 4 + 1, dtype=torch.float32, device=device)
    out = torch.empty(D, dtype=torch.float32, device=device)
    _lib.check(lib.loki_weighted_sum(w.data_ptr(), V.data_ptr(), V.stride(0), _core.cache_dtype_code(V), D,
                                     _lib.ptr(idx), n, out.data_ptr(), partial.data_ptr(), nbytes,
                                     _core.stream_of(device)))
    return out


def gathered_weighted_sum_kernel(weights, V, indices, tiles: TileSpec = DEFAULT_TILES):
    """out = sum_j weights[j] V[indices[j]] without a gathered copy (kernels.py:264-279).
    As in the reference, indices are canonicalised and weights keep their order."""
    w, host = _core.as_device(weights, torch.float32)
    w = w.reshape(-1)
    Vm = _matrix(V, w.device)
    if Vm.dim() != 2:
        raise ShapeError("values must be 2-D")
    idx = canonicalize_indices(_core.as_device(indices, torch.int64, device=w.device)[0], Vm.shape[0])
    if w.numel() != idx.numel():
        raise ShapeError(f"{w.numel()} weights for {idx.numel()} indices")
    return _core.back(_weighted_sum(w, Vm, idx, w.device), host)


def dense_weighted_sum_kernel(weights, V, tiles: TileSpec = DEFAULT_TILES):
    """out = sum_j weights[j] V[j] over every row (kernels.py:282-294)."""
    w, host = _core.as_device(weights, torch.float32)
    w = w.reshape(-1)
    Vm = _matrix(V, w.device)
    if Vm.dim() != 2 or w.numel() != Vm.shape[0]:
        raise ShapeError(f"{w.numel()} weights for {tuple(Vm.shape)} values")
    return _core.back(_weighted_sum(w, Vm, None, w.device), host)


def gather_copy_scores_reference(q_hat, K_hat, indices):
    """Copy-then-dense comparator (kernels.py:297-308): materialises K[indices]
    with torch and multiplies.  A benchmark baseline, not the product path."""
    q, squeeze, host = _query_block(q_hat)
    K = _matrix(K_hat, q.device).float()
    idx = canonicalize_indices(_core.as_device(indices, torch.int64, device=q.device)[0], K.shape[0])
    dense = K.index_select(0, idx)
    out = q @ dense.T
    res = out[0] if squeeze else out
    return _core.back(res, host)
