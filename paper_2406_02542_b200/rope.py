"""Rotary position embeddings on the GPU -- mirrors lokiattn/rope.py:14-75.

Half-split pairing (i, i + D/2) rotated by position * base**(-2i/D); the
rotation runs in fp64 on the device (explicitly rounded products, matching
numpy's evaluation order) and returns the input's float dtype.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _core, _lib
from .errors import DomainError, ShapeError

DEFAULT_BASE = 10000.0


@dataclass(frozen=True)
class RopeParams:
    head_dim: int
    base: float = DEFAULT_BASE

    def __post_init__(self):
        if self.head_dim <= 0 or self.head_dim % 2 != 0:
            raise ShapeError(f"head_dim must be a positive even number, got {self.head_dim}")
        if not self.base > 1.0:
            raise DomainError(f"base must exceed 1, got {self.base}")


def rope_angles(position: int, params: RopeParams) -> np.ndarray:
    """Per-pair angles at one position, fp64, length D/2 (rope.py:29-35). Host helper."""
    if position < 0:
        raise DomainError(f"position must be nonnegative, got {position}")
    return position * _core.inv_freq_host(params.head_dim, params.base)


def _rope_rows(m: torch.Tensor, positions: torch.Tensor, params: RopeParams) -> torch.Tensor:
    io = _lib.DTYPE_F64 if m.dtype == torch.float64 else _lib.DTYPE_F32
    out = torch.empty_like(m)
    lib = _lib.lib_for(m.device)
    inv = _core.inv_freq_device(params.head_dim, params.base, m.device)
    _lib.check(lib.loki_rope(m.data_ptr(), out.data_ptr(), io, m.shape[0], params.head_dim, positions.data_ptr(),
                             inv.data_ptr(), _core.stream_of(m.device)))
    return out


def _float_input(v):
    is64 = (isinstance(v, np.ndarray) and v.dtype == np.float64) or \
        (isinstance(v, torch.Tensor) and v.dtype == torch.float64)
    return _core.as_device(v, torch.float64 if is64 else torch.float32)


def rope_apply(v, position: int, params: RopeParams):
    """Rotate one head vector to `position` (rope.py:38-55)."""
    a, host = _float_input(v)
    if a.dim() != 1 or a.numel() != params.head_dim:
        raise ShapeError(f"vector length {tuple(a.shape)} does not match head_dim {params.head_dim}")
    if position < 0:
        raise DomainError(f"position must be nonnegative, got {position}")
    pos = torch.tensor([int(position)], dtype=torch.int64, device=a.device)
    return _core.back(_rope_rows(a.reshape(1, -1), pos, params).reshape(-1), host)


def rope_apply_rows(mat, params: RopeParams, start_position: int = 0):
    """Rotate every row, row i at start_position + i (rope.py:58-75)."""
    m, host = _float_input(mat)
    if m.dim() != 2 or m.shape[1] != params.head_dim:
        raise ShapeError(f"matrix shape {tuple(m.shape)} does not match head_dim {params.head_dim}")
    if start_position < 0:
        raise DomainError("start_position must be nonnegative")
    pos = torch.arange(start_position, start_position + m.shape[0], dtype=torch.int64, device=m.device)
    return _core.back(_rope_rows(m, pos, params), host)
