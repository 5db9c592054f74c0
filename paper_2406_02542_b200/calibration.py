"""Offline PCA calibration -- mirrors lokiattn/calibration.py:32-148.

Covariance (fp64, centred, 1/(S-1), symmetrised), symmetric eigensolve,
descending stable order, canonical signs (largest-|entry| of each column
positive), clipped + normalised spectrum, P in fp32 with principal directions
as columns.  Runs on the keys' CUDA device in fp64 (torch GEMM + cuSOLVER
eigh): calibration is offline, once per (layer, KV head), not per step.
Numpy input returns numpy P / eigenvalues, CUDA input returns CUDA tensors.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np
import torch

from . import _core
from .errors import DegenerateCalibrationError, DomainError, InsufficientDataError, ShapeError

logger = logging.getLogger(__name__)

ROTARY_STAGES = ("pre", "post")


@dataclass(frozen=True)
class ProjectionSet:
    """Per-(layer, head) orthogonal projection P [D, D] (or a bank [Hkv, D, D])
    with its normalised spectrum (calibration.py:32-48)."""

    layer: int
    head: int
    P: object
    eigenvalues: object
    rotary_stage: str

    @property
    def head_dim(self) -> int:
        return int(self.P.shape[-1])


def compute_covariance(keys, center: bool = True):
    """Sample covariance (1/(S-1)) K'K in fp64 (calibration.py:51-67)."""
    k, host = _core.as_device(keys, torch.float64)
    if k.dim() != 2:
        raise ShapeError(f"keys must be 2-D, got ndim={k.dim()}")
    s = k.shape[0]
    if s < 2:
        raise InsufficientDataError(f"need at least 2 key rows, got {s}")
    if center:
        k = k - k.mean(dim=0)
    cov = (k.T @ k) / (s - 1)
    return _core.back((cov + cov.T) * 0.5, host)


def eigh_symmetric(c):
    """Descending eigen-pairs with canonical signs (calibration.py:70-91)."""
    a, host = _core.as_device(c, torch.float64)
    if a.dim() != 2 or a.shape[0] != a.shape[1]:
        raise ShapeError(f"expected a square matrix, got {tuple(a.shape)}")
    scale = max(1.0, float(a.abs().max()))
    asym = float((a - a.T).abs().max())
    if asym > 1e-5 * scale:
        raise DomainError(f"matrix is not symmetric: max asymmetry {asym:.3e}")
    vals, vecs = torch.linalg.eigh((a + a.T) * 0.5)
    order = torch.argsort(-vals, stable=True)
    vals, vecs = vals[order], vecs[:, order]
    picks = vecs.abs().argmax(dim=0)
    signs = torch.where(vecs[picks, torch.arange(vecs.shape[1], device=vecs.device)] < 0.0, -1.0, 1.0)
    return _core.back(vals, host), _core.back(vecs * signs, host)


def build_projection(keys, rotary_stage: str, layer: int = 0, head: int = 0) -> ProjectionSet:
    """Calibrate P from an S x D key matrix (calibration.py:94-123)."""
    if rotary_stage not in ROTARY_STAGES:
        raise DomainError(f"rotary_stage must be one of {ROTARY_STAGES}, got {rotary_stage!r}")
    k, host = _core.as_device(keys, torch.float64)
    if k.dim() != 2:
        raise ShapeError(f"keys must be 2-D, got ndim={k.dim()}")
    if not bool(torch.isfinite(k).all()):
        raise DomainError("keys contain NaN or Inf")
    s, d = k.shape
    if s < d:
        logger.warning("calibrating with S=%d < D=%d rows; spectrum will be rank-deficient", s, d)
    cov = compute_covariance(k, center=True)
    vals, vecs = eigh_symmetric(cov)
    vals = vals.clamp(min=0.0)
    total = float(vals.sum())
    if total <= 0.0:
        raise DegenerateCalibrationError("keys carry no variance in any direction")
    P = vecs.to(torch.float32).contiguous()
    eig = (vals / total).to(torch.float32)
    return ProjectionSet(layer=layer, head=head, P=_core.back(P, host), eigenvalues=_core.back(eig, host),
                         rotary_stage=rotary_stage)


def stack_projections(projs) -> ProjectionSet:
    """Bank of per-KV-head projections -> one ProjectionSet with P [Hkv, D, D]."""
    projs = list(projs)
    P = torch.stack([torch.as_tensor(np.asarray(p.P) if not isinstance(p.P, torch.Tensor) else p.P)
                     .to(torch.float32) for p in projs])
    eig = torch.stack([torch.as_tensor(np.asarray(p.eigenvalues) if not isinstance(p.eigenvalues, torch.Tensor)
                                       else p.eigenvalues).to(torch.float32) for p in projs])
    return ProjectionSet(layer=projs[0].layer, head=-1, P=P, eigenvalues=eig, rotary_stage=projs[0].rotary_stage)


def rank_at_v(eigenvalues, v) -> int:
    """Smallest d whose leading normalised eigenvalues reach v percent (calibration.py:126-148)."""
    lam = np.asarray(eigenvalues.cpu() if isinstance(eigenvalues, torch.Tensor) else eigenvalues,
                     dtype=np.float64).reshape(-1)
    if lam.size == 0:
        raise DomainError("empty spectrum")
    if not 0.0 < v <= 100.0:
        raise DomainError(f"v must lie in (0, 100], got {v}")
    if np.any(lam < -1e-9) or np.any(np.diff(lam) > 1e-9):
        raise DomainError("eigenvalues must be nonnegative and descending")
    total = float(lam.sum())
    if abs(total - 1.0) > 1e-6:
        raise DomainError(f"eigenvalues must sum to 1 (+-1e-6), got {total}")
    cum = np.cumsum(lam)
    target = total * (1.0 - 1e-12) if v >= 100.0 else v / 100.0 - 1e-9
    return int(np.searchsorted(cum, target) + 1)
