"""Loki attention on B200 -- mirrors lokiattn/attention.py:40-341 (hot path).

Reference semantics per (batch, query head): approximate scores over the
leading d PCA columns, top-k with the lowest-index tie rule, softmax over the
selected full-width logits / sqrt(D), weighted sum of the selected values.
The reference is single-head and single-query; this module keeps those call
forms (q [D], K [S, D]) and adds batched forms (q [B, Hq, D], caches
[B, Hkv, S_cap, D], GQA head h -> KV head h // (Hq / Hkv)) defined as
independent per-(batch, head) applications of the same semantics.

Every compute step runs in libloki_b200.so (sm_100a): fused decode
(phase 1 approx scores, phase 2 radix top-k, phase 3 sparse flash-decode)
and the K0 transform/append kernel.  No CPU fallback.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _core, _lib
from .calibration import ProjectionSet
from .errors import BudgetError, DomainError, ShapeError
from .rope import RopeParams

# ------------------------------------------------------------------ budgets


def resolve_fraction(fraction: float, total: int) -> int:
    """clamp(floor(f * total + 0.5), 1, total) (attention.py:40-46)."""
    if not 0.0 < fraction <= 1.0:
        raise DomainError(f"budget fraction must lie in (0, 1], got {fraction}")
    if total < 1:
        raise BudgetError(f"total must be >= 1, got {total}")
    return int(min(max(math.floor(fraction * total + 0.5), 1), total))


@dataclass(frozen=True)
class LokiConfig:
    """Budget fractions: k_f of cached tokens, d_f of the head dim (attention.py:49-64)."""

    k_f: float
    d_f: float

    def __post_init__(self):
        for name in ("k_f", "d_f"):
            f = getattr(self, name)
            if not 0.0 < f <= 1.0:
                raise DomainError(f"{name} must lie in (0, 1], got {f}")

    def resolve(self, head_dim: int, seq_len: int):
        """Integer (d, k) for a head dim and cache length."""
        return resolve_fraction(self.d_f, head_dim), resolve_fraction(self.k_f, seq_len)


@dataclass(frozen=True)
class LokiDiagnostics:
    """indices int64 [.., k] ascending, approx_scores fp32 [.., S], weights fp32 [.., k]."""

    indices: object
    approx_scores: object
    weights: object


class RotaryComposition(str, Enum):
    """How a calibrated P composes with rotary application (attention.py:309-313)."""

    ROTATE_THEN_PROJECT = "rotate-then-project"
    PROJECT_THEN_ROTATE = "project-then-rotate"


_ROPE_CODE = {RotaryComposition.ROTATE_THEN_PROJECT: _lib.ROPE_ROTATE_THEN_PROJECT,
              RotaryComposition.PROJECT_THEN_ROTATE: _lib.ROPE_PROJECT_THEN_ROTATE}

# ------------------------------------------------------------------ cache


class KvCache:
    """Append-only cache of transformed keys and values in HBM (attention.py:67-113).

    KvCache(head_dim) is the reference's single-head cache ([len, D] views).
    KvCache(head_dim, batch=B, kv_heads=H, dtype=torch.bfloat16) is the batched
    layout [B, H, capacity, D] used by the decode kernels.  Capacity doubles on
    overflow like the reference; rows are never reordered or dropped.
    """

    def __init__(self, head_dim: int, capacity: int = 64, *, batch: int | None = None,
                 kv_heads: int | None = None, dtype=torch.float32, device=None):
        if head_dim < 1:
            raise ShapeError("head_dim must be >= 1")
        self.head_dim = head_dim
        self.batched = batch is not None or kv_heads is not None
        self.batch = batch or 1
        self.kv_heads = kv_heads or 1
        self.dtype = dtype
        self.device = torch.device(device) if device is not None else _core.current_device()
        cap = max(int(capacity), 1)
        shape = (self.batch, self.kv_heads, cap, head_dim)
        self._k = torch.empty(shape, dtype=dtype, device=self.device)
        self._v = torch.empty(shape, dtype=dtype, device=self.device)
        self._len = 0
        self.lens = torch.zeros(self.batch, dtype=torch.int32, device=self.device)

    def __len__(self) -> int:
        return self._len

    @property
    def capacity(self) -> int:
        return self._k.shape[2]

    @property
    def storage(self):
        """Full [B, H, capacity, D] key / value buffers (kernel geometry)."""
        return self._k, self._v

    def _view(self, t):
        v = t[:, :, : self._len]
        return v if self.batched else v[0, 0]

    @property
    def keys(self):
        return self._view(self._k)

    @property
    def values(self):
        return self._view(self._v)

    def reserve(self, rows: int) -> None:
        """Grow capacity to hold `rows` (doubling), copying the filled prefix."""
        cap = self.capacity
        if rows <= cap:
            return
        while cap < rows:
            cap *= 2
        shape = (self.batch, self.kv_heads, cap, self.head_dim)
        k = torch.empty(shape, dtype=self.dtype, device=self.device)
        v = torch.empty(shape, dtype=self.dtype, device=self.device)
        k[:, :, : self._len] = self._k[:, :, : self._len]
        v[:, :, : self._len] = self._v[:, :, : self._len]
        self._k, self._v = k, v

    def _rows_tensor(self):
        return self.lens  # the next free row per batch == current length

    def advance(self, n: int = 1) -> None:
        self._len += n
        self.lens.fill_(self._len)

    def append(self, k_hat, v) -> None:
        """Append already-transformed rows (attention.py:97-113)."""
        kk, _ = _core.as_device(k_hat, torch.float32, device=self.device)
        vv, _ = _core.as_device(v, torch.float32, device=self.device)
        want = (self.batch, self.kv_heads, self.head_dim) if self.batched else (self.head_dim,)
        if not self.batched:
            kk, vv = kk.reshape(-1), vv.reshape(-1)
        if tuple(kk.shape) != want or tuple(vv.shape) != want:
            raise ShapeError(f"appended rows must have length {self.head_dim}, "
                             f"got {tuple(kk.shape)} and {tuple(vv.shape)}")
        self.reserve(self._len + 1)
        _append_call(None, kk, vv, None, None, _lib.ROPE_NONE, self, None, None)
        self.advance(1)


def cache_append(cache: KvCache, k_hat, v) -> KvCache:
    """Functional spelling of KvCache.append (attention.py:116-119)."""
    cache.append(k_hat, v)
    return cache


def _append_call(q_raw, k_raw, v_new, P, inv_freq, rope_mode, cache, positions, q_hat_out, Hq=None):
    K, V = cache.storage
    geom = _core.geom_of(K, Hq or cache.kv_heads)
    P_stride = 0
    if P is not None and P.dim() == 3:
        P_stride = P.stride(0)
    lib = _lib.lib_for(cache.device)
    with _core.on_device(cache.device):
        _lib.check(lib.loki_append_kv(_lib.ptr(q_raw), _lib.ptr(k_raw), _lib.ptr(v_new), _lib.ptr(P), P_stride,
                                      _lib.ptr(inv_freq), _lib.ptr(positions), rope_mode, K.data_ptr(),
                                      V.data_ptr(), geom, cache._rows_tensor().data_ptr(), _lib.ptr(q_hat_out),
                                      _core.stream_of(cache.device)))


# ------------------------------------------------------------------ validation


def _check_qkv(q, K, V):
    """attention.py:122-134, same messages."""
    q, host = _core.as_device(q, torch.float32)
    q = q.reshape(-1)
    K, _ = _core.as_device(K, torch.float32, device=q.device, keep_dtype=True)
    V, _ = _core.as_device(V, torch.float32, device=q.device, keep_dtype=True)
    if K.dim() != 2 or V.dim() != 2:
        raise ShapeError("keys and values must be 2-D")
    if K.shape != V.shape:
        raise ShapeError(f"keys {tuple(K.shape)} and values {tuple(V.shape)} disagree")
    if K.shape[0] < 1:
        raise ShapeError("attention needs at least one cached token")
    if K.shape[1] != q.shape[0]:
        raise ShapeError(f"query dim {q.shape[0]} does not match key dim {K.shape[1]}")
    if K.dtype not in (torch.float32, torch.bfloat16):
        K = K.float()
    if V.dtype != K.dtype:
        V = V.to(K.dtype)
    return q, K, V, host


def _single(q, K, V, d, select_mode, k, want_idx=True, want_approx=True, want_weights=True):
    S, D = K.shape
    dev = q.device
    lens, _ = _core.lens_tensor(S, 1, dev)
    kk = S if select_mode == _lib.SELECT_ALL else k
    out = torch.empty((1, 1, D), dtype=torch.float32, device=dev)
    idx = torch.empty((1, 1, kk), dtype=torch.int32, device=dev) if want_idx else None
    approx = torch.empty((1, 1, S), dtype=torch.float32, device=dev) if want_approx else None
    weights = torch.empty((1, 1, kk), dtype=torch.float32, device=dev) if want_weights else None
    call = _core.DecodeCall(q.reshape(1, 1, D), K.reshape(1, 1, S, D), V.reshape(1, 1, S, D), lens, S, d,
                            k_fixed=kk if select_mode != _lib.SELECT_ALL else 0, select_mode=select_mode,
                            idx_stride=kk, out=out, idx_out=idx, approx_out=approx, weights_out=weights)
    call.run()
    return out.reshape(D), idx, approx, weights


# ------------------------------------------------------------------ public API


def vanilla_attention(q, K, V):
    """Full attention: (output [D], softmax weights [S]) (attention.py:137-142)."""
    q, K, V, host = _check_qkv(q, K, V)
    y, _, _, w = _single(q, K, V, 1, _lib.SELECT_ALL, 0, want_idx=False, want_approx=False)
    return _core.back(y, host), _core.back(w.reshape(-1), host)


def exact_topk_attention(q, K, V, k: int):
    """Rank by exact logits K q, attend to the top k (attention.py:145-156).
    On the GPU this is the fused kernel with full-width ranking (d = D)."""
    q, K, V, host = _check_qkv(q, K, V)
    S, D = K.shape
    if not 1 <= k <= S:
        raise BudgetError(f"k={k} outside [1, {S}]")
    y, idx, _, _ = _single(q, K, V, D, _lib.SELECT_TOPK, k, want_approx=False, want_weights=False)
    return _core.back(y, host), _core.back(idx.reshape(-1).to(torch.int64), host)


def pca_attn(q, K_hat_d, V, P_d):
    """Attend to every token using only leading-d coordinates (attention.py:209-232): the
    cache holds K_hat[:, :d]; logits q_hat[:d] . K_hat[j, :d] / sqrt(D) (the full head
    dimension), softmax over all rows, no selection.  A quality baseline,
    composed from the device kernels: the query projection (cuBLAS matvec), the sliced
    score kernel, the fp64 softmax kernel and the dense weighted-sum kernel."""
    from .kernels import dense_weighted_sum_kernel, sliced_score_kernel
    from .linalg import softmax_rows

    qt, host = _core.as_device(q, torch.float32)
    qt = qt.reshape(-1)
    Kd, _ = _core.as_device(K_hat_d, torch.float32, device=qt.device)
    Vt, _ = _core.as_device(V, torch.float32, device=qt.device)
    Pd, _ = _core.as_device(P_d, torch.float32, device=qt.device)
    if Pd.dim() != 2 or Pd.shape[0] != qt.shape[0]:
        raise ShapeError(f"P_d shape {tuple(Pd.shape)} does not match query dim {qt.shape[0]}")
    d = Pd.shape[1]
    if Kd.dim() != 2 or Kd.shape[1] != d:
        raise ShapeError(f"reduced keys {tuple(Kd.shape)} do not match P_d width {d}")
    if Vt.dim() != 2 or Vt.shape[0] != Kd.shape[0] or Vt.shape[0] < 1:
        raise ShapeError(f"values {tuple(Vt.shape)} do not match keys {tuple(Kd.shape)}")
    D = Pd.shape[0]
    q_hat_d = (qt @ Pd).contiguous()
    logits = sliced_score_kernel(q_hat_d, Kd.contiguous(), d) / np.float32(math.sqrt(D))
    w = softmax_rows(logits.reshape(1, -1)).reshape(-1)
    return _core.back(dense_weighted_sum_kernel(w, Vt), host)


def loki_rank_and_attend(q_hat, K_hat, V, d: int, k: int):
    """Reduced-dimension top-k step over an existing cache (attention.py:166-185).

    Single head: q_hat [D], K_hat / V [S, D] -> (y [D], LokiDiagnostics).
    Batched:     q_hat [B, Hq, D], K_hat / V [B, Hkv, S, D] -> (y [B, Hq, D], diag).
    """
    qt = q_hat if isinstance(q_hat, torch.Tensor) else np.asarray(q_hat)
    if getattr(qt, "ndim", 1) == 3:
        y, diag = loki_decode(q_hat, K_hat, V, None, d=d, k=k, diagnostics=True)
        return y, diag
    q, K, V, host = _check_qkv(q_hat, K_hat, V)
    S, D = K.shape
    if not 1 <= d <= D:
        raise BudgetError(f"d={d} outside [1, {D}]")
    if not 1 <= k <= S:
        raise BudgetError(f"k={k} outside [1, {S}]")
    y, idx, approx, w = _single(q, K, V, d, _lib.SELECT_TOPK, k)
    diag = LokiDiagnostics(indices=_core.back(idx.reshape(-1).to(torch.int64), host),
                           approx_scores=_core.back(approx.reshape(-1), host),
                           weights=_core.back(w.reshape(-1), host))
    return _core.back(y, host), diag


def _proj_tensor(proj: ProjectionSet, device) -> torch.Tensor:
    P = proj.P if isinstance(proj.P, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(proj.P))
    return P.to(device=device, dtype=torch.float32).contiguous()


def loki_attention(q, k_new, v_new, cache: KvCache, proj: ProjectionSet, cfg: LokiConfig):
    """One generation step: project, append, rank in leading-d, attend (attention.py:188-206).

    q / k_new / v_new are in the rotary stage P was built for.  Single-head
    caches take [D] vectors; batched caches take q [B, Hq, D] and
    k_new / v_new [B, Hkv, D] with P [D, D] (shared) or [Hkv, D, D].
    """
    if proj.head_dim != cache.head_dim:
        raise ShapeError(f"projection dim {proj.head_dim} does not match cache dim {cache.head_dim}")
    dev = cache.device
    qq, host = _core.as_device(q, torch.float32, device=dev)
    kk, _ = _core.as_device(k_new, torch.float32, device=dev)
    vv, _ = _core.as_device(v_new, torch.float32, device=dev)
    D = cache.head_dim
    if cache.batched:
        B, Hkv = cache.batch, cache.kv_heads
        if qq.dim() != 3 or qq.shape[0] != B or qq.shape[2] != D or qq.shape[1] % Hkv:
            raise ShapeError(f"queries {tuple(qq.shape)} do not match cache [B={B}, Hkv={Hkv}, D={D}]")
        Hq = qq.shape[1]
    else:
        qq = qq.reshape(1, 1, -1)
        Hq = 1
    want = (cache.batch, cache.kv_heads, D)
    if kk.numel() != math.prod(want) or vv.numel() != math.prod(want) or qq.shape[-1] != D:
        raise ShapeError(f"appended rows must have length {D}, got {tuple(kk.shape)} and {tuple(vv.shape)}")
    kk, vv = kk.reshape(want).contiguous(), vv.reshape(want).contiguous()
    P = _proj_tensor(proj, dev)
    q_hat = torch.empty((cache.batch, Hq, D), dtype=torch.float32, device=dev)
    cache.reserve(len(cache) + 1)
    _append_call(qq.contiguous(), kk, vv, P, None, _lib.ROPE_NONE, cache, None, q_hat, Hq=Hq)
    cache.advance(1)
    d, k = cfg.resolve(D, len(cache))
    Kc, Vc = cache.storage
    if cache.batched:
        y, diag = loki_decode(q_hat, Kc, Vc, cache.lens, d=d, k=k, diagnostics=True, S_max=len(cache))
    else:
        y, diag = loki_rank_and_attend(q_hat.reshape(-1), cache.keys, cache.values, d, k)
    if host:
        y = y.cpu().numpy()
        diag = LokiDiagnostics(*(x.cpu().numpy() for x in (diag.indices, diag.approx_scores, diag.weights)))
    return y, diag


def transform_step(q_raw, k_raw, position: int, proj: ProjectionSet, rope_params: RopeParams,
                   mode: RotaryComposition = RotaryComposition.ROTATE_THEN_PROJECT):
    """(q_hat, k_hat) for one raw pre-rotary pair (attention.py:316-341), on the K0 kernel."""
    qq, host = _core.as_device(q_raw, torch.float32)
    dev = qq.device
    kk, _ = _core.as_device(k_raw, torch.float32, device=dev)
    qq, kk = qq.reshape(-1), kk.reshape(-1)
    D = rope_params.head_dim
    if qq.numel() != D or kk.numel() != D:
        raise ShapeError(f"vector length {tuple(qq.shape)} does not match head_dim {D}")
    if position < 0:
        raise DomainError(f"position must be nonnegative, got {position}")
    mode = RotaryComposition(mode)
    P = _proj_tensor(proj, dev)
    scratch = KvCache(D, 1, batch=1, kv_heads=1, dtype=torch.float32, device=dev)
    q_hat = torch.empty((1, 1, D), dtype=torch.float32, device=dev)
    pos = torch.tensor([int(position)], dtype=torch.int64, device=dev)
    inv = _core.inv_freq_device(D, rope_params.base, dev)
    _append_call(qq.reshape(1, 1, D), kk.reshape(1, 1, D), None, P, inv, _ROPE_CODE[mode], scratch, pos, q_hat)
    k_hat = scratch.storage[0][0, 0, 0].clone()
    return _core.back(q_hat.reshape(D), host), _core.back(k_hat, host)


# ------------------------------------------------------------------ batched hot path


def loki_decode(q_hat, K_hat, V, lens=None, *, d=None, k=None, k_f=None, cfg: LokiConfig | None = None,
                diagnostics=False, S_max=None, out=None, cluster=0, group_select="per_head"):
    """Batched Loki decode attention on the device (the north-star hot path).

    q_hat [B, Hq, D] fp32 (PCA basis); K_hat / V [B, Hkv, S_cap, D] fp32 or bf16
    (row-contiguous views are used in place: a [:, :, :S] slice of a capacity
    buffer is addressed as that buffer, never copied); lens [B] valid rows per
    batch (default S_cap).  Budget: d and either a fixed k or a fraction k_f (resolved per
    batch on the device exactly like resolve_fraction), or cfg=LokiConfig.
    Returns y [B, Hq, D] fp32 and, with diagnostics=True, LokiDiagnostics with
    indices int64 [B, Hq, k_max] (-1 past a row's k), approx_scores
    [B, Hq, S_cap] and weights [B, Hq, k_max].

    group_select (GQA): "per_head" (default, the reference's semantics: every query head ranks
    and selects on its own scores) or "shared" (opt-in: the heads of a KV group share one
    selection, ranked on the group's summed leading-d scores -- the composition of the
    reference's sliced_score_kernel on the [G, D] query block, a sum over the group,
    topk_indices, then per-head attention; bf16 caches).  The two coincide when Hq == Hkv.
    """
    mode = _select_mode(group_select)
    q, host = _core.as_device(q_hat, torch.float32)
    K, _ = _core.as_device(K_hat, torch.float32, device=q.device, keep_dtype=True, rows_only=True)
    Vt, _ = _core.as_device(V, torch.float32, device=q.device, keep_dtype=True, rows_only=True)
    if q.dim() != 3 or K.dim() != 4 or Vt.shape != K.shape:
        raise ShapeError(f"expected q [B, Hq, D] and K, V [B, Hkv, S, D]; got {tuple(q.shape)}, "
                         f"{tuple(K.shape)}, {tuple(Vt.shape)}")
    B, Hq, D = q.shape
    if K.shape[0] != B or K.shape[3] != D or Hq % K.shape[1]:
        raise ShapeError(f"queries {tuple(q.shape)} do not match cache {tuple(K.shape)}")
    S_cap = K.shape[2]  # the view's rows; the kernels may address a larger buffer behind it (geom_of)
    if K.stride() != Vt.stride():  # one geometry describes both caches
        K, Vt = K.contiguous(), Vt.contiguous()
    phys = _core.row_capacity(K)
    lens_t, lens_h = _core.lens_tensor(S_cap if lens is None else lens, B, q.device)
    if S_max is None:
        S_max = max(lens_h) if lens_h is not None else S_cap
    if not 1 <= S_max <= S_cap:
        raise ShapeError(f"S_max {S_max} outside [1, {S_cap}]")
    if lens_h is not None and max(lens_h) > S_cap:
        raise ShapeError(f"lens {max(lens_h)} exceed the cache view's {S_cap} rows")
    if lens_h is not None and min(lens_h) < 1:
        raise ShapeError("attention needs at least one cached token")
    if cfg is not None:
        d = resolve_fraction(cfg.d_f, D)
        k_f = cfg.k_f
    if d is None or not 1 <= d <= D:
        raise BudgetError(f"d={d} outside [1, {D}]")
    if k is not None:
        lo = min(lens_h) if lens_h is not None else S_max
        if not 1 <= k <= lo:
            raise BudgetError(f"k={k} outside [1, {lo}]")
        kmax = int(k)
    elif k_f is not None:
        if not 0.0 < k_f <= 1.0:
            raise DomainError(f"budget fraction must lie in (0, 1], got {k_f}")
        kmax = resolve_fraction(k_f, S_max)
    else:
        raise BudgetError("one of k, k_f or cfg is required")
    y = out if out is not None else torch.empty((B, Hq, D), dtype=torch.float32, device=q.device)
    idx = approx = w = None
    if diagnostics:
        idx = torch.full((B, Hq, kmax), -1, dtype=torch.int32, device=q.device)
        approx = torch.zeros((B, Hq, phys), dtype=torch.float32, device=q.device)
        w = torch.zeros((B, Hq, kmax), dtype=torch.float32, device=q.device)
    call = _core.DecodeCall(q, K, Vt, lens_t, S_max, d, k_f=k_f or 0.0, k_fixed=k or 0,
                            select_mode=mode, idx_stride=kmax, out=y, idx_out=idx,
                            approx_out=approx, weights_out=w, cluster=cluster)
    call.run()
    if not diagnostics:
        return _core.back(y, host)
    diag = LokiDiagnostics(indices=_core.back(idx.to(torch.int64), host),
                           approx_scores=_core.back(approx[..., :S_cap], host),
                           weights=_core.back(w, host))
    return _core.back(y, host), diag


def _select_mode(group_select) -> int:
    if group_select == "per_head":
        return _lib.SELECT_TOPK
    if group_select == "shared":
        return _lib.SELECT_TOPK_SHARED
    raise DomainError(f"group_select must be 'per_head' or 'shared', got {group_select!r}")


def dense_decode(q, K, V, lens=None, *, S_max=None, out=None, cluster=0):
    """Batched full attention softmax(K q / sqrt(D)) V (vanilla_attention,
    attention.py:137-142) on the same kernel with every row selected."""
    qq, host = _core.as_device(q, torch.float32)
    Kt, _ = _core.as_device(K, torch.float32, device=qq.device, keep_dtype=True, rows_only=True)
    Vt, _ = _core.as_device(V, torch.float32, device=qq.device, keep_dtype=True, rows_only=True)
    if Kt.stride() != Vt.stride():
        Kt, Vt = Kt.contiguous(), Vt.contiguous()
    B, Hq, D = qq.shape
    S_cap = Kt.shape[2]
    lens_t, lens_h = _core.lens_tensor(S_cap if lens is None else lens, B, qq.device)
    if S_max is None:
        S_max = max(lens_h) if lens_h is not None else S_cap
    y = out if out is not None else torch.empty((B, Hq, D), dtype=torch.float32, device=qq.device)
    _core.DecodeCall(qq, Kt, Vt, lens_t, S_max, D, select_mode=_lib.SELECT_ALL, out=y, cluster=cluster).run()
    return _core.back(y, host)


class LokiDecoder:
    """Prepared decode step for the serving loop (no per-step allocation or
    Python-side validation; CUDA-graph capturable).

    Holds a KvCache-style storage and runs, per step:
      K0  loki_append_kv: q_raw/k_raw (+RoPE) -> q_hat, K_hat row, V row
      K1-3 loki_decode:   fused approx scores -> top-k -> sparse attention
    `rows` / `lens` are device int32 [B] tensors owned by the caller.  S_max (default: the
    cache capacity K.shape[2]) sizes the launch plan and is frozen into a captured graph:
    a row whose len exceeds it attends over its first S_max rows only, so a serving loop
    that grows lens between replays keeps the default.
    """

    def __init__(self, K, V, P, *, Hq, d, k_f=None, k=None, rows, lens, S_max=None, q_raw, k_raw, v_new,
                 rope_mode=_lib.ROPE_NONE, rope_base=10000.0, positions=None, dense=False, out=None, cluster=0,
                 group_select="per_head"):
        self.device = K.device
        self.lib = _lib.lib_for(self.device)
        self.K, self.V, self.P = K, V, P
        self.geom = _core.geom_of(K, Hq)
        B, _, _, D = K.shape
        self.q_raw, self.k_raw, self.v_new = q_raw, k_raw, v_new
        self.rows, self.lens, self.positions = rows, lens, positions
        self.rope_mode = rope_mode
        self.inv = _core.inv_freq_device(D, rope_base, self.device) if rope_mode != _lib.ROPE_NONE else None
        self.q_hat = torch.empty((B, Hq, D), dtype=torch.float32, device=self.device)
        self.out = out if out is not None else torch.empty((B, Hq, D), dtype=torch.float32, device=self.device)
        self.P_stride = P.stride(0) if (P is not None and P.dim() == 3) else 0
        self.dense = dense
        self._append_args = None
        S_max = K.shape[2] if S_max is None else int(S_max)
        if not 1 <= S_max <= K.shape[2]:
            raise ShapeError(f"S_max {S_max} outside [1, {K.shape[2]}]")
        self.call = _core.DecodeCall(self.q_hat, K, V, lens, S_max, d, k_f=k_f or 0.0, k_fixed=k or 0,
                                     select_mode=_lib.SELECT_ALL if dense else _select_mode(group_select),
                                     out=self.out,
                                     Hq=Hq, cluster=cluster)

    def append(self, stream):
        if self._append_args is None:  # pointers are stable: build the argument list once
            self._append_args = (
                _lib.ptr(self.q_raw), _lib.ptr(self.k_raw), _lib.ptr(self.v_new), _lib.ptr(self.P), self.P_stride,
                _lib.ptr(self.inv), _lib.ptr(self.positions), self.rope_mode, self.K.data_ptr(), self.V.data_ptr(),
                self.geom, self.rows.data_ptr(), self.q_hat.data_ptr())
        with _core.on_device(self.device):
            _lib.check(self.lib.loki_append_kv(*self._append_args, stream))

    def attend(self, stream):
        self.call.run(stream)

    def step(self, stream=None):
        s = stream if stream is not None else _core.stream_of(self.device)
        self.append(s)
        self.attend(s)
        return self.out


class DecodeGraph:
    """One decode step over a stack of layers -- `LokiDecoder.step` per layer in
    order, optionally followed by `between(layer)` (e.g. the head all-gather of a
    sharded layer) -- captured once as a CUDA graph and replayed per token, so the
    serving loop pays one graph launch instead of ~3 host launches per layer.

    Replays read the decoders' q_raw / k_raw / v_new / rows / lens buffers as they
    are at replay time (write the next token's inputs into them, then `replay()`).
    Capture runs the step `warmup` + 1 times on a side stream: like any step, each
    run writes the new K_hat / V rows at `rows` (the caller advances rows / lens).

    Host-fed steps: `inputs[layer]` = [(device_tensor, pinned_host_tensor), ...]
    makes the graph copy that layer's inputs from host memory on a copy stream,
    each layer waiting only for its own copies, so layer l + 1's transfer overlaps
    layer l's kernels; `output` = (pinned_host_tensor, device_tensor) copies the
    result back at the end of the graph.  The host tensors are read / written at
    replay time.
    """

    def __init__(self, decoders, between=None, warmup: int = 2, inputs=None, output=None):
        if not decoders:
            raise ShapeError("DecodeGraph needs at least one LokiDecoder")
        self.decoders = list(decoders)
        self.between = between
        if inputs is not None and len(inputs) != len(self.decoders):
            raise ShapeError(f"{len(inputs)} input lists for {len(self.decoders)} layers")
        self.inputs = inputs
        self.output = output
        dev = self.decoders[0].device
        self._copy = torch.cuda.Stream(dev) if inputs is not None else None
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for _ in range(warmup):
                self._run()
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._run()
        torch.cuda.synchronize(dev)

    def _run(self):
        main = torch.cuda.current_stream()
        events = []
        if self.inputs is not None:  # every layer's host -> device copies, queued ahead on the copy stream
            self._copy.wait_stream(main)
            with torch.cuda.stream(self._copy):
                for pairs in self.inputs:
                    for dst, src in pairs:
                        dst.copy_(src, non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(self._copy)
                    events.append(ev)
        for layer, dec in enumerate(self.decoders):
            if events:
                main.wait_event(events[layer])
            dec.step()
            if self.between is not None:
                self.between(layer)
        if self.output is not None:
            host, dev_t = self.output
            host.copy_(dev_t, non_blocking=True)

    def replay(self):
        """Launch the captured step on the current stream; returns the last layer's output."""
        self.graph.replay()
        return self.decoders[-1].out

