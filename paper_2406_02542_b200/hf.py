"""HF transformers integration of the Loki decode path.

Llama / Mistral-style decoders (transformers 5.x) switch to Loki attention:

    from paper_2406_02542_b200 import hf
    P = hf.calibrate(model, calib_ids)               # per layer [Hkv, D, D] PCA bases
    hf.install(model, P, k_f=0.25, d_f=0.25)         # attn implementation "loki"
    cache = hf.LokiCache(P)
    out = model.generate(ids, past_key_values=cache, max_new_tokens=...)

* The cache stores the PCA-rotated keys K_hat = RoPE(k) . P ("rotate then
  project", attention.py:309-341 RotaryComposition; HF hands the cache
  post-RoPE keys, which fixes the composition).  P is orthogonal, so
  q_hat . k_hat == q . k: exact attention is unchanged and the leading d
  principal components give the approximate scores (attention.py:166-185).
* Single-token decode steps run `loki_decode` (the B200 pipe kernel) on
  (q_hat, K_hat, V).  Prefill (q_len > 1) is dense causal attention on the same
  rotated tensors (library SDPA: Loki is a decode-time method).
* Projections of new keys and of the queries run `loki_project_rows`
  (csrc/loki_kernels.cu); calibration (`calibrate`) runs a prefill, collects the
  post-RoPE keys per (layer, KV head) and calls `build_projection`
  (calibration.py:51-123, `rotary_stage="post"`).

Padding masks are not supported on the Loki decode path (one sequence length
per batch row, as `loki_decode` lens); batched prompts of equal length are.
"""

from __future__ import annotations

import ctypes

import torch
import torch.nn.functional as F

from . import _core, _lib
from .attention import LokiConfig, loki_decode, resolve_fraction
from .calibration import build_projection
from .errors import ShapeError, UnsupportedShapeError

try:  # transformers is optional for the rest of the package
    from transformers import AttentionInterface, DynamicCache
    from transformers.cache_utils import Cache, CacheLayerMixin
except ImportError:  # pragma: no cover - depends on the environment
    AttentionInterface = None
    DynamicCache = Cache = CacheLayerMixin = object

ATTN_NAME = "loki"


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return _lib.DTYPE_F32
    if t.dtype == torch.bfloat16:
        return _lib.DTYPE_BF16
    raise UnsupportedShapeError(f"projection dtype {t.dtype} (float32 or bfloat16 only)")


def project_rows(x: torch.Tensor, P: torch.Tensor, out_dtype=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """out[b, h, s] = x[b, h, s] . P[h // (H / P.shape[0])] on the device (loki_project_rows).

    x [B, H, S, D] (D contiguous, f32 / bf16), P [Hp, D, D] fp32 with H % Hp == 0.  `out` (any
    [B, H, S, D] view with contiguous rows, e.g. a slice of a cache buffer) receives the result in place.
    """
    if x.dim() != 4 or x.stride(3) != 1:
        raise ShapeError(f"expected x [B, H, S, D] with contiguous rows, got {tuple(x.shape)}")
    B, H, S, D = x.shape
    if P.dim() != 3 or P.shape[1:] != (D, D) or H % P.shape[0]:
        raise ShapeError(f"projection {tuple(P.shape)} does not match x {tuple(x.shape)}")
    if P.dtype != torch.float32 or not P.is_contiguous() or P.device != x.device:
        P = P.to(device=x.device, dtype=torch.float32).contiguous()
    if out is None:
        out = torch.empty((B, H, S, D), dtype=out_dtype or x.dtype, device=x.device)
    elif out.shape != x.shape or out.stride(3) != 1:
        raise ShapeError(f"out {tuple(out.shape)} does not match x {tuple(x.shape)}")
    xs = (ctypes.c_int64 * 3)(x.stride(0), x.stride(1), x.stride(2))
    os_ = (ctypes.c_int64 * 3)(out.stride(0), out.stride(1), out.stride(2))
    lib = _lib.lib_for(x.device)
    _lib.check(lib.loki_project_rows(x.data_ptr(), _dtype_code(x), ctypes.addressof(xs), P.data_ptr(),
                                     out.data_ptr(), _dtype_code(out), ctypes.addressof(os_), B, H, S, D,
                                     H // P.shape[0], torch.cuda.current_stream(x.device).cuda_stream))
    return out


class LokiLayer(CacheLayerMixin):
    """One layer of a LokiCache: preallocated [B, Hkv, capacity, D] buffers of PCA-rotated keys
    K_hat = k_rot . P and values (attention.py:67-119 KvCache, B200 layout: rows are written in
    place, never concatenated).  Decode steps append through K0 (loki_append_kv: P . k on the
    device, the row written at `rows`); prefill chunks are projected straight into the buffer
    slice.  Capacity doubles when exceeded (the reference KvCache's growth rule).  The decode
    attention runs one persistent DecodeCall per layer (workspace allocated once)."""

    is_sliding = False
    is_compileable = False

    def __init__(self, P: torch.Tensor, capacity: int = 0, storage_dtype=torch.bfloat16):
        super().__init__()
        self.P = P.to(torch.float32).contiguous()
        self.capacity = int(capacity)
        self.storage_dtype = storage_dtype
        self.n = 0
        self._call = None
        self._call_key = None

    def lazy_initialization(self, key_states, value_states):
        B, Hkv, _, D = key_states.shape
        self.device = key_states.device
        self.dtype = key_states.dtype
        if self.P.device != self.device:
            self.P = self.P.to(self.device)
        if self.P.shape != (Hkv, D, D):
            raise ShapeError(f"projection {tuple(self.P.shape)} does not match {Hkv} KV heads of dim {D}")
        cap = max(self.capacity, key_states.shape[2], 16)
        self._alloc(B, Hkv, cap, D)
        self.rows = torch.zeros(B, dtype=torch.int32, device=self.device)
        self.lens = torch.zeros(B, dtype=torch.int32, device=self.device)
        self.is_initialized = True

    def _alloc(self, B, Hkv, cap, D):
        self.Kbuf = torch.zeros((B, Hkv, cap, D), dtype=self.storage_dtype, device=self.device)
        self.Vbuf = torch.zeros((B, Hkv, cap, D), dtype=self.storage_dtype, device=self.device)
        self.capacity = cap
        self._call = None

    def _grow(self, need):
        B, Hkv, cap, D = self.Kbuf.shape
        new = max(2 * cap, need)
        K, V = self.Kbuf, self.Vbuf
        self._alloc(B, Hkv, new, D)
        self.Kbuf[:, :, :self.n].copy_(K[:, :, :self.n])
        self.Vbuf[:, :, :self.n].copy_(V[:, :, :self.n])

    def _views(self):
        k = self.Kbuf[:, :, :self.n]
        k._loki_layer = self  # the "loki" attention function finds the layer's persistent launch state here
        self.keys, self.values = k, self.Vbuf[:, :, :self.n]
        return self.keys, self.values

    def update(self, key_states, value_states, *args, **kwargs):
        if not self.is_initialized:
            self.lazy_initialization(key_states, value_states)
        q_len = key_states.shape[2]
        if self.n + q_len > self.capacity:
            self._grow(self.n + q_len)
        if q_len == 1:  # decode: K0 writes P . k and v at row n of every batch row
            self.rows.fill_(self.n)
            geom = _core.geom_of(self.Kbuf, self.Kbuf.shape[1])
            k = key_states[:, :, 0].float().contiguous()
            v = value_states[:, :, 0].float().contiguous()
            lib = _lib.lib_for(self.device)
            _lib.check(lib.loki_append_kv(None, k.data_ptr(), v.data_ptr(), self.P.data_ptr(), self.P.stride(0),
                                          None, None, _lib.ROPE_NONE, self.Kbuf.data_ptr(), self.Vbuf.data_ptr(),
                                          geom, self.rows.data_ptr(), None, _core.stream_of(self.device)))
        else:  # prefill chunk: projected straight into the buffer slice
            sl = slice(self.n, self.n + q_len)
            project_rows(key_states, self.P, out=self.Kbuf[:, :, sl])
            self.Vbuf[:, :, sl].copy_(value_states)
        self.n += q_len
        self.lens.fill_(self.n)
        return self._views()

    def load(self, K_hat: torch.Tensor, V: torch.Tensor, n: int):
        """Adopt existing [B, Hkv, capacity, D] buffers (already PCA-rotated keys) holding n valid rows."""
        if K_hat.shape != V.shape or K_hat.dim() != 4 or K_hat.dtype != V.dtype:
            raise ShapeError(f"K_hat {tuple(K_hat.shape)} and V {tuple(V.shape)} must match")
        if self.P.shape != (K_hat.shape[1], K_hat.shape[3], K_hat.shape[3]):
            raise ShapeError(f"projection {tuple(self.P.shape)} does not match cache {tuple(K_hat.shape)}")
        self.device, self.dtype, self.storage_dtype = K_hat.device, K_hat.dtype, K_hat.dtype
        self.P = self.P.to(self.device)
        self.Kbuf, self.Vbuf = K_hat, V
        self.capacity = K_hat.shape[2]
        self.rows = torch.zeros(K_hat.shape[0], dtype=torch.int32, device=self.device)
        self.lens = torch.zeros(K_hat.shape[0], dtype=torch.int32, device=self.device)
        self._call = self._call_key = None
        self.is_initialized = True
        self.set_length(n)

    def set_length(self, n: int):
        """Serve from the first n rows (e.g. synthetic caches, or re-decoding the token at row n)."""
        if not 0 <= n <= self.capacity:
            raise ShapeError(f"length {n} outside [0, {self.capacity}]")
        self.n = int(n)
        self.lens.fill_(self.n)
        self._views()

    def get_mask_sizes(self, query_length: int):
        return self.n + query_length, 0

    def get_seq_length(self) -> int:
        return self.n

    def get_max_cache_shape(self) -> int:
        return -1

    def attend(self, q_hat: torch.Tensor, cfg: LokiConfig, group_select: str = "per_head") -> torch.Tensor:
        """Loki decode over the layer's buffers for q_hat [B, Hq, D] fp32; returns the layer's output buffer."""
        B, Hq, D = q_hat.shape
        key = (Hq, self.capacity, cfg, group_select)
        if self._call_key != key:  # plan once per (heads, capacity): no per-token allocation or planning
            from .attention import _select_mode

            self.q_hat = torch.empty((B, Hq, D), dtype=torch.float32, device=self.device)
            self.out = torch.empty((B, Hq, D), dtype=torch.float32, device=self.device)
            d = resolve_fraction(cfg.d_f, D)
            self._call = _core.DecodeCall(self.q_hat, self.Kbuf, self.Vbuf, self.lens, self.capacity, d,
                                          k_f=cfg.k_f, select_mode=_select_mode(group_select), out=self.out,
                                          Hq=Hq)
            self._call_key = key
        self.q_hat.copy_(q_hat)
        self._call.run()
        return self.out


class LokiCache(Cache):
    """HF cache whose layers store PCA-rotated keys in preallocated buffers (LokiLayer)."""

    def __init__(self, projections, capacity: int = 0, storage_dtype=torch.bfloat16, **kwargs):
        layers = [LokiLayer(P, capacity, storage_dtype) for P in projections]
        super().__init__(layers=layers, **kwargs)
        self.loki_P = [layer.P for layer in layers]

    def set_length(self, n: int):
        for layer in self.layers:
            layer.set_length(n)


def _bottom_right_causal(q_len: int, S: int, device) -> torch.Tensor:
    """Boolean [q_len, S] mask: query i (at position S - q_len + i) sees keys j <= that position."""
    i = torch.arange(q_len, device=device)[:, None]
    j = torch.arange(S, device=device)[None, :]
    return j <= (S - q_len) + i


def loki_attention_forward(module, query, key, value, attention_mask, scaling, dropout=0.0, **kwargs):
    """The "loki" attention implementation: query [B, Hq, q, D] post-RoPE, key =
    K_hat [B, Hkv, S, D] from a LokiCache, value [B, Hkv, S, D]."""
    P = getattr(module, "loki_P", None)
    cfg = getattr(module, "loki_cfg", None)
    if P is None or cfg is None:
        raise UnsupportedShapeError("attention module has no Loki projection: call hf.install(model, ...)")
    B, Hq, q_len, D = query.shape
    if abs(scaling - D ** -0.5) > 1e-6 * D ** -0.5:
        raise UnsupportedShapeError(f"attention scale {scaling} != 1/sqrt({D}): the Loki kernels use 1/sqrt(D)")
    layer = getattr(key, "_loki_layer", None)
    if attention_mask is not None and attention_mask.dim() == 4 and attention_mask.shape[-2] >= 1:
        m = attention_mask[..., -1, :]
        blocked = (~m) if m.dtype == torch.bool else (m < 0)
        if bool(blocked.any()):  # a padded row: the decode kernels take one length per batch row
            raise UnsupportedShapeError("padding masks are not supported on the Loki path")
    q_hat = project_rows(query if query.stride(3) == 1 else query.contiguous(), P, out_dtype=torch.float32)
    if q_len == 1 and key.shape[2] > 1 and getattr(module, "loki_dense", False):
        # comparator: exact dense decode on the same rotated cache (P orthogonal: the logits of q . k)
        out = F.scaled_dot_product_attention(q_hat.to(key.dtype), key, value, scale=scaling,
                                             enable_gqa=Hq != key.shape[1])
        return out.transpose(1, 2).contiguous(), None
    if q_len == 1 and key.shape[2] > 1:
        group = getattr(module, "loki_group_select", "per_head")
        if layer is not None:  # LokiCache: persistent launch state over the preallocated buffers
            y = layer.attend(q_hat[:, :, 0], cfg, group)
        else:
            y = loki_decode(q_hat[:, :, 0], key, value, None, cfg=cfg, group_select=group)
        return y.to(query.dtype)[:, None], None
    # prefill / multi-token steps: dense attention on the rotated tensors (P orthogonal: same logits),
    # causal mask aligned to the end of the cache (the queries are its last q_len positions)
    S = key.shape[2]
    mask = _bottom_right_causal(q_len, S, query.device)
    out = F.scaled_dot_product_attention(q_hat.to(key.dtype), key, value, attn_mask=mask, scale=scaling,
                                         enable_gqa=Hq != key.shape[1])
    return out.transpose(1, 2).contiguous(), None


def _attention_modules(model):
    layers = model.model.layers
    return [layer.self_attn for layer in layers]


def install(model, projections, k_f: float = 0.25, d_f: float = 0.25, group_select: str = "per_head",
            dense: bool = False):
    """Route the model's attention through Loki (k_f, d_f as LokiConfig); returns the model.
    dense=True keeps the Loki cache but decodes with exact dense attention (a comparator)."""
    if AttentionInterface is None:
        raise UnsupportedShapeError("transformers is not installed")
    AttentionInterface.register(ATTN_NAME, loki_attention_forward)
    mods = _attention_modules(model)
    if len(projections) != len(mods):
        raise ShapeError(f"{len(projections)} projections for {len(mods)} layers")
    cfg = LokiConfig(k_f=k_f, d_f=d_f)
    for m, P in zip(mods, projections):
        m.loki_P = P.to(device=next(model.parameters()).device, dtype=torch.float32).contiguous()
        m.loki_cfg = cfg
        m.loki_group_select = group_select
        m.loki_dense = dense
    model.config._attn_implementation = ATTN_NAME
    for sub in model.modules():  # submodules keep their own config handle in some models
        cfgs = getattr(sub, "config", None)
        if cfgs is not None and hasattr(cfgs, "_attn_implementation"):
            cfgs._attn_implementation = ATTN_NAME
    return model


class _KeyCapture(DynamicCache):
    def __init__(self, *args, **kwargs):
        super().__init__(*args, **kwargs)
        self.captured = {}

    def update(self, key_states, value_states, layer_idx, *args, **kwargs):
        self.captured.setdefault(layer_idx, []).append(key_states.detach().float())
        return super().update(key_states, value_states, layer_idx, *args, **kwargs)


@torch.no_grad()
def calibrate(model, input_ids: torch.Tensor):
    """Per-layer PCA bases [Hkv, D, D] from the post-RoPE keys of one prefill
    (calibration.py:51-123 per (layer, KV head))."""
    cache = _KeyCapture()
    model(input_ids=input_ids, past_key_values=cache, use_cache=True)
    bases = []
    for layer in range(len(_attention_modules(model))):
        keys = torch.cat(cache.captured[layer], dim=2)  # [B, Hkv, S, D]
        B, Hkv, S, D = keys.shape
        per_head = []
        for h in range(Hkv):
            ps = build_projection(keys[:, h].reshape(B * S, D), rotary_stage="post")
            per_head.append(torch.as_tensor(ps.P, dtype=torch.float32))
        bases.append(torch.stack(per_head).to(keys.device))
    return bases
