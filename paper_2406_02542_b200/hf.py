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

from . import _lib
from .attention import LokiConfig, loki_decode
from .calibration import build_projection
from .errors import ShapeError, UnsupportedShapeError

try:  # transformers is optional for the rest of the package
    from transformers import AttentionInterface, DynamicCache
except ImportError:  # pragma: no cover - depends on the environment
    AttentionInterface = None
    DynamicCache = object

ATTN_NAME = "loki"


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return _lib.DTYPE_F32
    if t.dtype == torch.bfloat16:
        return _lib.DTYPE_BF16
    raise UnsupportedShapeError(f"projection dtype {t.dtype} (float32 or bfloat16 only)")


def project_rows(x: torch.Tensor, P: torch.Tensor, out_dtype=None) -> torch.Tensor:
    """out[b, h, s] = x[b, h, s] . P[h // (H / P.shape[0])] on the device (loki_project_rows).

    x [B, H, S, D] (D contiguous, f32 / bf16), P [Hp, D, D] fp32 with H % Hp == 0.
    """
    if x.dim() != 4 or x.stride(3) != 1:
        raise ShapeError(f"expected x [B, H, S, D] with contiguous rows, got {tuple(x.shape)}")
    B, H, S, D = x.shape
    if P.dim() != 3 or P.shape[1:] != (D, D) or H % P.shape[0]:
        raise ShapeError(f"projection {tuple(P.shape)} does not match x {tuple(x.shape)}")
    P = P.to(device=x.device, dtype=torch.float32).contiguous()
    out = torch.empty((B, H, S, D), dtype=out_dtype or x.dtype, device=x.device)
    xs = (ctypes.c_int64 * 3)(x.stride(0), x.stride(1), x.stride(2))
    os_ = (ctypes.c_int64 * 3)(out.stride(0), out.stride(1), out.stride(2))
    lib = _lib.lib_for(x.device)
    _lib.check(lib.loki_project_rows(x.data_ptr(), _dtype_code(x), ctypes.addressof(xs), P.data_ptr(),
                                     out.data_ptr(), _dtype_code(out), ctypes.addressof(os_), B, H, S, D,
                                     H // P.shape[0], torch.cuda.current_stream(x.device).cuda_stream))
    return out


class LokiCache(DynamicCache):
    """DynamicCache whose keys are stored PCA-rotated: K_hat = k_rot . P[layer]."""

    def __init__(self, projections, *args, **kwargs):
        super().__init__(*args, **kwargs)
        self.loki_P = [p.to(torch.float32).contiguous() for p in projections]

    def update(self, key_states, value_states, layer_idx, *args, **kwargs):
        k_hat = project_rows(key_states.contiguous(), self.loki_P[layer_idx])
        return super().update(k_hat, value_states, layer_idx, *args, **kwargs)


def loki_attention_forward(module, query, key, value, attention_mask, scaling, dropout=0.0, **kwargs):
    """The "loki" attention implementation: query [B, Hq, q, D] post-RoPE, key =
    K_hat [B, Hkv, S, D] from a LokiCache, value [B, Hkv, S, D]."""
    P = getattr(module, "loki_P", None)
    cfg = getattr(module, "loki_cfg", None)
    if P is None or cfg is None:
        raise UnsupportedShapeError("attention module has no Loki projection: call hf.install(model, ...)")
    q_hat = project_rows(query.contiguous(), P, out_dtype=torch.float32)
    B, Hq, q_len, D = query.shape
    if q_len == 1 and key.shape[2] > 1:
        if attention_mask is not None and attention_mask.dim() == 4 and bool((attention_mask[..., -1, :] < 0).any()):
            raise UnsupportedShapeError("padding masks are not supported on the Loki decode path")
        y = loki_decode(q_hat[:, :, 0], key.contiguous(), value.contiguous(), None, cfg=cfg)
        return y.to(query.dtype)[:, None], None
    # prefill: dense causal attention on the rotated tensors (P orthogonal: same logits)
    out = F.scaled_dot_product_attention(q_hat.to(key.dtype), key, value, attn_mask=None, is_causal=q_len > 1,
                                         scale=scaling, enable_gqa=Hq != key.shape[1])
    return out.transpose(1, 2).contiguous(), None


def _attention_modules(model):
    layers = model.model.layers
    return [layer.self_attn for layer in layers]


def install(model, projections, k_f: float = 0.25, d_f: float = 0.25):
    """Route the model's attention through Loki (k_f, d_f as LokiConfig); returns the model."""
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
