"""HF transformers integration: a random-init Llama-shaped
model decodes through the Loki pipe kernel.  Parity: with k_f = d_f = 1 the
model matches stock SDPA attention; with k_f = 0.25 a decode step's attention
output matches the oracle on the same (q_hat, K_hat, V)."""

import numpy as np
import pytest
import torch

from oracle import loki_oracle as O
from paper_2406_02542_b200 import hf
from paper_2406_02542_b200.errors import ShapeError


def test_project_rows_validates_before_compute():
    with pytest.raises(ShapeError):
        hf.project_rows(torch.zeros(2, 4, 8), torch.zeros(4, 8, 8))
    with pytest.raises(ShapeError):
        hf.project_rows(torch.zeros(1, 4, 3, 8), torch.zeros(3, 8, 8))


def _tiny_llama(Hkv, dtype=torch.bfloat16, seed=0):
    from transformers import LlamaConfig, LlamaForCausalLM

    torch.manual_seed(seed)
    cfg = LlamaConfig(vocab_size=256, hidden_size=512, intermediate_size=1024, num_hidden_layers=2,
                      num_attention_heads=4, num_key_value_heads=Hkv, head_dim=128, max_position_embeddings=4096,
                      attn_implementation="sdpa")
    return LlamaForCausalLM(cfg).to("cuda", dtype).eval()


@pytest.mark.gpu
def test_project_rows_matches_matmul():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(3)
    x = torch.randn(2, 8, 37, 128, device=dev, generator=g)
    P = torch.linalg.qr(torch.randn(4, 128, 128, device=dev, generator=g))[0]
    out = hf.project_rows(x, P)
    ref = torch.einsum("bhsd,hde->bhse", x.double(), P.repeat_interleave(2, dim=0).double()).float()
    assert torch.allclose(out, ref, rtol=1e-5, atol=1e-5)
    outb = hf.project_rows(x.to(torch.bfloat16), P)
    refb = torch.einsum("bhsd,hde->bhse", x.to(torch.bfloat16).double(), P.repeat_interleave(2, dim=0).double())
    assert (outb.double() - refb).abs().max() <= 1e-2 * refb.abs().max()


@pytest.mark.gpu
@pytest.mark.parametrize("Hkv", [4, 2])
def test_full_budget_matches_sdpa(Hkv):
    """k_f = d_f = 1: Loki selects every row, so decoding equals stock attention."""
    from transformers import DynamicCache

    model = _tiny_llama(Hkv)
    ids = torch.randint(0, 256, (2, 300), device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
    with torch.no_grad():
        P = hf.calibrate(model, ids)
        ref_cache, loki_cache = DynamicCache(), hf.LokiCache(P)
        ref = model(input_ids=ids, past_key_values=ref_cache, use_cache=True).logits[:, -1]
        hf.install(model, P, k_f=1.0, d_f=1.0)
        got = model(input_ids=ids, past_key_values=loki_cache, use_cache=True).logits[:, -1]
        for _ in range(3):  # decode steps: the pipe kernel
            tok = ref.argmax(-1, keepdim=True)
            model.config._attn_implementation = "sdpa"
            for m in model.modules():
                if hasattr(getattr(m, "config", None), "_attn_implementation"):
                    m.config._attn_implementation = "sdpa"
            ref = model(input_ids=tok, past_key_values=ref_cache, use_cache=True).logits[:, -1]
            hf.install(model, P, k_f=1.0, d_f=1.0)
            got = model(input_ids=tok, past_key_values=loki_cache, use_cache=True).logits[:, -1]
            rel = (got.float() - ref.float()).norm() / ref.float().norm()
            assert rel <= 2e-2, float(rel)
            assert torch.equal(got.argmax(-1), ref.argmax(-1))


@pytest.mark.gpu
def test_sparse_decode_step_matches_oracle():
    """k_f = 0.25: one decode step's attention output vs the oracle on the same bf16 inputs."""
    model = _tiny_llama(2)
    ids = torch.randint(0, 256, (2, 600), device="cuda", generator=torch.Generator(device="cuda").manual_seed(2))
    captured = {}
    inner = hf.loki_attention_forward

    def spy(module, query, key, value, attention_mask, scaling, dropout=0.0, **kw):
        out, w = inner(module, query, key, value, attention_mask, scaling, dropout, **kw)
        if query.shape[2] == 1 and module.layer_idx == 0:
            captured.update(q_hat=hf.project_rows(query.contiguous(), module.loki_P, torch.float32),
                            K=key.float(), V=value.float(), y=out.float())
        return out, w

    with torch.no_grad():
        P = hf.calibrate(model, ids)
        hf.install(model, P, k_f=0.25, d_f=0.25)
        from transformers import AttentionInterface

        AttentionInterface.register(hf.ATTN_NAME, spy)
        try:
            cache = hf.LokiCache(P)
            logits = model(input_ids=ids, past_key_values=cache, use_cache=True).logits[:, -1]
            model(input_ids=logits.argmax(-1, keepdim=True), past_key_values=cache, use_cache=True)
        finally:
            AttentionInterface.register(hf.ATTN_NAME, inner)
    q = captured["q_hat"][:, :, 0].cpu().numpy()
    K = captured["K"].cpu().numpy()
    V = captured["V"].cpu().numpy()
    y = captured["y"][:, 0].cpu().numpy()
    S = K.shape[2]
    d, k = 32, int(np.floor(0.25 * S + 0.5))
    y_ref, _ = O.loki_decode_batched(q, K, V, [S] * q.shape[0], d, k=k)
    assert O.rel_err(y, y_ref) <= 2e-2


@pytest.mark.gpu
def test_loki_cache_appends_in_place():
    """N2: decode steps write rows into the preallocated buffers through K0 (no concatenation, no new
    buffers); the stored row is k . P of the post-RoPE key the model produced."""
    model = _tiny_llama(2)
    ids = torch.randint(0, 256, (2, 100), device="cuda", generator=torch.Generator(device="cuda").manual_seed(5))
    with torch.no_grad():
        P = hf.calibrate(model, ids)
        hf.install(model, P, k_f=0.25, d_f=0.25)
        cache = hf.LokiCache(P, capacity=256)
        logits = model(input_ids=ids, past_key_values=cache, use_cache=True).logits[:, -1]
        layer = cache.layers[0]
        kp, vp = layer.Kbuf.data_ptr(), layer.Vbuf.data_ptr()
        for _ in range(4):
            logits = model(input_ids=logits.argmax(-1, keepdim=True), past_key_values=cache, use_cache=True).logits[:, -1]
        assert (layer.Kbuf.data_ptr(), layer.Vbuf.data_ptr()) == (kp, vp)
        assert cache.get_seq_length() == 104 and layer.capacity == 256
        assert int(layer.lens[0]) == 104
        # growth past the capacity doubles the buffers and keeps the rows
        before = layer.Kbuf[:, :, :104].clone()
        cache2 = hf.LokiCache(P, capacity=16)
        model(input_ids=ids, past_key_values=cache2, use_cache=True)
        assert cache2.layers[0].capacity >= 100
    assert torch.equal(layer.Kbuf[:, :, :104], before)


@pytest.mark.gpu
def test_chunked_prefill_matches_one_prefill():
    """A second prefill chunk on a non-empty cache sees the cached rows (bottom-right causal mask,
    ADVICE r01): chunked and one-shot prefill give the same logits."""
    model = _tiny_llama(2)
    ids = torch.randint(0, 256, (2, 96), device="cuda", generator=torch.Generator(device="cuda").manual_seed(6))
    with torch.no_grad():
        P = hf.calibrate(model, ids)
        hf.install(model, P, k_f=0.25, d_f=0.25)
        one = model(input_ids=ids, past_key_values=hf.LokiCache(P), use_cache=True).logits[:, -8:]
        c = hf.LokiCache(P)
        model(input_ids=ids[:, :64], past_key_values=c, use_cache=True)
        two = model(input_ids=ids[:, 64:], past_key_values=c, use_cache=True).logits[:, -8:]
    rel = (one.float() - two.float()).norm() / one.float().norm()
    assert rel <= 2e-2, float(rel)


@pytest.mark.gpu
def test_non_default_scale_is_rejected():
    from paper_2406_02542_b200.errors import UnsupportedShapeError

    model = _tiny_llama(2)
    ids = torch.randint(0, 256, (1, 40), device="cuda")
    with torch.no_grad():
        P = hf.calibrate(model, ids)
        hf.install(model, P)
        for m in hf._attention_modules(model):
            m.scaling = 0.5
        with pytest.raises(UnsupportedShapeError):
            model(input_ids=ids, past_key_values=hf.LokiCache(P), use_cache=True)
