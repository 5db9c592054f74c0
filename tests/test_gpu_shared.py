"""Group-shared selection (opt-in GQA mode, LOKI_SELECT_TOPK_SHARED) against its oracle.

The oracle (oracle/loki_oracle.py loki_rank_and_attend_shared) composes the
reference's own primitives -- sliced_score_kernel on the [G, D] query block
(kernels.py:223-241), summed over the group, topk_indices (linalg.py:95-118),
then the per-head exact path (attention.py:180-184) -- and is pinned to
reference outputs of that composition (tests/test_oracle.py).  Here the CUDA
path (through the C ABI) must match it: one selection per (b, KV head),
identical outside the fp32 tie band of the group score, every query head of the
group reporting it; outputs within 1e-3 of the oracle on the same bf16 inputs.
"""

import numpy as np
import pytest
import torch

from oracle import loki_oracle as O

pytestmark = pytest.mark.gpu

L = pytest.importorskip("paper_2406_02542_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    yield


def _inputs(B, Hq, Hkv, S, seed, correlated=True):
    rng = np.random.default_rng(seed)
    D = 128
    keys = O.gen_synthetic_keys(S + 512, D, 16, 1e-3, seed + 1)
    P, _ = O.build_projection(keys[:512])
    K = np.stack([np.stack([O.round_bf16((keys[512:] * (1 + 0.05 * (b + h))) @ P) for h in range(Hkv)])
                  for b in range(B)])
    V = O.round_bf16(rng.standard_normal((B, Hkv, S, D)).astype(np.float32))
    G = Hq // Hkv
    if correlated:  # q_g = q_0 + 0.5 eps_g
        q0 = rng.standard_normal((B, Hkv, 1, D))
        q = (q0 + 0.5 * rng.standard_normal((B, Hkv, G, D))).reshape(B, Hq, D).astype(np.float32)
    else:
        q = rng.standard_normal((B, Hq, D)).astype(np.float32)
    return q, K, V


def _check(q, K, V, lens, d, k_f, y, diag, y_prod):
    B, Hq, D = q.shape
    Hkv = K.shape[1]
    G = Hq // Hkv
    idx = diag.indices.cpu().numpy()
    approx = diag.approx_scores.cpu().numpy()
    w = diag.weights.cpu().numpy()
    y = y.cpu().numpy()
    assert np.array_equal(y, y_prod.cpu().numpy()), "production and diagnostics launches disagree"
    swaps = 0
    for b in range(B):
        S = int(lens[b])
        k = O.resolve_fraction(k_f, S)
        for g in range(Hkv):
            Qb, Kb, Vb = q[b, g * G:(g + 1) * G], K[b, g, :S], V[b, g, :S]
            y_ref, ref_idx, grp, w_ref = O.loki_rank_and_attend_shared(Qb, Kb, Vb, d, k)
            got = idx[b, g * G, :k]
            for h in range(1, G):  # one selection per group
                assert np.array_equal(idx[b, g * G + h, :k], got), (b, g, h)
            assert np.all(idx[b, g * G:(g + 1) * G, k:] == -1)
            assert np.all(np.diff(got) > 0)
            band = O.tie_band_shared(Qb, Kb, d, k)
            assert O.sets_match_outside_band(got, ref_idx, band), (b, g, int(band.sum()))
            if not np.array_equal(got, ref_idx):
                swaps += 1
                outs = [O.attend_on(Qb[h], Kb, Vb, got) for h in range(G)]
                y_ref = np.stack([o[0] for o in outs])
                w_ref = np.stack([o[1] for o in outs])
            assert O.rel_err(y[b, g * G:(g + 1) * G], y_ref) <= 1e-3, (b, g)
            assert np.abs(w[b, g * G:(g + 1) * G, :k] - w_ref).max() <= 1e-4, (b, g)
            for h in range(G):  # every head reports the group score
                assert O.rel_err(approx[b, g * G + h, :S], grp) <= 1e-5, (b, g, h)
    return swaps


CASES = [  # B, Hq, Hkv, S, lens (None = S), d
    (2, 8, 2, 4096, None, 32),          # single-chunk units: on-chip selection, ordered entry lists
    (2, 8, 2, 8192, [8192, 5000], 32),  # ragged
    (1, 16, 2, 32768, None, 32),        # G = 8, long units: keys streamed back from L2
    (2, 8, 2, 16384, [16384, 9001], 64),  # d = 64 (128 B lead rows)
    (3, 4, 2, 20000, [20000, 12345, 7], 32),  # G = 2, a 7-row unit
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"B{c[0]}_Hq{c[1]}_Hkv{c[2]}_S{c[3]}_d{c[5]}")
def test_shared_selection_matches_oracle(case):
    B, Hq, Hkv, S, lens, d = case
    lens = [S] * B if lens is None else lens
    q, K, V = _inputs(B, Hq, Hkv, S, seed=S + Hq)
    dev = "cuda"
    qt = torch.from_numpy(q).to(dev)
    Kt = torch.from_numpy(K).to(dev, torch.bfloat16)
    Vt = torch.from_numpy(V).to(dev, torch.bfloat16)
    lt = torch.tensor(lens, dtype=torch.int32, device=dev)
    y, diag = L.loki_decode(qt, Kt, Vt, lt, d=d, k_f=0.25, diagnostics=True, group_select="shared")
    y_prod = L.loki_decode(qt, Kt, Vt, lt, d=d, k_f=0.25, group_select="shared")
    torch.cuda.synchronize()
    _check(q, K, V, lens, d, 0.25, y, diag, y_prod)


def test_shared_equals_per_head_for_mha():
    """With one query head per KV head the two modes are the same computation (bit for bit)."""
    q, K, V = _inputs(2, 4, 4, 8192, seed=3, correlated=False)
    qt = torch.from_numpy(q).cuda()
    Kt = torch.from_numpy(K).cuda().to(torch.bfloat16)
    Vt = torch.from_numpy(V).cuda().to(torch.bfloat16)
    a = L.loki_decode(qt, Kt, Vt, None, d=32, k_f=0.25)
    b = L.loki_decode(qt, Kt, Vt, None, d=32, k_f=0.25, group_select="shared")
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_shared_decoder_graph_replays():
    """LokiDecoder(group_select="shared") under DecodeGraph: K0 append + the shared launch pair, replayed."""
    B, Hq, Hkv, D, S = 2, 8, 2, 128, 9000
    gen = torch.Generator(device="cuda").manual_seed(4)
    K = torch.randn(B, Hkv, S, D, device="cuda", generator=gen).to(torch.bfloat16)
    V = torch.randn(B, Hkv, S, D, device="cuda", generator=gen).to(torch.bfloat16)
    P = torch.linalg.qr(torch.randn(Hkv, D, D, device="cuda", generator=gen))[0].contiguous()
    rows = torch.full((B,), S - 1, dtype=torch.int32, device="cuda")
    lens = torch.full((B,), S, dtype=torch.int32, device="cuda")
    dec = L.LokiDecoder(K, V, P, Hq=Hq, d=32, k_f=0.25, rows=rows, lens=lens,
                        q_raw=torch.randn(B, Hq, D, device="cuda", generator=gen),
                        k_raw=torch.randn(B, Hkv, D, device="cuda", generator=gen),
                        v_new=torch.randn(B, Hkv, D, device="cuda", generator=gen), group_select="shared")
    dg = L.DecodeGraph([dec])
    dg.replay()
    y = dec.out.clone()
    y_ref = L.loki_decode(dec.q_hat, K, V, lens, d=32, k_f=0.25, group_select="shared")
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref)


def test_shared_rejects_fp32_caches():
    q = torch.randn(1, 4, 128, device="cuda")
    K = torch.randn(1, 2, 4096, 128, device="cuda")
    with pytest.raises(L.UnsupportedShapeError):
        L.loki_decode(q, K, K.clone(), None, d=32, k_f=0.25, group_select="shared")
