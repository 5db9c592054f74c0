"""Parity at the benchmarked configurations, through the bench's own decoders.

Each case builds bench.py's Workload for BASELINE's config (one or two layers,
same shapes, same synthetic recipe, same LokiDecoder launch plan as the timed
run: split A / B launches, the planner's chunk sizes, grid and ticket lag),
replays the serving path (DecodeGraph: K0 append + decode per layer) and checks
the result against the CPU oracle with the tie-band rule (SURVEY 8(c) O4,
oracle/loki_oracle.py:312-346):

  - the production output (no diagnostics) equals a diagnostics run on the same
    inputs bit for bit;
  - the diagnostics run's selections equal the oracle's outside the fp32 tie
    band, ascending, exactly k per (batch, query head);
  - outputs are within 1e-3 relative of the oracle on the same bf16 inputs
    (re-evaluated on the GPU's set when a tie-band swap happened).

C2 is checked on every (batch, head) unit of layer 0 (512 units, one 8192-row
A chunk each on the 3-CTA/SM A grid, B tickets lagging across many waves) and
a sample of layer 1 (the layer boundary of the graph); the other configs on a
seeded sample of 64 units.  Reference: attention.py:166-185.
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
    torch.cuda.empty_cache()


def _check_units(wl, layer, q_hat, y_prod, units):
    y_diag, diag = L.loki_decode(q_hat, wl.K[layer], wl.V[layer], wl.lens, d=wl.d, k_f=wl.cfg["k_f"],
                                 diagnostics=True, S_max=wl.S)
    torch.cuda.synchronize()
    assert torch.equal(y_diag, y_prod), "production and diagnostics launches disagree"
    qh = q_hat.cpu().numpy()
    idx = diag.indices.cpu().numpy()
    y = y_prod.cpu().numpy()
    swaps = 0
    by_unit = {}
    for b, h in units:
        by_unit.setdefault((b, h // wl.G), []).append(h)
    for (b, g), heads in by_unit.items():
        Kb = wl.K[layer][b, g].float().cpu().numpy()
        Vb = wl.V[layer][b, g].float().cpu().numpy()
        for h in heads:
            y_ref, ref_idx, _, _ = O.loki_rank_and_attend(qh[b, h], Kb, Vb, wl.d, wl.k)
            got = idx[b, h, :wl.k]
            assert got.size == wl.k and np.all(got >= 0) and np.all(np.diff(got) > 0), (b, h)
            band = O.tie_band(qh[b, h], Kb, wl.d, wl.k)
            assert O.sets_match_outside_band(got, ref_idx, band), (layer, b, h, int(band.sum()))
            if not np.array_equal(got, ref_idx):
                swaps += 1
                y_ref = O.attend_on(qh[b, h], Kb, Vb, got)[0]
            err = O.rel_err(y[b, h], y_ref)
            assert err <= 1e-3, (layer, b, h, err)
    return swaps


def _sample(B, Hq, n, seed):
    rng = np.random.default_rng(seed)
    pick = rng.choice(B * Hq, size=min(n, B * Hq), replace=False)
    return sorted((int(u) // Hq, int(u) % Hq) for u in pick)


CONFIGS = [  # name, layers, units checked on layer 0 (None = all), expected plan (split launches?)
    ("C1", 1, None, False),
    ("C2", 2, None, True),
    ("TGT", 1, 64, True),
    ("C3", 1, 64, True),
    ("C4", 1, 64, True),
    ("C5s", 1, 48, True),
]


@pytest.mark.parametrize("name,layers,n_units,split", CONFIGS, ids=[c[0] for c in CONFIGS])
def test_bench_config_parity(name, layers, n_units, split):
    import bench

    cfg = dict(bench.CONFIGS[name], layers=layers, name=name)
    wl = bench.Workload(cfg, 1, 0, seed=11)
    decs = wl.decoders()
    plan = decs[0].call.plan()
    assert (plan["ctas_per_unit"] == -2) == split, plan
    dg = L.DecodeGraph(decs)  # the serving path: one CUDA graph of LokiDecoder.step per layer
    for dec in decs:
        dec.out.zero_()
    dg.replay()
    dg.replay()  # a second replay reuses the self-reset workspace (counters, histograms, flags)
    torch.cuda.synchronize()
    units = ([(b, h) for b in range(wl.B) for h in range(wl.Hq_l)] if n_units is None
             else _sample(wl.B, wl.Hq_l, n_units, seed=len(name)))
    _check_units(wl, 0, decs[0].q_hat, decs[0].out, units)
    if layers > 1:
        _check_units(wl, layers - 1, decs[-1].q_hat, decs[-1].out, _sample(wl.B, wl.Hq_l, 32, seed=99))
    del dg, decs, wl


def test_graph_follows_growing_lens():
    """A DecodeGraph planned at the cache capacity (LokiDecoder's default S_max) stays correct while
    the serving loop advances rows / lens between replays (lens past the planned rows)."""
    B, Hq, Hkv, D, cap = 2, 4, 4, 128, 9000
    gen = torch.Generator(device="cuda").manual_seed(5)
    K = torch.randn(B, Hkv, cap, D, device="cuda", generator=gen).to(torch.bfloat16)
    V = torch.randn(B, Hkv, cap, D, device="cuda", generator=gen).to(torch.bfloat16)
    P = torch.linalg.qr(torch.randn(Hkv, D, D, device="cuda", generator=gen))[0].contiguous()
    S0 = 4000
    rows = torch.full((B,), S0, dtype=torch.int32, device="cuda")
    lens = torch.full((B,), S0 + 1, dtype=torch.int32, device="cuda")
    q_raw = torch.randn(B, Hq, D, device="cuda", generator=gen)
    k_raw = torch.randn(B, Hkv, D, device="cuda", generator=gen)
    v_new = torch.randn(B, Hkv, D, device="cuda", generator=gen)
    dec = L.LokiDecoder(K, V, P, Hq=Hq, d=32, k_f=0.25, rows=rows, lens=lens, q_raw=q_raw, k_raw=k_raw,
                        v_new=v_new)
    dg = L.DecodeGraph([dec])
    for S in (S0 + 1, 8191, 8192, 8193, cap):
        rows.fill_(S - 1)
        lens.fill_(S)
        dg.replay()
        y = dec.out.clone()
        y_ref = L.loki_decode(dec.q_hat, K, V, lens, d=32, k_f=0.25, S_max=S)
        torch.cuda.synchronize()
        assert O.rel_err(y.cpu().numpy(), y_ref.cpu().numpy()) <= 1e-5, S


def test_prefix_view_is_not_copied():
    """A [:, :, :S] view of a capacity buffer runs in place and equals the packed copy."""
    B, Hq, Hkv, D, cap, S = 2, 4, 2, 128, 6000, 4100
    gen = torch.Generator(device="cuda").manual_seed(9)
    Kb = torch.randn(B, Hkv, cap, D, device="cuda", generator=gen).to(torch.bfloat16)
    Vb = torch.randn(B, Hkv, cap, D, device="cuda", generator=gen).to(torch.bfloat16)
    q = torch.randn(B, Hq, D, device="cuda", generator=gen)
    Kv, Vv = Kb[:, :, :S], Vb[:, :, :S]
    assert L._core.row_capacity(Kv) == cap
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    before = torch.cuda.memory_allocated()
    y, diag = L.loki_decode(q, Kv, Vv, None, d=32, k_f=0.25, diagnostics=True)
    torch.cuda.synchronize()
    # no cache-sized temporary: the diagnostics and workspace are far smaller than a copy of K
    assert torch.cuda.max_memory_allocated() - before < Kv.numel() * 2
    y2, diag2 = L.loki_decode(q, Kv.contiguous(), Vv.contiguous(), None, d=32, k_f=0.25, diagnostics=True)
    assert torch.equal(diag.indices, diag2.indices)
    assert torch.equal(diag.approx_scores, diag2.approx_scores)
    assert O.rel_err(y.cpu().numpy(), y2.cpu().numpy()) <= 1e-6


def test_decode_graph_with_host_inputs_matches_manual_copies():
    """DecodeGraph(inputs=..., output=...): per-layer host->device copies on a copy stream inside the graph and
    the result copied back give the same bits as copying by hand and stepping eagerly."""
    B, Hq, Hkv, D, S, nl = 2, 8, 8, 128, 9000, 3
    gen = torch.Generator(device="cuda").manual_seed(12)
    Ks = [torch.randn(B, Hkv, S, D, device="cuda", generator=gen).to(torch.bfloat16) for _ in range(nl)]
    Vs = [torch.randn(B, Hkv, S, D, device="cuda", generator=gen).to(torch.bfloat16) for _ in range(nl)]
    Ps = [torch.linalg.qr(torch.randn(Hkv, D, D, device="cuda", generator=gen))[0].contiguous() for _ in range(nl)]
    rows = torch.full((B,), S - 1, dtype=torch.int32, device="cuda")
    lens = torch.full((B,), S, dtype=torch.int32, device="cuda")
    q = torch.zeros(nl, B, Hq, D, device="cuda")
    k = torch.zeros(nl, B, Hkv, D, device="cuda")
    v = torch.zeros(nl, B, Hkv, D, device="cuda")
    decs = [L.LokiDecoder(Ks[i], Vs[i], Ps[i], Hq=Hq, d=32, k_f=0.25, rows=rows, lens=lens, q_raw=q[i], k_raw=k[i],
                          v_new=v[i]) for i in range(nl)]
    hq = torch.randn(nl, B, Hq, D, generator=torch.Generator().manual_seed(1)).pin_memory()
    hk = torch.randn(nl, B, Hkv, D, generator=torch.Generator().manual_seed(2)).pin_memory()
    hv = torch.randn(nl, B, Hkv, D, generator=torch.Generator().manual_seed(3)).pin_memory()
    hout = torch.zeros(B, Hq, D).pin_memory()
    ins = [[(q[i], hq[i]), (k[i], hk[i]), (v[i], hv[i])] for i in range(nl)]
    dg = L.DecodeGraph(decs, inputs=ins, output=(hout, decs[-1].out))
    q.zero_(), k.zero_(), v.zero_()
    dg.replay()
    torch.cuda.synchronize()
    got = hout.clone()
    q.copy_(hq), k.copy_(hk), v.copy_(hv)
    for dec in decs:
        dec.step()
    torch.cuda.synchronize()
    assert torch.equal(got, decs[-1].out.cpu())


@pytest.mark.parametrize("B,Hq,Hkv,S,gs", [(2, 8, 8, 9000, "per_head"),    # split MHA layer (entry lists)
                                           (4, 4, 4, 4096, "per_head"),    # one launch
                                           (1, 32, 32, 4096, "per_head"),  # cluster-per-unit plan
                                           (2, 16, 4, 9000, "per_head"),   # per-head GQA (tcgen05 phase 1)
                                           (2, 16, 4, 9000, "shared")])    # group-shared selection
def test_interleaved_kv_layout_matches_separate(B, Hq, Hkv, S, gs):
    """bench --kv-layout interleaved: K and V as views of one [B, Hkv, S, 2, D] buffer (a row's K and V
    adjacent in HBM; row stride 2 D) run in place through the C-ABI's strides and give the same bits as
    separate packed caches -- selections, approx scores and outputs."""
    D = 128
    gen = torch.Generator(device="cuda").manual_seed(21)
    KV = torch.randn(B, Hkv, S, 2, D, device="cuda", generator=gen).to(torch.bfloat16)
    K, V = KV[:, :, :, 0], KV[:, :, :, 1]
    assert K.stride(2) == 2 * D
    q = torch.randn(B, Hq, D, device="cuda", generator=gen)
    y, diag = L.loki_decode(q, K, V, None, d=32, k_f=0.25, diagnostics=True, group_select=gs)
    y0 = L.loki_decode(q, K, V, None, d=32, k_f=0.25, group_select=gs)
    y2, diag2 = L.loki_decode(q, K.contiguous(), V.contiguous(), None, d=32, k_f=0.25, diagnostics=True,
                              group_select=gs)
    torch.cuda.synchronize()
    assert torch.equal(diag.indices, diag2.indices)
    assert torch.equal(diag.approx_scores, diag2.approx_scores)
    assert torch.equal(y, y2) and torch.equal(y0, y)


def test_interleaved_kv_layout_decoder_step():
    """K0 appends into the interleaved views (the new token's K and V rows land side by side) and the
    decode step that follows equals the one on separate caches bit for bit."""
    B, Hq, Hkv, D, S = 2, 8, 8, 128, 9000
    gen = torch.Generator(device="cuda").manual_seed(22)
    KV = torch.randn(B, Hkv, S, 2, D, device="cuda", generator=gen).to(torch.bfloat16)
    Ks, Vs = KV[:, :, :, 0].contiguous(), KV[:, :, :, 1].contiguous()
    P = torch.linalg.qr(torch.randn(Hkv, D, D, device="cuda", generator=gen))[0].contiguous()
    rows = torch.full((B,), S - 1, dtype=torch.int32, device="cuda")
    lens = torch.full((B,), S, dtype=torch.int32, device="cuda")
    q = torch.randn(B, Hq, D, device="cuda", generator=gen)
    k = torch.randn(B, Hkv, D, device="cuda", generator=gen)
    v = torch.randn(B, Hkv, D, device="cuda", generator=gen)
    pos = torch.full((B,), S - 1, dtype=torch.int64, device="cuda")
    outs = []
    for K, V in ((KV[:, :, :, 0], KV[:, :, :, 1]), (Ks, Vs)):
        dec = L.LokiDecoder(K, V, P, Hq=Hq, d=32, k_f=0.25, rows=rows, lens=lens, q_raw=q.clone(), k_raw=k.clone(),
                            v_new=v.clone(), rope_mode=1, positions=pos)
        dec.step()
        torch.cuda.synchronize()
        outs.append((dec.out.clone(), K[:, :, S - 1].clone(), V[:, :, S - 1].clone()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)
