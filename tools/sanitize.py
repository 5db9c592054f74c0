"""Small decode launches for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python tools/sanitize.py [--case all|split|single|gqa]

Covers the persistent pipe kernel's plans -- one launch (S < 8192), the split
A-only + B-only pair (S >= 8192, PDL-chained, ready flags), a GQA group, the
group-shared selection (entry lists, the weights finalize launch) -- with and
without diagnostics, plus K0 (append) and the dense B-only launch, at sizes the
instrumented run finishes in minutes.  Not part of the product.
"""

import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_02542_b200 as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--case", default="all")
a = ap.parse_args()

dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev).manual_seed(0)
CASES = {  # B, Hq, Hkv, S
    "single": (2, 2, 2, 4096),
    "split": (1, 2, 2, 8192),
    "gqa": (1, 8, 2, 8192),
    "shared": (2, 8, 2, 9000),  # group-shared selection (chunked A launch + entry lists)
    "ws_gqa": (37, 16, 4, 8192),  # 148 units: the warp-specialised per-head A launch (tcgen05 phase 1)
    "ws_mha": (5, 32, 32, 8192),  # 160 units: the warp-specialised MHA A launch (on-chip keys, lists)
}
for name, (B, Hq, Hkv, S) in CASES.items():
    if a.case not in ("all", name):
        continue
    K = torch.randn(B, Hkv, S, 128, device=dev, generator=gen).to(torch.bfloat16)
    V = torch.randn(B, Hkv, S, 128, device=dev, generator=gen).to(torch.bfloat16)
    q = torch.randn(B, Hq, 128, device=dev, generator=gen)
    gs = "shared" if name == "shared" else "per_head"
    y = L.loki_decode(q, K, V, None, d=32, k_f=0.25, group_select=gs)
    y2, diag = L.loki_decode(q, K, V, None, d=32, k_f=0.25, diagnostics=True, group_select=gs)
    torch.cuda.synchronize()
    assert torch.equal(y, y2), name
    rows = torch.full((B,), S - 1, dtype=torch.int32, device=dev)
    lens = torch.full((B,), S, dtype=torch.int32, device=dev)
    P = torch.linalg.qr(torch.randn(Hkv, 128, 128, device=dev, generator=gen))[0].contiguous()
    dec = L.LokiDecoder(K, V, P, Hq=Hq, d=32, k_f=0.25, rows=rows, lens=lens, q_raw=q.clone(),
                        k_raw=torch.randn(B, Hkv, 128, device=dev, generator=gen),
                        v_new=torch.randn(B, Hkv, 128, device=dev, generator=gen), rope_mode=1,
                        positions=torch.full((B,), S - 1, dtype=torch.int64, device=dev))
    dec.step()
    dec.step()
    if name in ("single", "gqa"):
        L.dense_decode(q, K, V)  # bf16: the B-only dense launch
    torch.cuda.synchronize()
    print(f"sanitize case {name}: ok (plan {dec.call.plan()})", flush=True)
