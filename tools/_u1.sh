cat > /tmp/ucheck.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2406_02542_b200 as L
B, Hq, Hkv, S = 40, 16, 4, 8192   # 160 units (>= 148): the warp-specialised per-head A launch
g = torch.Generator(device="cuda").manual_seed(3)
K = torch.randn(B, Hkv, S, 128, device="cuda", generator=g).to(torch.bfloat16)
V = torch.randn(B, Hkv, S, 128, device="cuda", generator=g).to(torch.bfloat16)
q = torch.randn(B, Hq, 128, device="cuda", generator=g)
for d in (32, 64):
    y, diag = L.loki_decode(q, K, V, None, d=d, k_f=0.25, diagnostics=True)
    torch.cuda.synchronize()
    torch.save((y.cpu(), diag.indices.cpu()), f"/tmp/u_{os.environ.get('LOKI_UMMA')}_{d}.pt")
    print("d", d, "ok", float(y.abs().max()), int((diag.indices >= 0).sum()))
PY
for um in 0 1; do echo "== LOKI_UMMA=$um"; LOKI_TUNING=1 LOKI_UMMA=$um timeout 120 python /tmp/ucheck.py 2>&1 | tail -4; done
python - <<'PY'
import torch
for d in (32, 64):
    y0, i0 = torch.load(f"/tmp/u_0_{d}.pt"); y1, i1 = torch.load(f"/tmp/u_1_{d}.pt")
    same = (i0 == i1).all(dim=-1).float().mean().item()
    print("d", d, "index rows identical", same, "max |dy|", float((y0 - y1).abs().max()))
PY
timeout 900 python -m pytest tests/test_bench_parity.py tests/test_gpu_parity.py tests/test_gpu_shared.py -m gpu -q --tb=short -x 2>&1 | tail -4
for c in C3 C4; do for um in 0 1; do echo "== $c umma $um"; LOKI_TUNING=1 LOKI_UMMA=$um timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['loki_attention_us_per_layer'], d['parity']['pass'], d['parity']['max_rel_err'], d['phases'].get('approx_scores_topk_us'))"; done; done
