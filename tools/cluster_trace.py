"""Per-phase stamps of the cluster-per-unit plan (tuning tool, not product):
    python tools/cluster_trace.py [--B 1] [--S 4096]
Stamps per CTA (loki_set_phase_trace): start, phase 1 done, radix passes, tie counts, selection emitted,
union built, phase 3 done, end."""
import argparse, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_02542_b200 as L  # noqa: E402
from paper_2406_02542_b200 import _core, _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=1)
ap.add_argument("--H", type=int, default=32)
ap.add_argument("--S", type=int, default=4096)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
K = torch.randn(a.B, a.H, a.S, 128, device=dev, generator=g).to(torch.bfloat16)
V = torch.randn(a.B, a.H, a.S, 128, device=dev, generator=g).to(torch.bfloat16)
q = torch.randn(a.B, a.H, 128, device=dev, generator=g)
out = torch.empty(a.B, a.H, 128, device=dev)
lens = torch.full((a.B,), a.S, dtype=torch.int32, device=dev)
call = _core.DecodeCall(q, K, V, lens, a.S, 32, k_f=0.25, out=out)
print("plan", call.plan())
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
tot = 0.0
for i in range(a.reps + 3):
    flush.zero_()
    e0.record(); call.run(); e1.record(); torch.cuda.synchronize()
    if i >= 3:
        tot += e0.elapsed_time(e1) * 1000
print(f"L2-cold launch: {tot / a.reps:.2f} us")
lib = _lib.load()
nct = 4096
buf = torch.zeros(nct * 8, dtype=torch.int64, device=dev)
_lib.check(lib.loki_set_phase_trace(buf.data_ptr(), nct))
flush.zero_(); torch.cuda.synchronize()
call.run(); torch.cuda.synchronize()
_lib.check(lib.loki_set_phase_trace(None, 0))
t = buf.view(nct, 8).cpu()
t = t[t[:, 0] != 0].double()
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
names = ["start", "phase1", "radix", "ties", "emitted", "union", "phase3", "end"]
print("CTAs", len(t))
for i, nm in enumerate(names):
    col = rel[:, i]
    col = col[col >= 0]
    print(f"  {nm:8s} median {col.median():7.2f} us  max {col.max():7.2f}")
