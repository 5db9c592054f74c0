"""One-layer timing / profiling driver (not part of the product).

    python tools/one_layer.py [--B 16] [--H 32] [--Hkv 32] [--S 8192] [--mode loki|dense] [--reps 20]

Builds a random bf16 cache, runs loki_decode (or dense) through the public
batched API and prints per-launch CUDA-event time and achieved algorithmic GB/s.
Env LOKI_TMA / LOKI_TMA_STAGES / LOKI_CLUSTER steer the launch plan.
"""

import argparse
import os
import sys

import torch

os.environ.setdefault("LOKI_TUNING", "1")  # honour LOKI_* tuning knobs (ignored by the library otherwise)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_02542_b200 as L  # noqa: E402
from paper_2406_02542_b200 import _core, _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=16)
ap.add_argument("--H", type=int, default=32)
ap.add_argument("--Hkv", type=int, default=32)
ap.add_argument("--S", type=int, default=8192)
ap.add_argument("--D", type=int, default=128)
ap.add_argument("--kf", type=float, default=0.25)
ap.add_argument("--df", type=float, default=0.25)
ap.add_argument("--mode", default="loki")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--cluster", type=int, default=0)
a = ap.parse_args()

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
K = torch.randn(a.B, a.Hkv, a.S, a.D, device=dev, generator=g).to(torch.bfloat16)
V = torch.randn(a.B, a.Hkv, a.S, a.D, device=dev, generator=g).to(torch.bfloat16)
q = torch.randn(a.B, a.H, a.D, device=dev, generator=g)
out = torch.empty(a.B, a.H, a.D, device=dev)
lens = torch.full((a.B,), a.S, dtype=torch.int32, device=dev)
d = max(1, min(a.D, int(a.df * a.D + 0.5)))
k = max(1, min(a.S, int(a.kf * a.S + 0.5)))
if a.mode == "dense":
    call = _core.DecodeCall(q, K, V, lens, a.S, a.D, select_mode=_lib.SELECT_ALL, out=out, cluster=a.cluster)
    nbytes = a.B * a.Hkv * a.S * a.D * 2 * 2
else:
    call = _core.DecodeCall(q, K, V, lens, a.S, d, k_fixed=k, out=out, cluster=a.cluster)
    nbytes = a.B * a.Hkv * 2 * (d * a.S + 2 * a.D * k)
print("plan", call.plan(), "TMA", os.environ.get("LOKI_TMA", "1"))
for _ in range(3):
    call.run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    call.run()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1000 / a.reps
print(f"{a.mode}: {us:.1f} us/launch, {nbytes / us / 1e3:.1f} GB/s algorithmic")

if os.environ.get("LOKI_TRACE") and call.plan()["ctas_per_unit"] <= 0:
    # persistent pipe kernel: per-ticket {start, end, smid | kind << 16 | block << 32}
    import numpy as np

    nbuf = 1 << 23
    buf = torch.zeros(nbuf, dtype=torch.int64, device=dev)
    lib = _lib.load()
    _lib.check(lib.loki_set_phase_trace(buf.data_ptr(), nbuf // 8))
    call.run()
    torch.cuda.synchronize()
    _lib.check(lib.loki_set_phase_trace(None, 0))
    t = buf.view(-1, 4).cpu().numpy()
    t = t[t[:, 0] != 0]
    kind = (t[:, 2] >> 16) & 0xFFFF
    t0 = t[:, 0].min()
    st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
    dur = en - st
    print(f"pipe: {len(t)} tickets, span {en.max():.1f} us, blocks {len(np.unique(t[:, 2] >> 32))}")
    for kd, nm in ((1, "A"), (3, "A+select"), (2, "B"), (4, "B+merge"), (0, "noop")):
        m = kind == kd
        if m.any():
            print(f"  {nm:9s} n={m.sum():5d} median {np.median(dur[m]):7.2f} us  mean {dur[m].mean():7.2f}  max {dur[m].max():7.2f}  busy-share {dur[m].sum() / dur.sum() * 100:5.1f}%")
    bm = (kind == 2) & (t[:, 3] != 0)
    if bm.any():
        wait = (t[bm, 3] - t[bm, 0]) / 1e3
        print(f"  B wait-for-ready: median {np.median(wait):6.2f} us  mean {wait.mean():6.2f}  max {wait.max():6.2f}")
    lastm = (t[:, 3] != 0) & (kind >= 3)
    tail = (t[lastm, 1] - t[lastm, 3]) / 1e3
    for kd, nm in ((3, "select"), (4, "merge")):
        m = kind[lastm] == kd
        if m.any():
            print(f"  {nm:9s} part: median {np.median(tail[m]):7.2f} us  mean {tail[m].mean():7.2f}  max {tail[m].max():7.2f}")
    ab = np.array([1 if k in (1, 3) else 0 for k in kind])
    bb_ = np.array([1 if k in (2, 4) else 0 for k in kind])
    grid = np.linspace(0, en.max(), 40)
    occA = [((st <= x) & (en > x) & (ab == 1)).sum() for x in grid]
    occB = [((st <= x) & (en > x) & (bb_ == 1)).sum() for x in grid]
    print("  CTAs in A / B over time:", " ".join(f"{a}/{b}" for a, b in zip(occA, occB)))
    if int(os.environ.get("LOKI_DEBUG", "0")) & 16:
        st8 = buf.view(-1).cpu().numpy()[1 << 21:(1 << 21) + a.B * a.Hkv * 8].reshape(-1, 8)
        ok = st8[:, 0] != 0
        st8 = st8[ok]
        names = ["find_bin", "compaction", "narrow+rank", "other heads", "emit/offsets", "fence+release"]
        for i, nm in enumerate(names):
            dd = (st8[:, i + 1] - st8[:, i]) / 1e3
            print(f"    sel {nm:14s} median {np.median(dd):6.2f} us  max {dd.max():6.2f}")
        print(f"    sel ncand median {np.median(st8[:, 7]):.0f} max {st8[:, 7].max()}")
    blk = t[:, 2] >> 32
    idle = []
    for bb in np.unique(blk):
        mm = blk == bb
        idle.append(en[mm].max() - dur[mm].sum())
    print(f"  per-CTA idle (span - busy): median {np.median(idle):.1f} us; last CTA end - first CTA end {en.max() - np.min([en[blk == bb].max() for bb in np.unique(blk)]):.1f} us")
elif os.environ.get("LOKI_TRACE"):
    import numpy as np

    plan = call.plan()
    ctas = a.B * a.Hkv * plan["ctas_per_unit"]
    buf = torch.zeros(ctas * 8, dtype=torch.int64, device=dev)
    lib = _lib.load()
    _lib.check(lib.loki_set_phase_trace(buf.data_ptr(), ctas))
    call.run()
    torch.cuda.synchronize()
    _lib.check(lib.loki_set_phase_trace(None, 0))
    t = buf.view(ctas, 8).cpu().numpy().astype(np.float64)
    for i in range(1, 8):  # steps a path skipped keep the previous stamp
        t[:, i] = np.where(t[:, i] == 0, t[:, i - 1], t[:, i])
    t0 = t[:, 0].min()
    t = (t - t0) / 1000.0  # us
    dur = np.diff(t, axis=1)
    names = ["phase1", "radix", "counts", "emit", "union", "phase3", "merge"]
    print(f"kernel span {t[:, 7].max():.1f} us; CTA start spread {t[:, 0].max():.1f} us")
    for i, n in enumerate(names):
        print(f"  {n:7s} median {np.median(dur[:, i]):7.2f} us  mean {dur[:, i].mean():7.2f}  max {dur[:, i].max():7.2f}"
              f"  sum-share {dur[:, i].sum() / dur.sum() * 100:5.1f}%")
