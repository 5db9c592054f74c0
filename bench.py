#!/usr/bin/env python
"""Loki decode-attention benchmark (BASELINE.json metric:
"Loki decode-attn us/layer & speedup vs full attn; achieved HBM GB/s").

Workload (default, BASELINE configs[1] = SURVEY C2): Llama2-7B-shaped decode
attention for all 32 layers, batch 16, 32 heads, D = 128, S = 8192 cached
tokens, k_f = d_f = 0.25, pre-rotary PCA per (layer, KV head), bf16 caches.
One step = for every layer: K0 (RoPE -> P -> append the new token) + the fused
Loki decode kernel; the layer loop is captured in one CUDA graph.  Reported
`value` is us per layer (lower is better), max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2]
  python bench.py --impl reference ...   # the reference's CPU path (oracle port)

N > 1 (torchrun): KV heads are sharded across ranks (strong scaling); after
each layer the per-rank outputs are all-gathered with NCCL.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Loki decode-attn µs/layer & speedup vs full attn; achieved HBM GB/s"

CONFIGS = {
    # name: layers, B, Hq, Hkv, D, S, k_f, d_f, rope base, description
    "C1": dict(layers=1, B=1, Hq=32, Hkv=32, D=128, S=4096, k_f=0.25, d_f=0.25, base=10000.0,
               desc="single Llama2-7B-shaped layer, B=1, S=4096"),
    "C2": dict(layers=32, B=16, Hq=32, Hkv=32, D=128, S=8192, k_f=0.25, d_f=0.25, base=10000.0,
               desc="Llama2-7B-shaped 32-layer decode attention, B=16, S=8192, pre-rotary PCA"),
    "C3": dict(layers=4, B=32, Hq=32, Hkv=8, D=128, S=32768, k_f=0.125, d_f=0.5, base=500000.0,
               desc="Llama3-8B GQA (8 KV heads) decode attention, B=32, S=32K, 4 of 32 layers"),
    "C4": dict(layers=4, B=64, Hq=32, Hkv=8, D=128, S=16384, k_f=0.25, d_f=0.25, base=10000.0,
               desc="Mistral-7B GQA decode attention, B=64, S=16K, 4 of 32 layers"),
    "TGT": dict(layers=4, B=16, Hq=32, Hkv=32, D=128, S=32768, k_f=0.25, d_f=0.25, base=10000.0,
                desc="north-star target: MHA 32 heads, B=16, S=32K, 4 layers"),
    # C5 is sharded by KV head over 8 GPUs: one GPU's shard = 1 KV head with its 8 query heads
    "C5s": dict(layers=2, B=128, Hq=8, Hkv=1, D=128, S=131072, k_f=0.25, d_f=0.25, base=500000.0,
                desc="Llama3-70B-shaped decode attention, one GPU's shard of 8 (1 KV head, 8 q heads), "
                     "B=128, S=128K, 2 layers"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------- distributed

def dist_setup():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi sampled DURING the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,utilization.gpu,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons, loaded = [], None, set(), 0
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 10:
                continue
            try:
                clk, mx, util = float(parts[1]), float(parts[2]), float(parts[4])
            except ValueError:
                continue
            smax = mx
            if util <= 0:
                continue
            loaded += 1
            sm.append(clk)
            for nm, v in zip(names, parts[6:10]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": loaded}


# ----------------------------------------------------------------------------- workload

class Workload:
    """Synthetic caches + projections + per-step inputs, resident in HBM."""

    def __init__(self, cfg, world, rank, seed=0):
        import torch

        self.cfg = cfg
        self.world, self.rank = world, rank
        L, B, Hq, Hkv, D, S = (cfg[k] for k in ("layers", "B", "Hq", "Hkv", "D", "S"))
        from paper_2406_02542_b200 import sharding

        try:
            self.shard = sharding.head_shard(Hq, Hkv, world, rank)
        except Exception as e:  # uneven split: the config cannot run at this world size
            raise SystemExit(str(e))
        self.Hkv_l = self.shard.kv_heads
        self.Hq_l = self.shard.q_heads
        self.G = Hq // Hkv
        self.L, self.B, self.D, self.S = L, B, D, S
        self.d = max(1, min(D, math.floor(cfg["d_f"] * D + 0.5)))
        self.k = max(1, min(S, math.floor(cfg["k_f"] * S + 0.5)))
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        gen = torch.Generator(device=dev)
        gen.manual_seed(1000 * seed + 7 + rank)
        rank_r, sigma, S_cal = 16, 1e-3, 8192
        half = D // 2
        inv = torch.from_numpy(cfg["base"] ** (-np.arange(half, dtype=np.float64) * 2.0 / D)).to(dev)
        pos = torch.arange(S, device=dev, dtype=torch.float64)
        ang = pos[:, None] * inv[None, :]
        cos, sin = torch.cos(ang).float(), torch.sin(ang).float()
        self.K, self.V, self.P = [], [], []
        t0 = time.time()
        for layer in range(L):
            # planted rank-16 pre-rotary keys per KV head, PCA on calibration rows
            basis = torch.linalg.qr(torch.randn(self.Hkv_l, D, rank_r, device=dev, generator=gen))[0]
            zc = torch.randn(self.Hkv_l, S_cal, rank_r, device=dev, generator=gen)
            cal = zc @ basis.transpose(1, 2) + sigma * torch.randn(self.Hkv_l, S_cal, D, device=dev, generator=gen)
            cal = cal.double()
            cal = cal - cal.mean(dim=1, keepdim=True)
            cov = cal.transpose(1, 2) @ cal / (S_cal - 1)
            vals, vecs = torch.linalg.eigh((cov + cov.transpose(1, 2)) * 0.5)
            vecs = vecs.flip(-1)
            pick = vecs.abs().argmax(dim=1, keepdim=True)
            vecs = vecs * torch.sign(torch.gather(vecs, 1, pick))
            P = vecs.float().contiguous()  # [Hkv_l, D, D], columns = principal directions
            Kl = torch.empty(B, self.Hkv_l, S, D, device=dev, dtype=torch.bfloat16)
            Vl = torch.randn(B, self.Hkv_l, S, D, device=dev, generator=gen).to(torch.bfloat16)
            for h in range(self.Hkv_l):
                z = torch.randn(B, S, rank_r, device=dev, generator=gen)
                kp = z @ basis[h].T + sigma * torch.randn(B, S, D, device=dev, generator=gen)
                lo, hi = kp[..., :half], kp[..., half:]
                kr = torch.cat([lo * cos - hi * sin, lo * sin + hi * cos], dim=-1)
                Kl[:, h] = (kr @ P[h]).to(torch.bfloat16)
                del z, kp, lo, hi, kr
            self.K.append(Kl)
            self.V.append(Vl)
            self.P.append(P)
        torch.cuda.synchronize()
        log(f"[bench] rank {rank}: built {L} layers of KV cache "
            f"({2 * L * B * self.Hkv_l * S * D * 2 / 1e9:.1f} GB bf16) in {time.time() - t0:.1f}s")
        if cfg.get("gqa_queries") == "correlated" and self.G > 1:
            # group-correlated queries q_g = q_0 + 0.5 eps_g
            q0 = torch.randn(L, B, self.Hkv_l, 1, D, device=dev, generator=gen)
            eps = torch.randn(L, B, self.Hkv_l, self.G, D, device=dev, generator=gen)
            self.q_raw = (q0 + 0.5 * eps).reshape(L, B, self.Hq_l, D).contiguous()
        else:
            self.q_raw = torch.randn(L, B, self.Hq_l, D, device=dev, generator=gen)
        self.k_raw = torch.randn(L, B, self.Hkv_l, D, device=dev, generator=gen)
        self.v_new = torch.randn(L, B, self.Hkv_l, D, device=dev, generator=gen)
        self.rows = torch.full((B,), S - 1, dtype=torch.int32, device=dev)
        self.lens = torch.full((B,), S, dtype=torch.int32, device=dev)
        self.positions = torch.full((B,), S - 1, dtype=torch.int64, device=dev)
        self.out = torch.empty(L, B, self.Hq_l, D, device=dev)
        self.gathered = torch.empty(L, world * B, self.Hq_l, D, device=dev) if world > 1 else None
        self.full_out = torch.empty(L, B, Hq, D, device=dev) if world > 1 else None

    def decoders(self, dense=False):
        from paper_2406_02542_b200 import LokiDecoder, _lib

        decs = []
        for layer in range(self.L):
            decs.append(LokiDecoder(
                self.K[layer], self.V[layer], None if dense else self.P[layer], Hq=self.Hq_l, d=self.d,
                k_f=self.cfg["k_f"], rows=self.rows, lens=self.lens, S_max=self.S, q_raw=self.q_raw[layer],
                k_raw=self.k_raw[layer], v_new=self.v_new[layer], rope_mode=_lib.ROPE_ROTATE_THEN_PROJECT,
                rope_base=self.cfg["base"], positions=self.positions, dense=dense, out=self.out[layer]))
        return decs


def gather_outputs(wl, layer, stream_ctx=None):
    """The one exchange step of a head-sharded layer: NCCL all-gather of the
    per-rank [B, Hq/world, D] outputs into [B, Hq, D] for the next layer."""
    from paper_2406_02542_b200 import sharding

    sharding.gather_heads(wl.out[layer], wl.world, out=wl.full_out[layer], staging=wl.gathered[layer])


def make_step(wl, decs, world, attend_only=False):
    import torch

    def step():
        s = torch.cuda.current_stream().cuda_stream
        for layer, dec in enumerate(decs):
            if not attend_only:
                dec.append(s)
            dec.attend(s)
            if world > 1 and not attend_only:
                gather_outputs(wl, layer)
    return step


def capture(fn, warm=2):
    """CUDA-graph the step (falls back to eager if capture is not possible)."""
    import torch

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(warm):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        torch.cuda.synchronize()
        return g.replay, "cuda-graph"
    except Exception as e:  # pragma: no cover - depends on driver / NCCL build
        log(f"[bench] graph capture failed ({e}); timing eager launches")
        torch.cuda.synchronize()
        return fn, "eager"


def time_region(fn, steps, world):
    """Barrier + sync on both sides, CUDA events on the launching stream; ms total (max over ranks)."""
    import torch

    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    barrier(world)
    return max_over_ranks(e0.elapsed_time(e1), world)


# ----------------------------------------------------------------------------- comparators

def sdpa_dense_us(wl, reps):
    """torch SDPA (cuDNN / flash backends) dense decode over the same caches -- library comparator."""
    import torch
    import torch.nn.functional as F

    q = torch.randn(wl.B, wl.Hq_l, 1, wl.D, device=wl.dev, dtype=torch.bfloat16)

    def fn():
        for layer in range(wl.L):
            F.scaled_dot_product_attention(q, wl.K[layer], wl.V[layer], enable_gqa=wl.G > 1)
    try:
        fn()
        torch.cuda.synchronize()
        ms = time_region(fn, reps, 1)
        return ms * 1000.0 / (reps * wl.L)
    except Exception as e:  # pragma: no cover
        log(f"[bench] sdpa comparator failed: {e}")
        return None


def flashinfer_dense_us(wl, reps):
    """flashinfer batch decode (paged HND, one page per sequence) -- library comparator."""
    import torch

    try:
        import flashinfer

        ws = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=wl.dev)
        w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, kv_layout="HND")
        B = wl.B
        indptr = torch.arange(B + 1, dtype=torch.int32, device=wl.dev)
        indices = torch.arange(B, dtype=torch.int32, device=wl.dev)
        last = torch.full((B,), wl.S, dtype=torch.int32, device=wl.dev)
        w.plan(indptr, indices, last, wl.Hq_l, wl.Hkv_l, wl.D, wl.S, q_data_type=torch.bfloat16,
               kv_data_type=torch.bfloat16)
        q = torch.randn(B, wl.Hq_l, wl.D, device=wl.dev, dtype=torch.bfloat16)

        def fn():
            for layer in range(wl.L):
                w.run(q, (wl.K[layer], wl.V[layer]))
        fn()
        torch.cuda.synchronize()
        ms = time_region(fn, reps, 1)
        return ms * 1000.0 / (reps * wl.L)
    except Exception as e:  # pragma: no cover
        log(f"[bench] flashinfer comparator unavailable: {e}")
        return None


# ----------------------------------------------------------------------------- CPU baseline

_CPU = {}


def _cpu_worker(units):
    from threadpoolctl import threadpool_limits

    from oracle import loki_oracle as O

    q, K, V, d, k = _CPU["q"], _CPU["K"], _CPU["V"], _CPU["d"], _CPU["k"]
    with threadpool_limits(1):
        t0 = time.perf_counter()
        for u in units:
            O.loki_unit_cpu(q[u], K[u], V[u], d, k)
        return time.perf_counter() - t0


def cpu_sample_from_device(wl, n_units):
    """Copy a seeded sample of (b, head) units of layer 0 (bf16 -> fp32) to the host."""
    import torch

    rng = np.random.default_rng(123)
    units = rng.choice(wl.B * wl.Hq_l, size=min(n_units, wl.B * wl.Hq_l), replace=False)
    qs, Ks, Vs = [], [], []
    q_hat = wl.decs_q_hat  # [B, Hq_l, D] after a step of layer 0
    for u in units:
        b, h = divmod(int(u), wl.Hq_l)
        g = h // wl.G
        qs.append(q_hat[b, h].cpu().numpy())
        Ks.append(wl.K[0][b, g].float().cpu().numpy())
        Vs.append(wl.V[0][b, g].float().cpu().numpy())
    return np.stack(qs), np.stack(Ks), np.stack(Vs)


def cpu_sample_host(cfg, n_units, seed=5):
    """Host-generated sample of the same workload (reference arm: no GPU needed)."""
    from oracle import loki_oracle as O

    D, S = cfg["D"], cfg["S"]
    rng = np.random.default_rng(seed)
    keys = O.gen_synthetic_keys(S + 2048, D, 16, 1e-3, seed)
    P, _ = O.build_projection(keys[:2048])
    Kr = O.rope_apply_rows(keys[2048:], D, cfg["base"]).astype(np.float32)
    Kh = (Kr @ P).astype(np.float32)
    Ks = np.stack([Kh[rng.permutation(S)] for _ in range(n_units)])
    Vs = rng.standard_normal((n_units, S, D)).astype(np.float32)
    qs = rng.standard_normal((n_units, D)).astype(np.float32)
    return qs, Ks, Vs


def cpu_baseline(q, K, V, d, k, units_per_layer, trials=3):
    """Reference CPU path (oracle port of attention.py:166-185 with the O(S)
    selection) over the sample, one forked worker per core, thread pools 1.
    Returns (us per layer extrapolated, cores, wall seconds per trial)."""
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    n = q.shape[0]
    _CPU.update(q=q, K=K, V=V, d=d, k=k)
    chunks = [list(range(i, n, cores)) for i in range(min(cores, n))]
    ctx = mp.get_context("fork")
    walls = []
    with ctx.Pool(len(chunks)) as pool:
        pool.map(_cpu_worker, [c[:1] for c in chunks])  # warm: imports, page-in
        for _ in range(trials):
            t0 = time.perf_counter()
            pool.map(_cpu_worker, chunks)
            walls.append(time.perf_counter() - t0)
    wall = statistics.median(walls)
    return wall * 1e6 * units_per_layer / n, len(chunks), wall


# ----------------------------------------------------------------------------- reference arm

def run_reference(args, cfg, world, rank):
    if rank != 0:
        return
    d = max(1, min(cfg["D"], math.floor(cfg["d_f"] * cfg["D"] + 0.5)))
    k = max(1, min(cfg["S"], math.floor(cfg["k_f"] * cfg["S"] + 0.5)))
    units_per_layer = cfg["B"] * cfg["Hq"]
    n = min(args.cpu_units, units_per_layer)
    q, K, V = cpu_sample_host(cfg, n)
    per_step = []
    for i in range(args.warmup + args.steps):
        us, cores, wall = cpu_baseline(q, K, V, d, k, units_per_layer, trials=1)
        if i >= args.warmup:
            per_step.append(us)
    value = statistics.median(per_step)
    sample = f"{n} of {units_per_layer} (batch, head) units of one layer per step, extrapolated linearly"
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "µs/layer",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(value * cfg["layers"] / 1000.0, 3), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_block(cfg, args, world, d, k),
        "cpu_baseline": {"value": round(value, 3), "unit": "µs/layer", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "µs/layer", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def union_rows(wl, dec):
    """Mean |union over the query group of the selected rows| per (b, kv head) unit of one layer."""
    import torch

    import paper_2406_02542_b200 as L

    _, diag = L.loki_decode(dec.q_hat, wl.K[0], wl.V[0], wl.lens, d=wl.d, k=wl.k, diagnostics=True)
    idx = diag.indices.view(wl.B, wl.Hkv_l, wl.G * wl.k)
    sizes = [torch.unique(idx[b, h]).numel() for b in range(wl.B) for h in range(wl.Hkv_l)]
    return float(sum(sizes)) / len(sizes)


def config_block(cfg, args, world, d, k):
    return {"workload": f"{args.config}: {cfg['desc']}", "layers": cfg["layers"], "global_batch": cfg["B"],
            "seq_len": cfg["S"], "q_heads": cfg["Hq"], "kv_heads": cfg["Hkv"], "head_dim": cfg["D"],
            "k_f": cfg["k_f"], "d_f": cfg["d_f"], "d": d, "k": k, "cache_dtype": "bf16",
            "rotary": f"pre-rotary PCA, rotate-then-project, base {cfg['base']:g}",
            "l2": "inputs larger than L2 (KV per layer >> 126 MB); no flush",
            "parallelism": f"kv-head shard x{world}" if world > 1 else "single GPU",
            **({"gqa_queries": cfg.get("gqa_queries", "independent")} if cfg["Hq"] > cfg["Hkv"] else {})}


# ----------------------------------------------------------------------------- main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-units", type=int, default=128)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the SDPA / flashinfer dense comparators")
    ap.add_argument("--gqa-queries", default="independent", choices=["independent", "correlated"],
                    help="GQA query heads: independent N(0,1), or q_0 + 0.5 eps per group (SURVEY 8(d) M2)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = dict(CONFIGS[args.config], gqa_queries=args.gqa_queries)
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, cfg, int(os.environ.get("WORLD_SIZE", "1")), rank)
        return

    import torch

    world, rank, local = dist_setup()
    import paper_2406_02542_b200 as L
    from paper_2406_02542_b200 import metrics

    wl = Workload(cfg, world, rank)
    decs = wl.decoders()
    step, mode = capture(make_step(wl, decs, world))
    attend, _ = capture(make_step(wl, decs, world, attend_only=True))
    dense_decs = wl.decoders(dense=True)
    dense_step, _ = capture(make_step(wl, dense_decs, world))
    dense_attend, _ = capture(make_step(wl, dense_decs, world, attend_only=True))
    plan = decs[0].call.plan()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ms = time_region(step, args.steps, world)
    clocks_rec = clocks.stop()
    us_layer = ms * 1000.0 / (args.steps * wl.L)

    # dominant kernel alone (fused decode), same stream, CUDA events
    reps = max(10, args.steps // 2)
    for _ in range(3):
        attend()
    fused_us = time_region(attend, reps, world) * 1000.0 / (reps * wl.L)
    for _ in range(3):
        dense_step()
    dense_us = time_region(dense_step, reps, world) * 1000.0 / (reps * wl.L)
    dense_attn_us = time_region(dense_attend, reps, world) * 1000.0 / (reps * wl.L)
    append_us = max(0.0, us_layer - fused_us)

    units = wl.B * wl.Hkv_l
    elem = 2
    U = float(wl.k)
    if wl.G > 1:  # GQA: rows gathered = |union of the group's selections|, measured on layer 0
        U = union_rows(wl, decs[0])
    algo_bytes = metrics.loki_bytes(units, wl.S, wl.D, wl.d, U, elem)
    dense_bytes = metrics.dense_bytes(units, wl.S, wl.D, elem)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"
    achieved = algo_bytes / (fused_us * 1e-6) / 1e9
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))
        traffic = prof.get(args.config, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        pass

    # e2e: the public API (LokiDecoder.step per layer) with pinned host inputs and a D2H of the result
    e2e = None
    if not args.no_e2e:
        hq = wl.q_raw.cpu().pin_memory()
        hk = wl.k_raw.cpu().pin_memory()
        hv = wl.v_new.cpu().pin_memory()
        hout = torch.empty_like(wl.out[-1], device="cpu").pin_memory()

        # the public serving API: L.DecodeGraph replays the captured layer loop (LokiDecoder.step per layer,
        # plus the head all-gather when sharded); eager LokiDecoder.step calls if capture is not possible
        try:
            dg = L.DecodeGraph(decs, between=(lambda layer: gather_outputs(wl, layer)) if world > 1 else None)
            run_layers, e2e_path = dg.replay, "paper_2406_02542_b200.DecodeGraph.replay (CUDA graph of LokiDecoder.step per layer; ctypes -> libloki_b200)"
        except Exception as e:  # pragma: no cover - depends on driver / NCCL build
            log(f"[bench] DecodeGraph capture failed ({e}); e2e through eager LokiDecoder.step")

            def run_layers():
                for layer, dec in enumerate(decs):
                    dec.step()
                    if world > 1:
                        gather_outputs(wl, layer)
            e2e_path = "paper_2406_02542_b200.LokiDecoder.step (ctypes -> libloki_b200), eager launches"

        def e2e_step():
            wl.q_raw.copy_(hq, non_blocking=True)
            wl.k_raw.copy_(hk, non_blocking=True)
            wl.v_new.copy_(hv, non_blocking=True)
            run_layers()
            hout.copy_(wl.out[-1], non_blocking=True)
        for _ in range(3):
            e2e_step()
        e_steps = max(5, args.steps // 4)
        e_ms = time_region(e2e_step, e_steps, world)
        bi = (hq.numel() + hk.numel() + hv.numel()) * 4
        e2e = {"value": round(e_ms * 1000.0 / (e_steps * wl.L), 3), "unit": "µs/layer",
               "h2d_bytes_per_step": bi, "d2h_bytes_per_step": hout.numel() * 4,
               "path": e2e_path}

    extras = {}
    if not args.no_extras and rank == 0 and world == 1:
        extras["dense_sdpa_us_per_layer"] = sdpa_dense_us(wl, 10)
        extras["dense_flashinfer_us_per_layer"] = flashinfer_dense_us(wl, 10)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        wl.decs_q_hat = decs[0].q_hat
        q, K, V = cpu_sample_from_device(wl, args.cpu_units)
        us_cpu, cores, wall = cpu_baseline(q, K, V, wl.d, wl.k, wl.B * wl.Hq_l)
        cpu = {"value": round(us_cpu, 1), "unit": "µs/layer", "cores": cores, "kind": "port",
               "sample": f"{q.shape[0]} of {wl.B * wl.Hq_l} (batch, head) units of layer 0 (bf16 cache upcast "
                         f"to fp32), one forked process per core, median of 3, extrapolated linearly"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(us_layer, 3), "unit": "µs/layer", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic: planted rank-16 pre-rotary keys (sigma 1e-3) rotated (RoPE) and PCA-projected "
                    "per (layer, KV head); V, q, k ~ N(0,1); random init, no checkpoint",
            "config": config_block(cfg, args, world, wl.d, wl.k),
            "speedup_vs_dense": round(dense_us / us_layer, 3),
            "speedup_vs_dense_attention_only": round(dense_attn_us / fused_us, 3),
            "loki_attention_us_per_layer": round(fused_us, 3),
            "append_us_per_layer": round(append_us, 3),
            "dense_us_per_layer": round(dense_us, 3),
            "dense_attention_us_per_layer": round(dense_attn_us, 3),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "kernel": "pipe_decode_kernel (persistent; approx scores + top-k + tensor-core sparse attention)",
                         "algorithmic_bytes_per_launch": int(algo_bytes), "peak_source": peak_src,
                         "rows_gathered_per_unit": round(U, 1),
                         "dense_achieved_gbs": round(dense_bytes / (dense_attn_us * 1e-6) / 1e9, 1)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": (1 + (2 if plan["ctas_per_unit"] == -2 else 1)) * wl.L * args.steps,
            "clocks": clocks_rec,
            "timing": f"{mode}; CUDA events on the launching stream, barrier + sync both sides, max over ranks",
            "plan": plan,
        }
        line.update(extras)
        best = [v for k_, v in extras.items() if k_.startswith("dense_") and v]
        if best:  # against the fastest dense attention on this GPU (ours, cuDNN/flash SDPA, flashinfer)
            line["speedup_vs_best_dense_attention"] = round(min(best + [dense_attn_us]) / fused_us, 3)
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
