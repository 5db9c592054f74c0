"""CPU oracle for the Loki decode-attention hot path.  TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` leg may import it.  The shipped package
(``paper_2406_02542_b200``) never imports anything under ``oracle/`` and has
no CPU fallback.

It restates, in plain numpy, the algorithm of the reference package
``lokiattn`` (``/root/reference/pkg/src/lokiattn``) for the path named by
BASELINE.json's north star.  Every function cites the reference file:line it
follows.  Arithmetic widths follow the reference exactly: fp32 products and
accumulation for the score / weighted-sum kernels (the reference's numba
kernels accumulate in float32 with ``fastmath`` reassociation), fp64 for
softmax, RoPE and calibration, and the reference's deterministic top-k
tie rule (ties at the threshold go to the lowest index, output ascending).

Parity is PINNED: ``tests/test_oracle.py`` checks every function here against
golden vectors produced by importing the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/ref_golden.npz``) and
against the reference's shipped ``hand4_expected*.tsv`` fixtures.
"""

from __future__ import annotations

import math

import numpy as np

F32 = np.float32
F64 = np.float64

ROTATE_THEN_PROJECT = "rotate-then-project"
PROJECT_THEN_ROTATE = "project-then-rotate"


# --------------------------------------------------------------------------
# budgets  (attention.py:40-64)
# --------------------------------------------------------------------------

def resolve_fraction(fraction: float, total: int) -> int:
    """clamp(floor(f * total + 0.5), 1, total)   -- attention.py:40-46."""
    assert 0.0 < fraction <= 1.0 and total >= 1
    n = math.floor(fraction * total + 0.5)
    return int(min(max(n, 1), total))


def resolve(k_f: float, d_f: float, head_dim: int, seq_len: int):
    """(d, k) for a head dim and post-append cache length -- attention.py:62-64, :204."""
    return resolve_fraction(d_f, head_dim), resolve_fraction(k_f, seq_len)


# --------------------------------------------------------------------------
# dtype helpers (not in the reference: the GPU stores bf16 caches, and the
# oracle is fed the bf16-rounded values upcast to fp32, SURVEY 7 hard part 4)
# --------------------------------------------------------------------------

def round_bf16(x) -> np.ndarray:
    """fp32 -> bf16 (round to nearest even) -> fp32, bit-exact with CUDA's __float2bfloat16_rn."""
    a = np.ascontiguousarray(x, dtype=F32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    nan = np.isnan(a)
    out = (r & 0xFFFFFFFF).astype(np.uint32).view(F32).reshape(a.shape)
    if nan.any():
        out = out.copy()
        out[nan] = np.nan
    return out


# --------------------------------------------------------------------------
# L2 kernels  (kernels.py)
# --------------------------------------------------------------------------

def _query_block(q):
    q = np.asarray(q, dtype=F32)
    return (q.reshape(1, -1), True) if q.ndim == 1 else (q, False)


def sliced_scores(q_hat, K_hat, d: int) -> np.ndarray:
    """out[i, j] = sum_{t<d} Q[i, t] K[j, t] in fp32 -- kernels.py:91-116, :223-241."""
    Q, squeeze = _query_block(q_hat)
    K = np.asarray(K_hat, dtype=F32)
    assert 1 <= d <= K.shape[1]
    out = (K[:, :d] @ Q[:, :d].T).T.astype(F32)
    return out[0] if squeeze else out


def gathered_scores(q_hat, K_hat, indices) -> np.ndarray:
    """out[i, j] = Q[i, :] . K[idx[j], :] in fp32 -- kernels.py:119-148, :244-261."""
    Q, squeeze = _query_block(q_hat)
    K = np.asarray(K_hat, dtype=F32)
    idx = np.asarray(indices, dtype=np.int64).reshape(-1)
    out = (K[idx] @ Q.T).T.astype(F32)
    return out[0] if squeeze else out


def gathered_wsum(weights, V, indices) -> np.ndarray:
    """y = sum_j w[j] V[idx[j], :] in fp32 -- kernels.py:151-181, :264-279."""
    w = np.asarray(weights, dtype=F32).reshape(-1)
    Vm = np.asarray(V, dtype=F32)
    idx = np.asarray(indices, dtype=np.int64).reshape(-1)
    return (w @ Vm[idx]).astype(F32)


def dense_wsum(weights, V) -> np.ndarray:
    """y = sum_j w[j] V[j, :] in fp32 -- kernels.py:184-211, :282-294."""
    return (np.asarray(weights, dtype=F32).reshape(-1) @ np.asarray(V, dtype=F32)).astype(F32)


# --------------------------------------------------------------------------
# L1 primitives  (linalg.py)
# --------------------------------------------------------------------------

def softmax_row(scores) -> np.ndarray:
    """fp64 max-subtract / exp / normalise, cast back to fp32 -- linalg.py:76-92."""
    s = np.asarray(scores).reshape(-1)
    assert s.size > 0
    z = s.astype(F64)
    e = np.exp(z - z.max())
    out = e / e.sum()
    return out.astype(s.dtype if s.dtype in (F32, F64) else F32)


def topk_indices(scores, k: int) -> np.ndarray:
    """Indices of the k largest scores, ascending, ties to the lower index -- linalg.py:95-118.

    Restated as a stable descending sort (an independent route from the
    reference's np.partition + threshold fill).  -0.0 and +0.0 compare equal,
    exactly as in the reference.  k == n short-circuits to arange (linalg.py:105).
    """
    s = np.asarray(scores).reshape(-1)
    n = s.size
    assert 1 <= k <= n
    if k == n:
        return np.arange(n, dtype=np.int64)
    order = np.argsort(-s.astype(F64), kind="stable")
    return np.sort(order[:k]).astype(np.int64)


def canonicalize_indices(indices, n: int) -> np.ndarray:
    """Ascending, unique, in-range -- linalg.py:121-138 / kernels.py:48-73."""
    idx = np.sort(np.asarray(indices, dtype=np.int64).reshape(-1))
    assert idx.size == 0 or (np.all(idx[1:] != idx[:-1]) and idx[0] >= 0 and idx[-1] < n)
    return idx


# --------------------------------------------------------------------------
# L3 attention  (attention.py)
# --------------------------------------------------------------------------

def loki_rank_and_attend(q_hat, K_hat, V, d: int, k: int):
    """approx -> topk -> exact/sqrt(D) -> softmax -> wsum -- attention.py:166-185.

    Returns (y fp32 [D], indices int64 [k], approx fp32 [S], weights fp32 [k]).
    """
    q = np.asarray(q_hat, dtype=F32).reshape(-1)
    K = np.asarray(K_hat, dtype=F32)
    Vm = np.asarray(V, dtype=F32)
    S, D = K.shape
    assert 1 <= d <= D and 1 <= k <= S
    approx = sliced_scores(q, K, d)
    idx = topk_indices(approx, k)
    exact = gathered_scores(q, K, idx) / F32(math.sqrt(D))
    w = softmax_row(exact.astype(F32))
    y = gathered_wsum(w, Vm, idx)
    return y, idx, approx, w


def vanilla_attention(q, K, V):
    """softmax(K q / sqrt(D)) V over all rows -- attention.py:137-142."""
    q = np.asarray(q, dtype=F32).reshape(-1)
    K = np.asarray(K, dtype=F32)
    logits = (K @ q).astype(F32) / F32(math.sqrt(K.shape[1]))
    w = softmax_row(logits)
    return (w @ np.asarray(V, dtype=F32)).astype(F32), w


def exact_topk_attention(q, K, V, k: int):
    """Select on unscaled exact logits, softmax over the selection -- attention.py:145-156."""
    q = np.asarray(q, dtype=F32).reshape(-1)
    K = np.asarray(K, dtype=F32)
    logits = (K @ q).astype(F32)
    idx = topk_indices(logits, k)
    w = softmax_row(logits[idx] / F32(math.sqrt(K.shape[1])))
    return (w @ np.asarray(V, dtype=F32)[idx]).astype(F32), idx


def loki_decode_batched(q_hat, K_hat, V, lens, d: int, k_f: float = None, k=None):
    """Batched/GQA restatement: every (b, query head) is an independent call of
    loki_rank_and_attend on its KV head (attention.py:166-185).

    q_hat [B, Hq, D]; K_hat, V [B, Hkv, S_cap, D]; lens [B] cache lengths.
    k: int or per-batch list; else resolved from k_f per batch (attention.py:204).
    Returns y [B, Hq, D] and a list-of-lists of (idx, approx, weights).
    """
    q_hat = np.asarray(q_hat, dtype=F32)
    B, Hq, D = q_hat.shape
    Hkv = K_hat.shape[1]
    G = Hq // Hkv
    y = np.zeros((B, Hq, D), dtype=F32)
    diags = []
    for b in range(B):
        S = int(lens[b])
        if k is None:
            kb = resolve_fraction(k_f, S)
        else:
            kb = int(k[b]) if np.ndim(k) else int(k)
        row = []
        for h in range(Hq):
            g = h // G
            yy, idx, approx, w = loki_rank_and_attend(
                q_hat[b, h], K_hat[b, g, :S], V[b, g, :S], d, kb)
            y[b, h] = yy
            row.append((idx, approx, w))
        diags.append(row)
    return y, diags


def loki_rank_and_attend_shared(q_block, K_hat, V, d: int, k: int):
    """Group-shared selection (opt-in GQA mode, SURVEY 7 hard part 3), composed from
    the reference's primitives: sliced_score_kernel on the [G, D] query block
    (kernels.py:223-241), summed over the group, ONE topk_indices (linalg.py:95-118),
    then per query head the exact path of attention.py:180-184.

    Returns (y fp32 [G, D], indices int64 [k], group scores fp32 [S], weights fp32 [G, k]).
    """
    Q = np.asarray(q_block, dtype=F32).reshape(-1, np.shape(K_hat)[1])
    K = np.asarray(K_hat, dtype=F32)
    Vm = np.asarray(V, dtype=F32)
    S, D = K.shape
    assert 1 <= d <= D and 1 <= k <= S
    group = sliced_scores(Q, K, d).reshape(Q.shape[0], S).sum(axis=0, dtype=F32)
    idx = topk_indices(group, k)
    ys, ws = [], []
    for g in range(Q.shape[0]):
        y, w = attend_on(Q[g], K, Vm, idx)
        ys.append(y)
        ws.append(w)
    return np.stack(ys).astype(F32), idx, group, np.stack(ws)


def loki_decode_batched_shared(q_hat, K_hat, V, lens, d: int, k_f: float = None, k=None):
    """Batched restatement of the group-shared mode: one selection per (b, KV head) on
    the group's summed leading-d scores, every query head of the group attends over it.
    Returns y [B, Hq, D] and per (b, kv head) (idx, group scores, weights [G, k])."""
    q_hat = np.asarray(q_hat, dtype=F32)
    B, Hq, D = q_hat.shape
    Hkv = K_hat.shape[1]
    G = Hq // Hkv
    y = np.zeros((B, Hq, D), dtype=F32)
    diags = []
    for b in range(B):
        S = int(lens[b])
        kb = resolve_fraction(k_f, S) if k is None else (int(k[b]) if np.ndim(k) else int(k))
        row = []
        for g in range(Hkv):
            yy, idx, grp, w = loki_rank_and_attend_shared(q_hat[b, g * G:(g + 1) * G], K_hat[b, g, :S],
                                                          V[b, g, :S], d, kb)
            y[b, g * G:(g + 1) * G] = yy
            row.append((idx, grp, w))
        diags.append(row)
    return y, diags


def pca_attn(q, K_hat_d, V, P_d):
    """Attend to every token on the leading-d coordinates only, logits scaled by
    sqrt(D) of the full head -- attention.py:209-232."""
    q = np.asarray(q, dtype=F32).reshape(-1)
    K = np.asarray(K_hat_d, dtype=F32)
    P_d = np.asarray(P_d, dtype=F32)
    D = P_d.shape[0]
    q_hat_d = (q @ P_d).astype(F32)
    logits = (K @ q_hat_d).astype(F32) / F32(math.sqrt(D))
    w = softmax_row(logits)
    return (w @ np.asarray(V, dtype=F32)).astype(F32)


# --------------------------------------------------------------------------
# rotary embedding  (rope.py)
# --------------------------------------------------------------------------

def rope_inv_freq(head_dim: int, base: float) -> np.ndarray:
    """base ** (-(2 i) / D) in fp64 -- rope.py:29-35, :66."""
    half = head_dim // 2
    return base ** (-np.arange(half, dtype=F64) * 2.0 / head_dim)


def rope_apply(v, position: int, head_dim: int, base: float = 10000.0) -> np.ndarray:
    """Half-split rotation of pair (i, i + D/2) by position * inv_freq[i], fp64 -- rope.py:38-55."""
    a = np.asarray(v)
    theta = position * rope_inv_freq(head_dim, base)
    c, s = np.cos(theta), np.sin(theta)
    x = a.astype(F64)
    h = head_dim // 2
    out = np.concatenate([x[:h] * c - x[h:] * s, x[:h] * s + x[h:] * c])
    return out.astype(a.dtype if a.dtype.kind == "f" else F64)


def rope_apply_rows(mat, head_dim: int, base: float = 10000.0, start_position: int = 0):
    """Row i rotated to start_position + i -- rope.py:58-75."""
    m = np.asarray(mat)
    pos = np.arange(start_position, start_position + m.shape[0], dtype=F64)
    theta = np.outer(pos, rope_inv_freq(head_dim, base))
    c, s = np.cos(theta), np.sin(theta)
    x = m.astype(F64)
    h = head_dim // 2
    out = np.concatenate([x[:, :h] * c - x[:, h:] * s, x[:, :h] * s + x[:, h:] * c], axis=1)
    return out.astype(m.dtype if m.dtype.kind == "f" else F64)


def transform_step(q_raw, k_raw, position: int, P, base: float = 10000.0,
                   mode: str = ROTATE_THEN_PROJECT):
    """(q_hat, k_hat) for one raw pair -- attention.py:316-341."""
    q = np.asarray(q_raw, dtype=F32).reshape(-1)
    kk = np.asarray(k_raw, dtype=F32).reshape(-1)
    P = np.asarray(P, dtype=F32)
    D = P.shape[0]
    if mode == ROTATE_THEN_PROJECT:
        return (rope_apply(q, position, D, base) @ P).astype(F32), \
               (rope_apply(kk, position, D, base) @ P).astype(F32)
    assert mode == PROJECT_THEN_ROTATE
    return rope_apply((q @ P).astype(F32), position, D, base), \
        rope_apply((kk @ P).astype(F32), position, D, base)


# --------------------------------------------------------------------------
# calibration  (calibration.py) and the synthetic generator (dataio.py)
# --------------------------------------------------------------------------

def build_projection(keys):
    """Centered fp64 covariance, eigh, descending stable order, largest-|entry|
    positive, clip + normalise spectrum; P fp32 -- calibration.py:51-123."""
    k = np.asarray(keys, dtype=F64)
    c = k - k.mean(axis=0)
    cov = (c.T @ c) / (k.shape[0] - 1)
    cov = (cov + cov.T) * 0.5
    vals, vecs = np.linalg.eigh((cov + cov.T) * 0.5)
    order = np.argsort(-vals, kind="stable")
    vals, vecs = vals[order], vecs[:, order]
    pick = np.abs(vecs).argmax(axis=0)
    sign = np.where(vecs[pick, np.arange(vecs.shape[1])] < 0.0, -1.0, 1.0)
    vecs = vecs * sign
    vals = np.clip(vals, 0.0, None)
    return np.ascontiguousarray(vecs, dtype=F32), (vals / vals.sum()).astype(F32)


def gen_synthetic_keys(seq_len: int, head_dim: int, rank: int, sigma: float = 0.0,
                       seed: int = 0) -> np.ndarray:
    """K = Z B' + sigma E from one PCG64 stream -- dataio.py:225-240."""
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((seq_len, rank))
    basis, r = np.linalg.qr(rng.standard_normal((head_dim, rank)))
    basis = basis * np.where(np.diag(r) < 0.0, -1.0, 1.0)
    e = rng.standard_normal((seq_len, head_dim))
    return (z @ basis.T + sigma * e).astype(F32)


# --------------------------------------------------------------------------
# parity helpers and the reference's relative error
# --------------------------------------------------------------------------

def rel_err(actual, expected) -> float:
    """max|a - e| / max|e|  -- tests/oracles.py:91-95."""
    a = np.asarray(actual, dtype=F64)
    e = np.asarray(expected, dtype=F64)
    return float(np.abs(a - e).max()) / max(1e-30, float(np.abs(e).max()))


def tie_band(q_hat, K_hat, d: int, k: int) -> np.ndarray:
    """Tokens whose approximate-score rank is not decided by fp32 arithmetic.

    a64 = fp64 leading-d scores; T = a64 at the k-th largest position j*;
    tau_j = gamma_d * sum_t |q_t K_jt| with gamma_d = d u / (1 - d u),
    u = 2^-24 (worst case of ANY fp32 summation order).  The band is
    {j : |a64_j - T| <= 2 (tau_j + tau_j*)}.  Returns a bool mask [S].
    """
    q = np.asarray(q_hat, dtype=F64).reshape(-1)[:d]
    K = np.asarray(K_hat, dtype=F64)[:, :d]
    a64 = K @ q
    S = a64.size
    if k >= S:
        return np.zeros(S, dtype=bool)
    u = 2.0 ** -24
    gamma = d * u / (1.0 - d * u)
    tau = gamma * (np.abs(K) @ np.abs(q))
    order = np.argsort(-a64, kind="stable")
    jstar = order[k - 1]
    T = a64[jstar]
    return np.abs(a64 - T) <= 2.0 * (tau + tau[jstar])


def tie_band_shared(q_block, K_hat, d: int, k: int) -> np.ndarray:
    """Tie band of the group-shared selection: the group score sum_g q_g . K_j[:d] is
    computed either as a sum of G per-head fp32 dots (the reference composition) or as
    one dot with the fp32-summed query (the kernel); both are within
    gamma_{d+G} sum_g sum_t |q_gt K_jt| of the exact value."""
    Q = np.asarray(q_block, dtype=F64).reshape(-1, np.shape(K_hat)[1])[:, :d]
    K = np.asarray(K_hat, dtype=F64)[:, :d]
    a64 = K @ Q.sum(axis=0)
    S = a64.size
    if k >= S:
        return np.zeros(S, dtype=bool)
    u = 2.0 ** -24
    n = d + Q.shape[0]
    gamma = n * u / (1.0 - n * u)
    tau = gamma * (np.abs(K) @ np.abs(Q).sum(axis=0))
    order = np.argsort(-a64, kind="stable")
    jstar = order[k - 1]
    return np.abs(a64 - a64[jstar]) <= 2.0 * (tau + tau[jstar])


def sets_match_outside_band(gpu_idx, ref_idx, band) -> bool:
    """|gpu| == |ref| and they agree on every token outside the tie band."""
    g = np.asarray(gpu_idx, dtype=np.int64).reshape(-1)
    r = np.asarray(ref_idx, dtype=np.int64).reshape(-1)
    if g.size != r.size or np.unique(g).size != g.size:
        return False
    out_band = ~band
    gm = np.zeros(band.size, dtype=bool)
    rm = np.zeros(band.size, dtype=bool)
    gm[g] = True
    rm[r] = True
    return bool(np.array_equal(gm[out_band], rm[out_band]))


def attend_on(q_hat, K_hat, V, indices):
    """Exact attention restricted to a given selection: gathered scores / sqrt(D),
    fp64 softmax, gathered weighted sum (attention.py:182-184).  Used when a GPU
    selection differs from the oracle's only inside the tie band."""
    q = np.asarray(q_hat, dtype=F32).reshape(-1)
    K = np.asarray(K_hat, dtype=F32)
    idx = np.asarray(indices, dtype=np.int64).reshape(-1)
    exact = gathered_scores(q, K, idx) / F32(math.sqrt(K.shape[1]))
    w = softmax_row(exact.astype(F32))
    return gathered_wsum(w, V, idx), w


# --------------------------------------------------------------------------
# timing-faithful restatement for the CPU baseline (bench.py cpu_baseline leg)
# --------------------------------------------------------------------------

def topk_indices_partition(scores, k: int) -> np.ndarray:
    """Same result as topk_indices, computed the reference's way: introselect
    for the threshold, everything above it, ties lowest-index-first, sorted
    (linalg.py:105-118).  O(S) like the reference, so the CPU timing is fair."""
    s = np.asarray(scores).reshape(-1)
    n = s.size
    if k == n:
        return np.arange(n, dtype=np.int64)
    t = np.partition(s, n - k)[n - k]
    above = np.flatnonzero(s > t)
    ties = np.flatnonzero(s == t)[: k - above.size]
    out = np.concatenate([above, ties])
    out.sort()
    return out.astype(np.int64, copy=False)


def loki_unit_cpu(q_hat, K_hat, V, d: int, k: int):
    """One (batch, head) unit of the reference's CPU path (attention.py:166-185)
    with the O(S) selection; returns y only.  Used to time the CPU baseline."""
    S, D = K_hat.shape
    approx = K_hat[:, :d] @ q_hat[:d]
    idx = topk_indices_partition(approx, k)
    exact = (K_hat[idx] @ q_hat) / F32(math.sqrt(D))
    z = exact.astype(F64)
    e = np.exp(z - z.max())
    w = (e / e.sum()).astype(F32)
    return w @ V[idx]


def dense_unit_cpu(q, K, V):
    """One unit of vanilla_attention (attention.py:137-142); returns y only."""
    logits = (K @ q) / F32(math.sqrt(K.shape[1]))
    z = logits.astype(F64)
    e = np.exp(z - z.max())
    return (e / e.sum()).astype(F32) @ V
