"""Regenerate the large golden inputs from seeds (tests/golden/make_golden.py).

Uses the oracle's restatements of gen_synthetic_keys / build_projection, so a
matching SHA-256 also pins those two functions bit-exactly to the reference.
"""

import hashlib

import numpy as np

from oracle import loki_oracle as O


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def gaussian_case(S, D, seed):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal(D).astype(np.float32)
    K = rng.standard_normal((S, D)).astype(np.float32)
    V = rng.standard_normal((S, D)).astype(np.float32)
    return rng, q, K, V


def loki_inputs(S, D, seed, rank, sigma):
    rng = np.random.default_rng(seed)
    if rank is None or rank < 0:
        K = rng.standard_normal((S, D)).astype(np.float32)
        calib = O.gen_synthetic_keys(max(4 * D, 256), D, D, 0.0, seed + 1)
    else:
        allk = O.gen_synthetic_keys(S + 1024, D, int(rank), sigma, seed)
        calib, K = allk[:1024], np.ascontiguousarray(allk[1024:])
    V = rng.standard_normal((S, D)).astype(np.float32)
    q = rng.standard_normal(D).astype(np.float32)
    P, _ = O.build_projection(calib)
    return q, K, V, P


def loki_case(golden, i):
    S, D, d, k, seed, r, sg = golden["loki/cases"][i]
    S, D, d, k, seed = int(S), int(D), int(d), int(k), int(seed)
    q, K, V, P = loki_inputs(S, D, seed, None if r < 0 else int(r), float(sg))
    assert digest(q, K, V, P) == str(golden[f"loki/{i}/sha"]), "input regeneration drifted"
    q_hat = np.asarray(q @ P, np.float32)
    K_hat = np.ascontiguousarray(K @ P, dtype=np.float32)
    return dict(S=S, D=D, d=d, k=k, q=q, K=K, V=V, P=P, q_hat=q_hat, K_hat=K_hat)


def ragged(golden, prefix, i):
    offs = golden[prefix + "/offsets"]
    return offs[i], offs[i + 1]


def shared_case(golden, i):
    """Inputs of make_golden.shared_cases() case i (same draw order), digest-checked."""
    S, D, G, d, k, seed = (int(x) for x in golden["shared/cases"][i])
    rng = np.random.default_rng(seed)
    Q = rng.standard_normal((G, D)).astype(np.float32)
    K = rng.standard_normal((S, D)).astype(np.float32)
    V = rng.standard_normal((S, D)).astype(np.float32)
    assert digest(Q, K, V) == str(golden[f"shared/{i}/sha"]), "input regeneration drifted"
    return dict(S=S, D=D, G=G, d=d, k=k, Q=Q, K=K, V=V)


def quality_inputs(golden):
    """Inputs of make_golden.quality_cases() (agreement sweep, pca_attn), digest-checked."""
    keys = O.gen_synthetic_keys(2048, 64, 8, 1e-2, 21)
    rng = np.random.default_rng(22)
    V = rng.standard_normal(keys.shape).astype(np.float32)
    Q = rng.standard_normal((6, 64)).astype(np.float32)
    assert digest(keys, V, Q) == str(golden["agree/keys_sha"]), "input regeneration drifted"
    return keys, V, Q
