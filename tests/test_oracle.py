"""Pin the CPU oracle (oracle/loki_oracle.py) to the reference's own outputs.

Every expected value comes from tests/golden/ref_golden.npz, which
tests/golden/make_golden.py produced by importing the reference package, or
from the reference's shipped hand4_expected*.tsv fixtures.  CPU only.
"""

import math

import numpy as np
import pytest

from golden_inputs import digest, gaussian_case, loki_case
from oracle import loki_oracle as O


def test_hand4_matches_shipped_tsv(golden):
    P = golden["hand4/P"]
    K_hat = np.ascontiguousarray(golden["hand4/keys"] @ P, dtype=np.float32)
    for qi, q in enumerate(golden["hand4/queries"]):
        y, idx, _, _ = O.loki_rank_and_attend(np.asarray(q @ P, np.float32), K_hat,
                                              golden["hand4/values"], 2, 2)
        assert idx.tolist() == golden["hand4/tsv_idx"][qi].tolist()
        assert np.abs(y - golden["hand4/tsv_y"][qi]).max() <= 1e-5
        assert np.array_equal(idx, golden["hand4/ref_idx"][qi])
        assert np.abs(y - golden["hand4/ref_y"][qi]).max() <= 1e-6


def test_resolve_fraction_matches_reference(golden):
    for (f, n), ref in zip(golden["budget/cases"], golden["budget/ref"]):
        assert O.resolve_fraction(float(f), int(n)) == int(ref)
    assert O.resolve(0.25, 0.25, 128, 4096) == (32, 1024)


def test_topk_bit_exact_vs_reference(golden):
    offs, roffs = golden["topk/offsets"], golden["topk/ref_offsets"]
    flat, ref = golden["topk/scores"], golden["topk/ref_flat"]
    for i, k in enumerate(golden["topk/k"]):
        s = flat[offs[i]:offs[i + 1]]
        assert O.topk_indices(s, int(k)).tolist() == ref[roffs[i]:roffs[i + 1]].tolist(), i


def test_softmax_vs_reference(golden):
    offs = golden["softmax/offsets"]
    for i in range(offs.size - 1):
        z = golden["softmax/flat"][offs[i]:offs[i + 1]]
        assert np.array_equal(O.softmax_row(z), golden["softmax/ref_flat"][offs[i]:offs[i + 1]])


@pytest.mark.parametrize("S", [1, 2, 1000, 2048, 3000, 4095])
def test_kernels_vs_reference(golden, S):
    rng, q, K, V = gaussian_case(S, 128, S)
    assert digest(q, K, V) == str(golden[f"kern/S{S}/sha"])
    for d in (1, 17, 32, 128):
        assert O.rel_err(O.sliced_scores(q, K, d), golden[f"kern/S{S}/sliced_d{d}"]) <= 1e-5
    idx = golden[f"kern/S{S}/idx"]
    assert O.rel_err(O.gathered_scores(q, K, idx), golden[f"kern/S{S}/gathered"]) <= 1e-5
    assert O.rel_err(O.gathered_wsum(golden[f"kern/S{S}/w"], V, idx),
                     golden[f"kern/S{S}/wsum"]) <= 1e-5
    assert O.rel_err(O.dense_wsum(golden[f"kern/S{S}/wd"], V), golden[f"kern/S{S}/dense_wsum"]) <= 1e-5


def test_query_block_vs_reference(golden):
    Q, K, idx = golden["kern/block/Q"], golden["kern/block/K"], golden["kern/block/idx"]
    assert O.rel_err(O.sliced_scores(Q, K, 9), golden["kern/block/sliced_d9"]) <= 1e-5
    assert O.rel_err(O.gathered_scores(Q, K, idx), golden["kern/block/gathered"]) <= 1e-5


@pytest.mark.parametrize("i", range(8))
def test_loki_rank_and_attend_vs_reference(golden, i):
    c = loki_case(golden, i)
    y, idx, approx, w = O.loki_rank_and_attend(c["q_hat"], c["K_hat"], c["V"], c["d"], c["k"])
    ref_idx = golden[f"loki/{i}/idx"]
    band = O.tie_band(c["q_hat"], c["K_hat"], c["d"], c["k"])
    assert O.sets_match_outside_band(idx, ref_idx, band)
    assert O.rel_err(approx, golden[f"loki/{i}/approx"]) <= 1e-5
    if np.array_equal(idx, ref_idx):
        assert O.rel_err(y, golden[f"loki/{i}/y"]) <= 1e-5
        assert np.abs(w - golden[f"loki/{i}/weights"]).max() <= 1e-6
    yv, _ = O.vanilla_attention(c["q"], c["K"], c["V"])
    assert O.rel_err(yv, golden[f"loki/{i}/vanilla_y"]) <= 1e-5
    ye, ie = O.exact_topk_attention(c["q"], c["K"], c["V"], c["k"])
    assert np.array_equal(ie, golden[f"loki/{i}/exact_idx"])
    assert O.rel_err(ye, golden[f"loki/{i}/exact_y"]) <= 1e-5


@pytest.mark.parametrize("base", [10000, 500000])
@pytest.mark.parametrize("D", [16, 128])
def test_rope_vs_reference(golden, base, D):
    tag = f"rope/b{base}/D{D}"
    X, pos = golden[tag + "/x"], golden[tag + "/pos"]
    out = np.stack([O.rope_apply(X[i], int(p), D, float(base)) for i, p in enumerate(pos)])
    assert np.array_equal(out, golden[tag + "/out"])
    rows = O.rope_apply_rows(golden[tag + "/rows_x"], D, float(base), start_position=131060)
    assert np.array_equal(rows, golden[tag + "/rows_out"])


@pytest.mark.parametrize("base", [10000, 500000])
@pytest.mark.parametrize("mode", ["ROTATE_THEN_PROJECT", "PROJECT_THEN_ROTATE"])
def test_transform_step_vs_reference(golden, base, mode):
    tag = f"xform/b{base}/{mode}"
    m = O.ROTATE_THEN_PROJECT if mode == "ROTATE_THEN_PROJECT" else O.PROJECT_THEN_ROTATE
    P = golden["xform/P"]
    for i, p in enumerate(golden[tag + "/pos"]):
        qh, kh = O.transform_step(golden[tag + "/q"][i], golden[tag + "/k"][i], int(p), P, float(base), m)
        assert O.rel_err(qh, golden[tag + "/q_hat"][i]) <= 1e-6
        assert O.rel_err(kh, golden[tag + "/k_hat"][i]) <= 1e-6


def test_calibration_and_generator_vs_reference(golden):
    for tag in ("calib/S256_D16", "calib/S8192_D128", "calib/S600_D64"):
        S, D, r, sg, seed = golden[tag + "/spec"]
        keys = O.gen_synthetic_keys(int(S), int(D), int(r), float(sg), int(seed))
        assert digest(keys) == str(golden[tag + "/keys_sha"])
        P, eig = O.build_projection(keys)
        assert np.array_equal(P, golden[tag + "/P"])
        assert np.array_equal(eig, golden[tag + "/eig"])
    assert np.array_equal(O.gen_synthetic_keys(64, 16, 4, 0.01, 3), golden["synth/S64_D16_r4_s0.01_seed3"])


def test_round_bf16_known_answers():
    x = np.array([1.0, 1.00390625, 1.005859375, -2.5, 3.0e38, 1e-40, 0.0, -0.0], np.float32)
    r = O.round_bf16(x)
    assert r[0] == 1.0 and r[1] == 1.0  # tie -> even
    assert r[2] == np.float32(1.0078125)
    assert r[3] == -2.5
    assert np.all(np.isfinite(r[:4]))
    assert (r.view(np.uint32) & 0xFFFF).max() == 0


def test_tie_band_contains_threshold_and_is_small():
    rng = np.random.default_rng(0)
    for S, d in ((4096, 32), (8192, 64)):
        q = rng.standard_normal(128).astype(np.float32)
        K = rng.standard_normal((S, 128)).astype(np.float32)
        k = S // 4
        band = O.tie_band(q, K, d, k)
        assert 1 <= band.sum() <= 16
        idx = O.topk_indices(O.sliced_scores(q, K, d), k)
        assert O.sets_match_outside_band(idx, idx, band)


def test_partition_topk_equals_sorted_topk(golden):
    offs = golden["topk/offsets"]
    flat = golden["topk/scores"]
    for i, k in enumerate(golden["topk/k"]):
        s = flat[offs[i]:offs[i + 1]]
        assert np.array_equal(O.topk_indices_partition(s, int(k)), O.topk_indices(s, int(k)))


def test_cpu_unit_matches_oracle(golden):
    c = loki_case(golden, 4)
    y = O.loki_unit_cpu(c["q_hat"], c["K_hat"], c["V"], c["d"], c["k"])
    assert O.rel_err(y, golden["loki/4/y"]) <= 1e-5
    yv = O.dense_unit_cpu(c["q"], c["K"], c["V"])
    assert O.rel_err(yv, golden["loki/4/vanilla_y"]) <= 1e-5


@pytest.mark.parametrize("i", range(5))
def test_shared_selection_vs_reference_composition(golden, i):
    """The group-shared mode's oracle against the reference primitives composed in make_golden.py."""
    from golden_inputs import shared_case

    c = shared_case(golden, i)
    y, idx, group, w = O.loki_rank_and_attend_shared(c["Q"], c["K"], c["V"], c["d"], c["k"])
    assert O.rel_err(group, golden[f"shared/{i}/group"]) <= 1e-5
    band = O.tie_band_shared(c["Q"], c["K"], c["d"], c["k"])
    assert O.sets_match_outside_band(idx, golden[f"shared/{i}/idx"], band)
    if np.array_equal(idx, golden[f"shared/{i}/idx"]):
        assert O.rel_err(y, golden[f"shared/{i}/y"]) <= 1e-5
        assert np.abs(w - golden[f"shared/{i}/weights"]).max() <= 1e-6


def test_pca_attn_vs_reference(golden):
    from golden_inputs import quality_inputs

    keys, V, Q = quality_inputs(golden)
    P = golden["agree/P"]
    K_hat = (keys @ P).astype(np.float32)
    for j, d in enumerate(golden["pca_attn/d"]):
        d = int(d)
        y = np.stack([O.pca_attn(Q[i], np.ascontiguousarray(K_hat[:, :d]), V, np.ascontiguousarray(P[:, :d]))
                      for i in range(Q.shape[0])])
        assert O.rel_err(y, golden["pca_attn/y"][j]) <= 1e-5, d
