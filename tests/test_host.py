"""CPU-only checks of the host side: the C-ABI library loads and exports every
symbol include/loki_b200.h declares, the ctypes layouts match the C structs,
host validation maps to the reference's exception classes, and the host
helpers mirror the reference's KATs.  No kernel is launched."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "loki_b200.h")

import paper_2406_02542_b200 as L  # noqa: E402
from paper_2406_02542_b200 import _lib  # noqa: E402


def _declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(loki_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2406_02542_b200 import _build

        _build.build()
    return _lib.load()


def test_library_exports_every_declared_symbol(lib):
    declared = _declared_symbols()
    assert len(declared) >= 12
    assert sorted(_lib.EXPORTED) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (loki_\w+)", out))
    assert set(declared) <= exported
    assert lib.loki_abi_version() == 1


def test_ctypes_layout_matches_c_header(tmp_path):
    src = tmp_path / "layout.c"
    fields = [f for f, _ in _lib.DecodeArgs._fields_]
    gfields = [f for f, _ in _lib.KvGeom._fields_]
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "loki_b200.h"', "int main(void){",
             'printf("%zu %zu\\n", sizeof(loki_decode_args), sizeof(loki_kv_geom));']
    lines += [f'printf("%zu\\n", offsetof(loki_decode_args, {f}));' for f in fields]
    lines += [f'printf("%zu\\n", offsetof(loki_kv_geom, {f}));' for f in gfields]
    lines.append("return 0;}")
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    vals = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert vals[0] == ctypes.sizeof(_lib.DecodeArgs)
    assert vals[1] == ctypes.sizeof(_lib.KvGeom)
    got = [getattr(_lib.DecodeArgs, f).offset for f in fields] + [getattr(_lib.KvGeom, f).offset for f in gfields]
    assert vals[2:] == got


def _args(**kw):
    a = _lib.DecodeArgs()
    a.g = _lib.KvGeom(1, 1, 1, 128, 4096, _lib.DTYPE_BF16, 4096 * 128, 4096 * 128, 128)
    a.q_hat = a.K = a.V = a.lens = a.out = 16  # never dereferenced: validation fails first
    a.S_max, a.d, a.k_fixed, a.select_mode = 4096, 32, 1024, _lib.SELECT_TOPK
    for k, v in kw.items():
        setattr(a, k, v)
    return a


@pytest.mark.parametrize("kw,exc,msg", [
    (dict(d=0), L.BudgetError, "d=0 outside [1, 128]"),
    (dict(d=129), L.BudgetError, "d=129 outside [1, 128]"),
    (dict(k_fixed=4097), L.BudgetError, "k=4097 outside [1, 4096]"),
    (dict(k_fixed=0, k_f=1.5), L.DomainError, "budget fraction must lie in (0, 1], got 1.5"),
    (dict(S_max=0), L.ShapeError, "attention needs at least one cached token"),
    (dict(g=_lib.KvGeom(1, 3, 2, 128, 4096, 1, 0, 0, 128)), L.ShapeError, "not a multiple"),
    (dict(g=_lib.KvGeom(1, 16, 1, 128, 4096, 1, 0, 0, 128)), L.UnsupportedShapeError, "group size 16"),
    (dict(g=_lib.KvGeom(1, 1, 1, 512, 4096, 1, 0, 0, 512)), L.UnsupportedShapeError, "head dim"),
])
def test_c_validation_maps_to_reference_errors(lib, kw, exc, msg):
    a = _args(**kw)
    status = lib.loki_decode(ctypes.byref(a), None)
    with pytest.raises(exc, match=re.escape(msg)):
        _lib.check(status)


def test_resolve_fraction_kats(golden):
    for (f, n), ref in zip(golden["budget/cases"], golden["budget/ref"]):
        assert L.resolve_fraction(float(f), int(n)) == int(ref)
    assert L.LokiConfig(k_f=0.25, d_f=0.25).resolve(128, 4096) == (32, 1024)
    with pytest.raises(L.DomainError):
        L.resolve_fraction(0.0, 10)
    with pytest.raises(L.DomainError):
        L.LokiConfig(k_f=0.0, d_f=0.5)


def test_speedup_model_kats():
    assert L.theoretical_speedup(0.25, 0.25) == pytest.approx(2.6667, abs=1e-4)
    assert L.exact_speedup(128, 4096, 32, 1024) == pytest.approx(1048576 / 425984)
    assert L.jaccard_topk([1, 2, 3], [2, 3, 4]) == 0.5


def test_synthetic_generator_matches_reference(golden):
    keys = L.gen_synthetic_keys(L.SyntheticSpec(64, 16, 4, 0.01, 3))
    assert np.array_equal(keys, golden["synth/S64_D16_r4_s0.01_seed3"])


def test_key_dump_and_projection_roundtrip(tmp_path):
    rng = np.random.default_rng(1111)
    keys = rng.standard_normal((48, 24)).astype(np.float32)
    header = L.KeyDumpHeader(layer=1, head=2, seq_len=48, head_dim=24, rotary_stage="post")
    path = tmp_path / "rt.lkd"
    L.write_key_dump(path, header, keys)
    h2, back = L.read_key_dump(path)
    assert h2 == header and np.array_equal(back, keys)
    from oracle import loki_oracle as O

    P, eig = O.build_projection(O.gen_synthetic_keys(256, 12, 12, 0.0, 1112))
    proj = L.ProjectionSet(0, 0, P, eig, "post")
    L.write_projection(tmp_path / "rt.lkp", proj)
    p2 = L.read_projection(tmp_path / "rt.lkp")
    assert np.array_equal(p2.P, P) and np.array_equal(p2.eigenvalues, eig)
    blob = bytearray(open(path, "rb").read())
    blob[:4] = b"XKD1"
    open(path, "wb").write(bytes(blob))
    from paper_2406_02542_b200.errors import MagicError

    with pytest.raises(MagicError):
        L.read_key_dump(path)


def test_compute_path_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.LibraryMissing):
        L.loki_rank_and_attend(np.ones(8, np.float32), np.ones((4, 8), np.float32), np.ones((4, 8), np.float32), 2, 2)


def test_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2406_02542_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            assert "oracle" not in re.sub(r"#.*", "", open(os.path.join(pkg, f)).read()).split("import")[0] or \
                "from oracle" not in open(os.path.join(pkg, f)).read(), f
            assert "from oracle" not in open(os.path.join(pkg, f)).read()
            assert "import oracle" not in open(os.path.join(pkg, f)).read()


def test_decode_graph_validates_before_capture():
    """DecodeGraph rejects an empty layer list with the reference's ShapeError
    before touching the device (capture itself needs a GPU: test_gpu_parity)."""
    with pytest.raises(L.ShapeError):
        L.DecodeGraph([])


def test_formats_byte_identical_to_reference_writers(golden, tmp_path):
    """N4: LKD1 / LKP1 files written by the reference's own writers (dataio.py:91-222, bytes recorded by
    tests/golden/make_golden.py) parse here, and this package writes the same bytes back."""
    import paper_2406_02542_b200 as L
    from paper_2406_02542_b200 import dataio

    ref_lkd = golden["fmt/lkd_bytes"].tobytes()
    p = tmp_path / "ref.lkd"
    p.write_bytes(ref_lkd)
    hdr, keys = dataio.read_key_dump(str(p))
    assert (hdr.layer, hdr.head, hdr.seq_len, hdr.head_dim, hdr.rotary_stage) == (3, 5, 40, 16, "post")
    np.testing.assert_array_equal(keys, golden["fmt/lkd_keys"])
    q = tmp_path / "ours.lkd"
    dataio.write_key_dump(str(q), hdr, keys)
    assert q.read_bytes() == ref_lkd

    ref_lkp = golden["fmt/lkp_bytes"].tobytes()
    p = tmp_path / "ref.lkp"
    p.write_bytes(ref_lkp)
    proj = dataio.read_projection(str(p))
    assert (proj.layer, proj.head, proj.rotary_stage) == (3, 5, "post")
    np.testing.assert_array_equal(np.asarray(proj.P), golden["fmt/lkp_P"])
    np.testing.assert_array_equal(np.asarray(proj.eigenvalues), golden["fmt/lkp_eig"])
    q = tmp_path / "ours.lkp"
    dataio.write_projection(str(q), proj)
    assert q.read_bytes() == ref_lkp
    assert L.ProjectionSet is type(proj)
