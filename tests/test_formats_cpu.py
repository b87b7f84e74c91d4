"""DZDL container parsing on the host (native parser dz_dzdl.cpp + zlib inflate) against fixtures
written by the REFERENCE writer (tests/golden/make_dzdl.py runs formats.write_delta on deltas
from compress_model): field-by-field equality with the reference's read_delta output, the
inspect_delta sizes, and the reference error contract (formats.py:102-169)."""

import json
import os

import numpy as np
import pytest

from conftest import ROOT

GOLD = os.path.join(ROOT, "tests", "golden")
CASES = ["dzdl_b4", "dzdl_b4_deflate", "dzdl_b2", "dzdl_b16_dense"]


@pytest.fixture(scope="module")
def F():
    from paper_2312_05215_b200 import formats
    return formats


@pytest.mark.parametrize("case", CASES)
def test_read_delta_matches_reference(F, case):
    cd = F.read_delta(os.path.join(GOLD, case + ".dzdl"))
    z = np.load(os.path.join(GOLD, case + ".npz"))
    meta = json.load(open(os.path.join(GOLD, case + ".json")))
    h = meta["header"]
    assert cd.base_model_id == h["base_model_id"] and cd.calibration_fingerprint == h["calibration_fingerprint"]
    assert (cd.config.bits, cd.config.sparsity, cd.config.group_size) == (h["bits"], h["sparsity"], h["group_size"])
    assert cd.config.lossless == h["codec"]
    assert len(cd.layers) == h["layer_count"] == len(meta["layers"])
    for i, (ld, lm) in enumerate(zip(cd.layers, meta["layers"])):
        assert (ld.name, ld.rows, ld.cols) == (lm["name"], lm["rows"], lm["cols"])
        assert np.array_equal(ld.packed_values, z[f"l{i}_packed"])
        assert ld.index_stream == z[f"l{i}_index"].tobytes()
        assert np.array_equal(ld.scales.view(np.uint32), z[f"l{i}_scales"].view(np.uint32))


@pytest.mark.parametrize("case", CASES)
def test_inspect_delta_matches_reference(F, case):
    header, sizes, ratio = F.inspect_delta(os.path.join(GOLD, case + ".dzdl"))
    meta = json.load(open(os.path.join(GOLD, case + ".json")))
    assert header == meta["header"]
    assert [[s.scales_bytes, s.index_bytes, s.payload_bytes] for s in sizes] == meta["sizes"]
    assert ratio == pytest.approx(meta["ratio"], rel=1e-12)


def _blob(case="dzdl_b4"):
    return open(os.path.join(GOLD, case + ".dzdl"), "rb").read()


def test_bad_magic(F, tmp_path):
    p = tmp_path / "bad.dzdl"
    p.write_bytes(b"NOPE" + bytes(64))
    with pytest.raises(F.FormatError, match="magic"):
        F.read_delta(p)


def test_truncation_reports_offset(F, tmp_path):
    blob = _blob()
    for cut in (len(blob) - 10, 30, 6):
        p = tmp_path / f"cut{cut}.dzdl"
        p.write_bytes(blob[:cut])
        with pytest.raises(F.FormatError, match="offset") as ei:
            F.read_delta(p)
        assert ei.value.offset is not None and ei.value.offset <= cut


def test_trailing_bytes(F, tmp_path):
    p = tmp_path / "t.dzdl"
    p.write_bytes(_blob() + b"xx")
    with pytest.raises(F.FormatError, match="trailing"):
        F.read_delta(p)


def test_unsupported_version(F, tmp_path):
    b = bytearray(_blob())
    b[4] = 7
    p = tmp_path / "v.dzdl"
    p.write_bytes(bytes(b))
    with pytest.raises(F.FormatError, match="version"):
        F.read_delta(p)


def test_corrupt_deflate_stream(F, tmp_path):
    cd = F.read_delta(os.path.join(GOLD, "dzdl_b4_deflate.dzdl"))
    blob = bytearray(_blob("dzdl_b4_deflate"))
    # flip bytes inside the first layer's payload (after its 4-byte length)
    from paper_2312_05215_b200 import _lib as L
    import ctypes as C
    info, off = L.DzDzdlInfo(), C.c_int64(0)
    arr = np.frombuffer(bytes(blob), np.uint8)
    assert L.lib().dz_dzdl_parse_header(arr.ctypes.data, arr.size, C.byref(info), C.byref(off)) == 0
    recs = (L.DzDzdlLayer * len(cd.layers))()
    assert L.lib().dz_dzdl_parse_layers(arr.ctypes.data, arr.size, info.layers_off, len(cd.layers), recs,
                                        C.byref(off)) == 0
    o = recs[0].payload_off + 10
    blob[o:o + 8] = b"\xff" * 8
    p = tmp_path / "z.dzdl"
    p.write_bytes(bytes(blob))
    with pytest.raises(F.FormatError, match="lossless"):
        F.read_delta(p)


def test_bad_header_json(F, tmp_path):
    b = bytearray(_blob())
    b[12] = ord("!")
    p = tmp_path / "j.dzdl"
    p.write_bytes(bytes(b))
    with pytest.raises(F.FormatError, match="header"):
        F.read_delta(p)


def test_compress_config_validation_matches_reference():
    """CompressConfig rejects what the reference rejects (compress.py:52-69)."""
    import pytest as _pt
    from paper_2312_05215_b200.formats import CompressConfig
    for kw in [dict(bits=5), dict(sparsity="1:4"), dict(group_size=0), dict(block_size=0),
               dict(block_size=6), dict(damping=-1.0), dict(lossless="lz4"), dict(solver="gptq")]:
        with _pt.raises(ValueError):
            CompressConfig(**kw)
    assert CompressConfig(bits=16).is_passthrough and not CompressConfig().is_passthrough
    CompressConfig(sparsity="none", block_size=6)  # block size only constrained under 2:4


def test_solver_output_sizes_match_reference_fixtures():
    """The GPU solver's output buffers are sized exactly like the reference's packed fields."""
    import os
    import numpy as np
    from paper_2312_05215_b200.formats import CompressConfig
    from paper_2312_05215_b200.solver import _n_words
    gold = os.path.join(os.path.dirname(__file__), "golden")
    for f in sorted(os.listdir(gold)):
        if not (f.startswith("obs_b") and f.endswith(".npz")):
            continue
        z = np.load(os.path.join(gold, f))
        bits, sp, gs, bs = (int(v) for v in z["cfg"])
        r, c = z["delta"].shape
        cfg = CompressConfig(bits=bits, sparsity="two_of_four" if sp else "none", group_size=gs, block_size=bs)
        assert _n_words(r, c, cfg) == z["packed"].size, f
        if sp:
            assert r * c // 8 + (1 if (r * c // 4) % 2 else 0) == z["index"].size, f


def test_write_delta_is_byte_identical_to_reference_files():
    """read_delta -> write_delta reproduces the reference's own DZDL files byte for byte."""
    import glob
    import os
    import tempfile
    from paper_2312_05215_b200.formats import read_delta, write_delta
    files = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "dzdl_*.dzdl")))
    assert files
    for f in files:
        cd = read_delta(f)
        with tempfile.TemporaryDirectory() as d:
            out = os.path.join(d, "x.dzdl")
            write_delta(cd, out)
            assert open(out, "rb").read() == open(f, "rb").read(), f


def test_inspect_delta_is_lenient_like_the_reference(F, tmp_path):
    """Reference inspect_delta (formats.py:189-218) checks only the magic and truncation: trailing
    bytes, an unknown version and out-of-range configuration values are reported, not rejected."""
    base = F.inspect_delta(os.path.join(GOLD, "dzdl_b4.dzdl"))
    p = tmp_path / "t.dzdl"
    p.write_bytes(_blob() + b"xx")
    header, sizes, _ = F.inspect_delta(p)
    assert header == base[0] and [s.payload_bytes for s in sizes] == [s.payload_bytes for s in base[1]]
    b = bytearray(_blob())
    b[4] = 7  # version 7
    p.write_bytes(bytes(b))
    assert F.inspect_delta(p)[0] == base[0]
    blob = _blob()
    hlen = int.from_bytes(blob[8:12], "little")
    hdr = json.loads(blob[12:12 + hlen])
    hdr["bits"] = 5  # CompressConfig would reject it; inspect does not validate
    hb = json.dumps(hdr, sort_keys=True).encode()
    p.write_bytes(blob[:8] + len(hb).to_bytes(4, "little") + hb + blob[12 + hlen:])
    assert F.inspect_delta(p)[0]["bits"] == 5
    with pytest.raises(F.FormatError, match="magic"):
        p.write_bytes(b"NOPE" + blob[4:])
        F.inspect_delta(p)
    p.write_bytes(blob[: len(blob) - 5])
    with pytest.raises(F.FormatError) as ei:
        F.inspect_delta(p)
    assert ei.value.offset is not None
