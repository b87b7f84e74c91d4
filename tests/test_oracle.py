"""Pin the CPU oracle against the reference's golden vectors and KATs (CPU only)."""

import os

import numpy as np
import pytest

import oracle as O
from conftest import golden_files, load_ld_fields


def _od(z, prefix=""):
    return O.OracleDelta(**load_ld_fields(z, prefix))


def test_pack_kats(kat):
    # pkg/tests/test_compress.py:126-134
    assert O.pack_codes([-7, 0, 7, 1, 2, 3, -1, -2], 4).tolist() == kat["pack_spec_word"] == [0x56A98E70]
    assert O.pack_codes([0] * 8, 4).tolist() == kat["pack_zero_word"] == [0x77777777]


def test_survey_kat(kat):
    keep = np.zeros((2, 8), dtype=bool)
    keep[0, [0, 1, 6, 7]] = True
    keep[1, [0, 3, 5, 6]] = True
    idx = O.encode_mask_indices(keep)
    assert idx.hex() == kat["survey_index_hex"] == "e49c"
    words = O.pack_codes([1, -2, 3, -7, 7, 0, -1, 2], 4)
    assert words.tolist() == kat["survey_packed"] == [0x967E0A58]
    ld = O.OracleDelta(2, 8, words, idx, np.array([0.5, 0.25], "<f4"), 4, O.SPARSITY_2_4, 128)
    assert np.array_equal(O.dequantize_layer(ld), np.array(kat["survey_dequant"]))


def test_group_by_delta_kat(kat):
    perm, groups = O.group_by_delta([2, 0, 2, 1])
    assert perm == kat["group_by_delta_perm"] == [2, 0, 3, 1]
    assert [list(g) for g in groups] == kat["group_by_delta_groups"]


def test_codec_round_trip():
    rng = np.random.default_rng(5)
    for bits in (2, 3, 4, 8, 16):
        q = (1 << (bits - 1)) - 1
        c = rng.integers(-q, q + 1, size=101)
        assert np.array_equal(O.unpack_codes(O.pack_codes(c, bits), bits, c.size), c)
    with pytest.raises(O.OracleError):
        O.pack_codes([8], 4)
    with pytest.raises(O.OracleError):
        O.unpack_codes(np.zeros(1, "<u4"), 4, 9)


def test_index_errors():
    with pytest.raises(O.OracleError) as e:
        O.decode_mask_indices(b"\x00", 4, 8)
    assert e.value.kind == "FormatError"
    with pytest.raises(O.OracleError):
        O.decode_mask_indices(bytes([0x33, 0x44]), 1, 16)  # p0 == p1


@pytest.mark.parametrize("path", golden_files("unpack_*.npz"), ids=os.path.basename)
def test_dequant_matches_reference(path):
    z = np.load(path)
    got = O.dequantize_layer(_od(z))
    assert got.dtype == np.float64
    assert np.array_equal(got, z["dequant"])


@pytest.mark.parametrize("path", golden_files("sbmm_*.npz"), ids=os.path.basename)
def test_sbmm_matches_reference(path):
    z = np.load(path)
    D = len([k for k in z.files if k.endswith("_meta")])
    deltas = {d: _od(z, f"d{d}_") for d in range(D)}
    rows = [(int(r), int(d), z["X"][i]) for i, (r, d) in enumerate(zip(z["rids"], z["ids"]))]
    out = O.sbmm(z["W"], deltas, rows)
    Y = np.stack([out[int(r)] for r in z["rids"]])
    assert np.array_equal(Y, z["Y"])  # same f64 ops in the same order
    perm, groups = O.group_by_delta(z["ids"].tolist())
    assert perm == z["perm"].tolist()
    assert [list(g) for g in groups] == z["groups"].tolist()
    Ym = O.sbmm_matrix(z["W"], deltas, z["ids"], z["X"])
    assert np.allclose(Ym, z["Y"], rtol=1e-12, atol=1e-12)


def test_tp_matches_reference():
    z = np.load(golden_files("tp_two_layer.npz")[0])
    for n in (1, 2, 4):
        y = O.tp_forward(O.tp_partition(z["w1"], "column", n), O.tp_partition(z["d1"], "column", n), z["x"], "column")
        zz = O.tp_forward(O.tp_partition(z["w2"], "row", n), O.tp_partition(z["d2"], "row", n), y, "row")
        assert np.array_equal(y, z[f"y{n}"])
        assert np.array_equal(zz, z[f"z{n}"])
    with pytest.raises(O.OracleError):
        O.tp_partition(np.zeros((2, 3)), "column", 2)


def test_random_packed_generator_is_reference_layout():
    rng = np.random.default_rng(3)
    for bits in (2, 3, 4):
        ld = O.random_packed_delta(rng, 6, 24, bits)
        dq = O.dequantize_layer(ld)
        assert dq.shape == (6, 24)
        assert ((dq != 0).reshape(6, 6, 4).sum(-1) <= 2).all()


def test_rtn_producer_round_trip():
    rng = np.random.default_rng(4)
    d = rng.normal(0, 0.02, (8, 256))
    ld = O.magnitude_rtn_2of4(d, 4)
    dq = O.dequantize_layer(ld)
    assert (((dq != 0).reshape(8, 64, 4).sum(-1)) <= 2).all()
    kept = dq != 0
    assert np.abs(dq - d)[kept].max() <= np.abs(d).max() / 7 / 2 + 1e-9


OBS_FILES = sorted(f for f in os.listdir(os.path.join(os.path.dirname(__file__), "golden"))
                   if f.startswith("obs_b") and f.endswith(".npz"))


@pytest.mark.parametrize("name", OBS_FILES)
def test_obs_solver_matches_reference(name):
    """The oracle's ΔCompress solver reproduces the reference's obs_compress_layer
    (compress.py:348-464) on its fixtures: same factor U, same packed bytes."""
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", name))
    bits, sp, gs, bs = (int(v) for v in z["cfg"])
    if not (bits == 16 and not sp):
        assert np.array_equal(O.inverse_cholesky_factor(z["hessian"]), z["u"])
    od, loss, quant = O.obs_compress_layer(z["delta"], z["hessian"], bits,
                                           O.SPARSITY_2_4 if sp else O.SPARSITY_NONE, gs, bs)
    assert np.array_equal(od.packed_values, z["packed"])
    assert od.index_stream == z["index"].tobytes()
    assert np.array_equal(od.scales, z["scales"])
    assert loss == pytest.approx(float(z["proxy_loss"]), rel=1e-12, abs=1e-300)
    assert np.array_equal(O.dequantize_layer(od), z["dequant"])
    assert np.array_equal(quant, z["dequant"])


def test_obs_model_hessian_matches_reference():
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "obs_model_2layer.npz"))
    h = O.compute_hessian(z["calib"], 0.01)
    u = O.inverse_cholesky_factor(h)
    d0 = z["wf0"] - z["wb0"]
    od, loss, _ = O.obs_compress_layer(d0, h, 4, O.SPARSITY_2_4, 32, 16, u=u)
    assert np.array_equal(od.packed_values, z["packed0"])
    assert loss == pytest.approx(float(z["loss0"]), rel=1e-12)
