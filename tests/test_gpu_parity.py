"""GPU parity: the CUDA path (through the C ABI) against the reference's golden vectors and the
CPU oracle. Bit-exact for the unpack (K1) and the re-layout; rel-err <= 1e-2 per token for
SBMM outputs (bf16 operands, fp32 accumulate vs the reference's f64, north star)."""

import os

import numpy as np
import pytest
import torch

import oracle as O
from conftest import golden_files, load_ld_fields

pytestmark = pytest.mark.gpu

REL_TOL = 1e-2  # north star: outputs within rel-err <= 1e-2 (bf16 vs the reference)


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2312_05215_b200 as P
    return P


def _ld(P, z, prefix=""):
    f = load_ld_fields(z, prefix)
    return P.LayerDelta(name="g", **f)


def rel_err_rows(Y, R):
    num = np.linalg.norm(Y - R, axis=-1)
    den = np.maximum(np.linalg.norm(R, axis=-1), 1e-30)
    return num / den


def bf16_round(a):
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().double().numpy()


# ------------------------------------------------------------------------------ K1 unpack


@pytest.mark.parametrize("path", golden_files("unpack_*.npz"), ids=os.path.basename)
def test_unpack_bit_exact(P, path):
    z = np.load(path)
    ld = _ld(P, z)
    ref = z["dequant"]
    got64 = P.dequantize_layer(ld)
    assert got64.dtype == np.float64 and np.array_equal(got64, ref)
    got32 = P.dequantize_layer_device(ld, torch.float32).cpu().numpy()
    assert np.array_equal(got32.view(np.uint32), ref.astype(np.float32).view(np.uint32))
    gotbf = P.dequantize_layer_device(ld, torch.bfloat16).cpu()
    assert torch.equal(gotbf.view(torch.int16), torch.from_numpy(ref).to(torch.bfloat16).view(torch.int16))


def _sparse_native_fixture(path):
    """2:4 with 2/3/4-bit codes and gs % 128 == 0 (or one group per row): the native-block layout
    (engine.NativeDelta.sparse_native_ok); the other fixtures are served through the dense path."""
    rows, cols, bits, sparse, gs = (int(v) for v in np.load(path)["meta"])
    return sparse and bits in (2, 3, 4) and (gs % 128 == 0 or -(-cols // gs) == 1)


@pytest.mark.parametrize("path", [p for p in golden_files("unpack_*.npz") if _sparse_native_fixture(p)],
                         ids=os.path.basename)
def test_native_relayout_lossless(P, path):
    from paper_2312_05215_b200.engine import NativeDelta
    z = np.load(path)
    ld = _ld(P, z)
    assert NativeDelta.sparse_native_ok(ld)
    nat = NativeDelta.from_layer_delta(ld)
    got = nat.to_dense_f32().cpu().numpy()
    assert np.array_equal(got, z["dequant"].astype(np.float32))


def test_codec_pieces(P):
    rng = np.random.default_rng(5)
    for bits in (2, 3, 4, 8, 16):
        q = (1 << (bits - 1)) - 1
        c = rng.integers(-q, q + 1, size=1001)
        assert np.array_equal(P.unpack_codes(O.pack_codes(c, bits), bits, c.size), c)
    with pytest.raises(P.EncodingError):
        P.unpack_codes(np.zeros(1, "<u4"), 4, 9)
    keep = np.zeros((5, 12), dtype=bool)
    for r in range(5):
        for g in range(3):
            keep[r, 4 * g + rng.choice(4, 2, replace=False)] = True
    assert np.array_equal(P.decode_mask_indices(O.encode_mask_indices(keep), 5, 12), keep)
    with pytest.raises(P.FormatError):
        P.decode_mask_indices(b"\x00", 4, 8)
    with pytest.raises(P.FormatError):
        P.decode_mask_indices(bytes([0x33, 0x44]), 1, 16)


def test_corrupt_index_raises_format_error(P):
    from paper_2312_05215_b200.engine import NativeDelta
    ld = O.random_packed_delta(np.random.default_rng(1), 16, 256, 4)
    bad = bytearray(ld.index_stream)
    bad[37] = (bad[37] & 0xF0) | 0x3  # p0=3 >= p1=0
    lb = P.LayerDelta(name="bad", rows=16, cols=256, packed_values=ld.packed_values, index_stream=bytes(bad),
                      scales=ld.scales, bits=4, sparsity="two_of_four", group_size=128)
    with pytest.raises(P.FormatError):
        P.dequantize_layer(lb)
    with pytest.raises(P.FormatError):
        NativeDelta.from_layer_delta(lb)
    with pytest.raises(P.FormatError):
        P.sbmm(np.zeros((16, 256)), {0: lb}, P.BatchInput([(0, 0, np.ones(256))]))
    short = P.LayerDelta(name="s", rows=16, cols=256, packed_values=ld.packed_values[:10],
                         index_stream=ld.index_stream, scales=ld.scales, bits=4, sparsity="two_of_four",
                         group_size=128)
    with pytest.raises(P.EncodingError):
        P.dequantize_layer(short)


# ------------------------------------------------------------------------------ K2 SBMM


@pytest.mark.parametrize("path", golden_files("sbmm_*.npz"), ids=os.path.basename)
def test_sbmm_matches_reference_golden(P, path):
    z = np.load(path)
    D = len([k for k in z.files if k.endswith("_meta")])
    deltas = {d: _ld(P, z, f"d{d}_") for d in range(D)}
    rows = [(int(r), int(d), z["X"][i]) for i, (r, d) in enumerate(zip(z["rids"], z["ids"]))]
    out = P.sbmm(z["W"], deltas, P.BatchInput(rows))
    Y = np.stack([out[int(r)] for r in z["rids"]])
    err = rel_err_rows(Y, z["Y"])
    assert err.max() <= REL_TOL, err.max()
    perm, groups = P.group_by_delta(P.BatchInput(rows))
    assert perm == z["perm"].tolist()
    assert [list(g) for g in groups] == z["groups"].tolist()


def test_sbmm_batch_invariance(P):
    """test_inference.py:105-147 / 233-245 and acceptance 5: bit-exact vs per-request loop."""
    z = np.load(golden_files("sbmm_cfg1_mini.npz")[0])
    deltas = {d: _ld(P, z, f"d{d}_") for d in range(4)}
    rows = [(int(r), int(d), z["X"][i]) for i, (r, d) in enumerate(zip(z["rids"], z["ids"]))]
    out = P.sbmm(z["W"], deltas, P.BatchInput(rows))
    for rid, did, x in rows[:6]:
        solo = P.sbmm(z["W"], {did: deltas[did]}, P.BatchInput([(rid, did, x)]))
        assert np.array_equal(out[rid], solo[rid])
        assert np.array_equal(out[rid], P.decoupled_linear(z["W"], deltas[did], x))
    shuffled = [rows[i] for i in np.random.default_rng(3).permutation(len(rows))]
    out2 = P.sbmm(z["W"], deltas, P.BatchInput(shuffled))
    for rid in out:
        assert np.array_equal(out[rid], out2[rid])


def test_sbmm_reference_test_cases(P):
    # test_inference.py:51-58 hand example (bits=16 dense passthrough) and unused/unknown deltas
    ld = P.LayerDelta(name="h", rows=2, cols=2, packed_values=O.float64_payload(np.array([[0.5, 0.0], [0.0, 0.0]])),
                      index_stream=b"", scales=np.zeros(0, "<f4"), bits=16, sparsity="none", group_size=128)
    out = P.decoupled_linear(np.eye(2), ld, np.array([1.0, 2.0]))
    assert np.allclose(out, [1.5, 2.0], rtol=1e-2)
    z4 = O.random_packed_delta(np.random.default_rng(0), 4, 8, 4)
    lz = P.LayerDelta(name="z", rows=4, cols=8, packed_values=z4.packed_values, index_stream=z4.index_stream,
                      scales=z4.scales, bits=4, sparsity="two_of_four", group_size=128)
    out = P.sbmm(np.eye(4, 8), {0: lz, 1: lz}, P.BatchInput([(0, 0, np.ones(8))]))
    assert set(out) == {0}
    with pytest.raises(P.UnknownDeltaError):
        P.sbmm(np.eye(4, 8), {0: lz}, P.BatchInput([(0, 9, np.ones(8))]))
    with pytest.raises(P.ShapeError):
        P.decoupled_linear(np.eye(3), lz, np.ones(3))
    # matrix input (in, n) to decoupled_linear
    xm = np.random.default_rng(2).normal(size=(8, 3))
    ym = P.decoupled_linear(np.eye(4, 8), lz, xm)
    ref = O.decoupled_linear(np.eye(4, 8), z4, bf16_round(xm))
    assert ym.shape == (4, 3)
    assert np.abs(ym - ref).max() <= REL_TOL * np.abs(ref).max()


def _random_case(P, rng, rows, cols, bits, D, T, gs=128, sparse=True):
    W = bf16_round(rng.normal(0, 1 / np.sqrt(cols), size=(rows, cols)))
    ods = {d: O.random_packed_delta(rng, rows, cols, bits, gs, sparse) for d in range(D)}
    pds = {d: P.LayerDelta(name=f"d{d}", rows=rows, cols=cols, packed_values=o.packed_values,
                           index_stream=o.index_stream, scales=o.scales, bits=bits, sparsity=o.sparsity,
                           group_size=gs) for d, o in ods.items()}
    X = bf16_round(rng.normal(0, 1, size=(T, cols)))
    ids = rng.integers(0, D, size=T)
    return W, ods, pds, X, ids


@pytest.mark.parametrize("rows,cols,bits,D,T,gs,sparse", [
    (256, 512, 4, 5, 37, 128, True),     # T not a multiple of 8, several deltas
    (100, 384, 2, 3, 20, 128, True),     # rows not multiple of 16, 2-bit
    (48, 200, 4, 2, 9, 128, True),       # cols not multiple of 128 (padded X path)
    (64, 256, 3, 2, 17, 128, True),      # 3-bit served as 4-bit fields
    (64, 512, 4, 2, 12, 256, True),      # group_size 256 (scale spans two blocks)
    (32, 256, 4, 2, 10, 64, True),       # group_size 64 -> dense path
    (32, 256, 8, 2, 10, 128, True),      # 8-bit 2:4 -> dense path
    (32, 256, 4, 2, 10, 128, False),     # dense (no 2:4) -> dense path
    (128, 256, 4, 1, 150, 128, True),    # one delta, T > 64 (several base and delta jobs)
])
def test_sbmm_vs_oracle(P, rows, cols, bits, D, T, gs, sparse):
    rng = np.random.default_rng(rows * 7 + cols + bits + T)
    W, ods, pds, X, ids = _random_case(P, rng, rows, cols, bits, D, T, gs, sparse)
    rows_in = [(i, int(d), X[i]) for i, d in enumerate(ids)]
    out = P.sbmm(W, pds, P.BatchInput(rows_in))
    Y = np.stack([out[i] for i in range(T)])
    R = O.sbmm_matrix(W, ods, ids, X)
    err = rel_err_rows(Y, R)
    assert err.max() <= REL_TOL, err.max()


def test_fused_kernel_mixed_table_and_no_base(P):
    """Sparse4 + sparse2 + dense deltas routed in one launch; and the delta-only path (no base)."""
    from paper_2312_05215_b200.engine import DeltaTable, NativeBase, NativeDelta, Plan, sbmm_forward
    rng = np.random.default_rng(9)
    rows, cols, T = 160, 384, 40
    W = bf16_round(rng.normal(0, 0.05, (rows, cols)))
    ods = [O.random_packed_delta(rng, rows, cols, 4), O.random_packed_delta(rng, rows, cols, 2),
           O.random_packed_delta(rng, rows, cols, 8)]
    nat = [NativeDelta.from_layer_delta(o) for o in ods]
    assert [n.kind for n in nat] == [1, 2, 3]
    table = DeltaTable(nat, rows, cols)
    ids = rng.integers(0, 3, T).astype(np.int32)
    X = bf16_round(rng.normal(0, 1, (T, cols)))
    Xd = torch.from_numpy(X.astype(np.float32)).cuda().to(torch.bfloat16)
    base = NativeBase(torch.from_numpy(W.astype(np.float32)).cuda().to(torch.bfloat16))
    for with_base in (True, False):
        plan = Plan(ids, table.kinds, 3, with_base=with_base)
        Y = sbmm_forward(Xd, plan, base if with_base else None, table, y_dtype=torch.float32).cpu().double().numpy()
        R = O.sbmm_matrix(W if with_base else np.zeros_like(W), dict(enumerate(ods)), ids, X)
        assert rel_err_rows(Y, R).max() <= REL_TOL


def test_fused_kernel_repeat_launches_deterministic(P):
    """Self-resetting scheduler/tile counters: many back-to-back launches, identical results."""
    from paper_2312_05215_b200.engine import DeltaTable, NativeBase, NativeDelta, Plan, sbmm_forward
    rng = np.random.default_rng(4)
    rows, cols, T, D = 512, 1024, 64, 8
    nat = [NativeDelta.from_layer_delta(O.random_packed_delta(rng, rows, cols, 4)) for _ in range(D)]
    table = DeltaTable(nat, rows, cols)
    base = NativeBase(torch.randn(rows, cols, device="cuda").to(torch.bfloat16))
    plan = Plan(rng.integers(0, D, T), table.kinds, D)
    X = torch.randn(T, cols, device="cuda").to(torch.bfloat16)
    Y0 = sbmm_forward(X, plan, base, table).clone()
    for grid in (0, 1, 7, 300):
        for _ in range(5):
            Y = sbmm_forward(X, plan, base, table, grid=grid)
            assert torch.equal(Y, Y0)


def test_tp_forward_golden(P):
    z = np.load(golden_files("tp_two_layer.npz")[0])
    for n in (1, 2, 4):
        y = P.tp_forward(P.tp_partition(z["w1"], "column", n), P.tp_partition(z["d1"], "column", n), z["x"],
                         "column")
        zz = P.tp_forward(P.tp_partition(z["w2"], "row", n), P.tp_partition(z["d2"], "row", n), bf16_round(y), "row")
        assert np.linalg.norm(y - z[f"y{n}"]) / np.linalg.norm(z[f"y{n}"]) <= REL_TOL
        assert np.linalg.norm(zz - z[f"z{n}"]) / np.linalg.norm(z[f"z{n}"]) <= 2 * REL_TOL
    with pytest.raises(P.PartitionError):
        P.tp_forward(P.tp_partition(np.zeros((4, 4)), "column", 2), P.tp_partition(np.zeros((4, 4)), "column", 2),
                     np.zeros((2, 3)), "column")


def test_forward_model_vs_oracle(P):
    rng = np.random.default_rng(21)
    dim, nl = 256, 3
    Ws = [bf16_round(rng.normal(0, 1 / np.sqrt(dim), (dim, dim))) for _ in range(nl)]
    stack = P.WeightStack([(f"l{i}", w) for i, w in enumerate(Ws)], axes=["column", "row", "column"])
    ods = {d: [O.random_packed_delta(rng, dim, dim, 4) for _ in range(nl)] for d in range(3)}
    handles = {d: P.DeltaHandle(d, [P.LayerDelta(name=f"l{i}", rows=dim, cols=dim, packed_values=o.packed_values,
                                                 index_stream=o.index_stream, scales=o.scales, bits=4,
                                                 sparsity="two_of_four", group_size=128)
                                    for i, o in enumerate(lst)]) for d, lst in ods.items()}
    rows = [(i, i % 3, bf16_round(rng.normal(size=dim))) for i in range(7)]
    out = P.forward_model(stack, handles, P.BatchInput(rows))
    ref = O.forward_model(Ws, ods, rows)
    for rid, _, _ in rows:
        assert np.linalg.norm(out[rid] - ref[rid]) / np.linalg.norm(ref[rid]) <= 2 * REL_TOL
    tp = P.forward_model(stack, handles, P.BatchInput(rows), layout=P.TpLayout(2, ("column", "row", "column")))
    for rid, _, _ in rows:
        assert np.linalg.norm(tp[rid] - ref[rid]) / np.linalg.norm(ref[rid]) <= 2 * REL_TOL
    # mixed batch == solo forwards (test_inference.py:233-245), bit-exact
    for rid, did, x in rows[:3]:
        solo = P.forward_model(stack, {did: handles[did]}, P.BatchInput([(rid, did, x)]))
        assert np.array_equal(out[rid], solo[rid])


@pytest.mark.slow
@pytest.mark.parametrize("out_f,in_f,bits", [(4096, 4096, 4), (11008, 4096, 4), (4096, 11008, 4), (5120, 5120, 2)])
def test_full_size_llama_linear(P, out_f, in_f, bits):
    """BASELINE shapes at decode batch 64 with 32 deltas: fused kernel vs an independent fp32 torch
    reference built from the bit-exact K1 unpack, plus the oracle on a few tokens."""
    from paper_2312_05215_b200.engine import DeltaTable, NativeBase, NativeDelta, Plan, sbmm_forward
    rng = np.random.default_rng(out_f + in_f + bits)
    D, T = 32, 64
    ods = [O.random_packed_delta(rng, out_f, in_f, bits) for _ in range(D)]
    nat = [NativeDelta.from_layer_delta(o) for o in ods]
    table = DeltaTable(nat, out_f, in_f)
    Wt = (torch.randn(out_f, in_f, device="cuda") / np.sqrt(in_f)).to(torch.bfloat16)
    base = NativeBase(Wt)
    ids = rng.permutation([i % D for i in range(T)]).astype(np.int32)
    X = torch.randn(T, in_f, device="cuda").to(torch.bfloat16)
    Y = sbmm_forward(X, Plan(ids, table.kinds, D), base, table, y_dtype=torch.float32)
    R = X.float() @ Wt.float().T
    for d in range(D):
        sel = torch.from_numpy(np.nonzero(ids == d)[0]).cuda()
        dq = P.dequantize_layer_device(ods[d], torch.float32)
        R[sel] += X[sel].float() @ dq.T
    err = (torch.linalg.norm(Y - R, dim=1) / torch.linalg.norm(R, dim=1)).max().item()
    assert err <= REL_TOL, err
    # oracle (f64 CPU) on 2 tokens
    Xh = X[:2].float().double().cpu().numpy()
    Wh = Wt.float().double().cpu().numpy()
    Ro = O.sbmm_matrix(Wh, dict(enumerate(ods)), ids[:2], Xh)
    assert rel_err_rows(Y[:2].double().cpu().numpy(), Ro).max() <= REL_TOL


def test_sbmm_api_large_group_batch_invariant(P):
    """The drop-in `sbmm` (inference.py:126-154) on a batch whose main group is far above the
    engine's prefill threshold stays on the decode kernel (pf_min=0): it matches the reference
    oracle, and every row equals its solo `decoupled_linear` call bit for bit (the reference's
    batch invariance, test_inference.py:105-147)."""
    from paper_2312_05215_b200.engine import PF_MIN
    rng = np.random.default_rng(31)
    W, ods, pds, X, _ = _random_case(P, rng, 192, 384, 4, 3, 8)
    ids = np.concatenate([np.zeros(PF_MIN + 50, np.int64), rng.integers(1, 3, 20)])
    X = bf16_round(rng.normal(0, 1, size=(ids.size, 384)))
    out = P.sbmm(W, pds, P.BatchInput([(i, int(d), X[i]) for i, d in enumerate(ids)]))
    Y = np.stack([out[i] for i in range(ids.size)])
    R = O.sbmm_matrix(W, ods, ids, X)
    assert rel_err_rows(Y, R).max() <= REL_TOL
    for i in (0, 1, PF_MIN + 49, ids.size - 1):
        assert np.array_equal(out[i], P.decoupled_linear(W, pds[int(ids[i])], X[i])), i
