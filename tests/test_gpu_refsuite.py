"""The reference's own hot-path test suite, run against this package.

Mirrors /root/reference/pkg/tests/test_inference.py (classes TestDecoupledLinear .. TestForwardModel,
same test names) and acceptance criteria 5 and 6 (test_acceptance.py:149-182). The operands are
the reference tests' own: `tests/golden/make_refsuite.py` ran the reference with the tests' seeds
(Philox `Rng`, OBS-compressed deltas, compress_model outputs) and stored inputs and reference
outputs in `tests/golden/refsuite.npz`.

What changes against the reference suite:
  * numeric tolerances: the reference's f64 bounds (<= 1e-9 / 1e-12 / allclose) become a relative
    error <= 1e-2 per output vector (north star: bf16 operands, fp32 accumulation);
  * the reference's bit-exactness contracts (sbmm == per-request decoupled_linear, row-order
    invariance, mixed batch == solo forwards) are kept bit for bit, evaluated on this package's
    own outputs;
  * everything else (exception types, group_by_delta permutations, partition shapes) is exact.
"""

import os

import numpy as np
import pytest
import torch

from conftest import ROOT, load_ld_fields

REL = 1e-2
GPU = pytest.mark.gpu


@pytest.fixture(scope="module")
def Z():
    return np.load(os.path.join(ROOT, "tests", "golden", "refsuite.npz"))


@pytest.fixture(scope="module")
def P():
    import paper_2312_05215_b200 as P
    return P


@pytest.fixture(scope="module")
def G(P):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return P


def ld(P, Z, key):
    return P.LayerDelta(name=key, **load_ld_fields(Z, key + "_"))


def rel(y, r):
    y, r = np.atleast_2d(np.asarray(y, np.float64).T).T, np.atleast_2d(np.asarray(r, np.float64).T).T
    return float((np.linalg.norm(y - r, axis=0) / np.maximum(np.linalg.norm(r, axis=0), 1e-30)).max())


# ------------------------------------------------------------------ test_inference.py:43-70


@GPU
class TestDecoupledLinear:
    def test_zero_delta(self, G, Z):
        w, x = Z["dl_zero_w"], Z["dl_zero_x"]
        out = G.decoupled_linear(w, ld(G, Z, "dl_zero_ld"), x)
        assert out.shape == (8, 3) and rel(out, w @ x) <= REL

    def test_hand_example(self, G, Z):
        out = G.decoupled_linear(np.eye(2), ld(G, Z, "dl_hand_ld"), np.array([1.0, 2.0]))
        assert np.allclose(out, [1.5, 2.0])  # the reference's own tolerance: all values are bf16-exact

    def test_merged_oracle(self, G, Z):
        for t in range(30):
            out = G.decoupled_linear(Z[f"dl_merged{t}_w"], ld(G, Z, f"dl_merged{t}_ld"), Z[f"dl_merged{t}_x"])
            assert rel(out, Z[f"dl_merged{t}_ref"]) <= REL, t

    def test_shape_error(self, G, Z):
        with pytest.raises(G.ShapeError):  # the reference raises inside _zero_delta(2, 2) already
            G.obs_compress_layer(np.zeros((2, 2)), np.eye(2), G.CompressConfig(bits=4, sparsity=G.SPARSITY_2_4))
        with pytest.raises(G.ShapeError):
            G.decoupled_linear(np.eye(3), ld(G, Z, "sb_zero4"), np.ones(3))


# ------------------------------------------------------------------ test_inference.py:73-102 (host)


class TestGroupByDelta:
    def test_spec_example(self, P):
        perm, groups = P.group_by_delta(P.BatchInput([(i, d, np.zeros(2)) for i, d in enumerate([2, 0, 2, 1])]))
        assert perm == [2, 0, 3, 1]
        assert groups == [(0, 0, 1), (1, 1, 2), (2, 2, 4)]

    def test_single_delta_identity(self, P):
        perm, groups = P.group_by_delta(P.BatchInput([(i, 5, np.zeros(2)) for i in range(4)]))
        assert perm == [0, 1, 2, 3] and groups == [(5, 0, 4)]

    def test_empty(self, P):
        assert P.group_by_delta(P.BatchInput([])) == ([], [])

    def test_stable_sort_oracle(self, P):
        rng = np.random.default_rng(17)
        for _ in range(50):
            ids = rng.integers(0, 5, size=int(rng.integers(0, 12))).tolist()
            perm, _ = P.group_by_delta(P.BatchInput([(i, d, np.zeros(1)) for i, d in enumerate(ids)]))
            expected = sorted(range(len(ids)), key=lambda i: ids[i])
            assert all(expected[pos] == orig for orig, pos in enumerate(perm))


# ------------------------------------------------------------------ test_inference.py:105-147


@GPU
class TestSbmm:
    def test_singleton_reduces_to_decoupled(self, G, Z):
        w, x, d = Z["sb_single_w"], Z["sb_single_x"], ld(G, Z, "sb_single_ld")
        out = G.sbmm(w, {7: d}, G.BatchInput([(42, 7, x)]))
        assert np.array_equal(out[42], G.decoupled_linear(w, d, x))

    def test_multi_delta_bit_exact_loop_oracle(self, G, Z):
        w = Z["sb_multi_w"]
        deltas = {d: ld(G, Z, f"sb_multi_d{d}") for d in range(3)}
        rows = [(int(r), int(d), x) for (r, d), x in zip(Z["sb_multi_rows"], Z["sb_multi_x"])]
        out = G.sbmm(w, deltas, G.BatchInput(rows))
        for (rid, did, x), ref in zip(rows, Z["sb_multi_ref"]):
            assert np.array_equal(out[rid], G.decoupled_linear(w, deltas[did], x))
            assert rel(out[rid], ref) <= REL

    def test_unused_delta_ok(self, G, Z):
        deltas = {0: ld(G, Z, "sb_zero4"), 1: ld(G, Z, "sb_zero4")}
        out = G.sbmm(np.eye(4) * 0.5, deltas, G.BatchInput([(0, 0, np.ones(4))]))
        assert set(out) == {0}

    def test_unknown_delta(self, G, Z):
        with pytest.raises(G.UnknownDeltaError):
            G.sbmm(np.eye(4), {0: ld(G, Z, "sb_zero4")}, G.BatchInput([(0, 9, np.ones(4))]))

    def test_order_preservation(self, G, Z):
        w = Z["sb_order_w"]
        deltas = {d: ld(G, Z, f"sb_order_d{d}") for d in range(2)}
        rows = [(i, i % 2, Z["sb_order_x"][i]) for i in range(5)]
        out = G.sbmm(w, deltas, G.BatchInput(rows))
        out2 = G.sbmm(w, deltas, G.BatchInput([rows[i] for i in (3, 0, 4, 2, 1)]))
        for rid in out:
            assert np.array_equal(out[rid], out2[rid])

    def test_duplicate_request_ids(self, G, Z):
        """Reference semantics (inference.py:153-154): one key per id, the last row in sorted
        order wins."""
        deltas = {d: ld(G, Z, f"fm_mixed_d{d}_l0") for d in range(3)}
        rows = [(int(r), int(d), x) for (r, d), x in zip(Z["fm_dup_rows"], Z["fm_dup_x"])]
        out = G.sbmm(Z["fm_mixed_base_w"][0], deltas, G.BatchInput(rows))
        assert list(out) == [7, 8]
        assert rel(out[7], Z["sb_dup_ref"][0]) <= REL and rel(out[8], Z["sb_dup_ref"][1]) <= REL


# ------------------------------------------------------------------ test_inference.py:150-186


class TestTpPartition:
    def test_column_split(self, P):
        shards = P.tp_partition(np.arange(4.0).reshape(2, 2), "column", 2)
        assert len(shards) == 2 and shards[0].shape == (2, 1)

    def test_row_split(self, P):
        shards = P.tp_partition(np.arange(8.0).reshape(4, 2), "row", 2)
        assert len(shards) == 2 and shards[0].shape == (2, 2)

    def test_not_divisible(self, P):
        with pytest.raises(P.PartitionError):
            P.tp_partition(np.zeros((2, 3)), "column", 2)


@GPU
class TestTpForward:
    def test_single_worker_matches_decoupled(self, G, Z):
        w, x, d = Z["tp_single_w"], Z["tp_single_x"], ld(G, Z, "tp_single_ld")
        dq = G.dequantize_layer(d)
        out = G.tp_forward(G.tp_partition(w.T, "column", 1), G.tp_partition(dq.T, "column", 1), x.T, "column")
        assert rel(out.T, G.decoupled_linear(w, d, x)) <= REL

    @pytest.mark.parametrize("n", [1, 2, 4])
    def test_two_layer_stack_equivalence(self, G, Z, n):
        k = lambda s: Z[f"tp_stack{n}_{s}"]  # noqa: E731
        y = G.tp_forward(G.tp_partition(k("w1"), "column", n), G.tp_partition(k("d1"), "column", n), k("x"), "column")
        z = G.tp_forward(G.tp_partition(k("w2"), "row", n), G.tp_partition(k("d2"), "row", n), y, "row")
        assert np.linalg.norm(z - k("ref")) / np.linalg.norm(k("ref")) <= REL

    def test_zero_delta_shards(self, G, Z):
        w, x = Z["tp_zero_w"], Z["tp_zero_x"]
        out = G.tp_forward(G.tp_partition(w, "column", 2), G.tp_partition(np.zeros_like(w), "column", 2), x, "column")
        assert rel(out.T, (x @ w).T) <= REL

    def test_layout_mismatch(self, G):
        w = np.zeros((4, 4))
        with pytest.raises(G.PartitionError):
            G.tp_forward(G.tp_partition(w, "column", 2), G.tp_partition(w, "column", 2), np.zeros((2, 3)), "column")


# ------------------------------------------------------------------ test_inference.py:202-256


def _stack(P, Z, key):
    ws = Z[f"{key}_w"]
    return P.WeightStack([(f"l{i}", ws[i]) for i in range(ws.shape[0])])


@GPU
class TestForwardModel:
    def test_zero_deltas_match_base_forward(self, G, Z):
        base = _stack(G, Z, "fm_zero_base")
        handles = {0: G.DeltaHandle(0, [ld(G, Z, "fm_zero_ld") for _ in range(3)])}
        out = G.forward_model(base, handles, G.BatchInput([(0, 0, Z["fm_zero_x"])]))
        assert rel(out[0], Z["fm_zero_ref"]) <= REL

    def test_lossless_delta_matches_finetuned_forward(self, G, Z):
        base = _stack(G, Z, "fm_lossless_base")
        handles = {0: G.DeltaHandle(0, [ld(G, Z, f"fm_lossless_l{i}") for i in range(3)])}
        out = G.forward_model(base, handles, G.BatchInput([(0, 0, Z["fm_lossless_x"])]))
        assert rel(out[0], Z["fm_lossless_ref"]) <= REL

    def _mixed(self, G, Z):
        base = _stack(G, Z, "fm_mixed_base")
        handles = {d: G.DeltaHandle(d, [ld(G, Z, f"fm_mixed_d{d}_l{i}") for i in range(3)]) for d in range(3)}
        return base, handles

    def test_mixed_batch_equals_independent_forwards(self, G, Z):
        base, handles = self._mixed(G, Z)
        rows = [(i, i % 3, Z["fm_mixed_x"][i]) for i in range(6)]
        out = G.forward_model(base, handles, G.BatchInput(rows))
        for (rid, did, x), ref in zip(rows, Z["fm_mixed_ref"]):
            solo = G.forward_model(base, {did: handles[did]}, G.BatchInput([(rid, did, x)]))
            assert np.array_equal(out[rid], solo[rid])
            assert rel(out[rid], ref) <= REL

    def test_duplicate_request_ids(self, G, Z):
        """inference.py:264-291: rows of one id all read current[rid] and the last delta-sorted row
        survives each layer — compared with the reference's own output on the same rows."""
        base, handles = self._mixed(G, Z)
        rows = [(int(r), int(d), x) for (r, d), x in zip(Z["fm_dup_rows"], Z["fm_dup_x"])]
        out = G.forward_model(base, handles, G.BatchInput(rows))
        assert list(out) == [7, 8]
        assert rel(out[7], Z["fm_dup_ref"][0]) <= REL and rel(out[8], Z["fm_dup_ref"][1]) <= REL

    def test_tp_layout_equivalence(self, G, Z):
        base = _stack(G, Z, "fm_tp_base")
        handles = {0: G.DeltaHandle(0, [ld(G, Z, f"fm_tp_l{i}") for i in range(2)])}
        batch = G.BatchInput([(0, 0, Z["fm_tp_x"])])
        plain = G.forward_model(base, handles, batch)
        tp = G.forward_model(base, handles, batch, layout=G.TpLayout(2, ("column", "row")))
        assert rel(plain[0], tp[0]) <= REL
        assert rel(plain[0], Z["fm_tp_ref"]) <= REL and rel(tp[0], Z["fm_tp_ref_tp2"]) <= REL


# ------------------------------------------------------------------ test_acceptance.py:149-182


@GPU
def test_criterion_5_decoupling_exactness(G, Z):
    """100 trials: grouped sbmm within 1e-2 of the merged weight's product (reference: 1e-9) and
    bit-exact against this package's per-request decoupled_linear (reference: bit-exact)."""
    for t in range(100):
        base = Z[f"acc5_{t}_base"]
        deltas = {d: ld(G, Z, f"acc5_{t}_d{d}") for d in range(3)}
        rows = [(j, j % 3, Z[f"acc5_{t}_x"][j]) for j in range(6)]
        out = G.sbmm(base, deltas, G.BatchInput(rows))
        for (rid, did, x), merged in zip(rows, Z[f"acc5_{t}_merged"]):
            assert rel(out[rid], merged) <= REL, (t, rid)
            assert np.array_equal(out[rid], G.decoupled_linear(base, deltas[did], x)), (t, rid)


@GPU
@pytest.mark.parametrize("n", [1, 2, 4])
def test_criterion_6_tp_equivalence(G, Z, n):
    for t in range(10):
        k = lambda s: Z[f"acc6_{n}_{t}_{s}"]  # noqa: E731
        y = G.tp_forward(G.tp_partition(k("w1"), "column", n), G.tp_partition(k("d1"), "column", n), k("x"), "column")
        z = G.tp_forward(G.tp_partition(k("w2"), "row", n), G.tp_partition(k("d2"), "row", n), y, "row")
        assert np.linalg.norm(z - k("ref")) / np.linalg.norm(k("ref")) <= REL, t
