"""Fixtures for the reference-suite shim (tests/test_gpu_refsuite.py), made by running the
REFERENCE package itself on the scenarios of its own hot-path tests:

  * /root/reference/pkg/tests/test_inference.py  classes TestDecoupledLinear .. TestForwardModel
  * /root/reference/pkg/tests/test_acceptance.py criteria 5 (decoupling exactness) and 6 (TP)

Every input the reference tests build (Philox `Rng` draws, OBS-compressed deltas, compress_model
outputs) is generated here by the reference's own functions with the tests' own seeds and stored
with the reference's outputs, so the shim feeds the B200 package exactly the reference tests'
operands. Nothing at test time reads /root/reference.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_refsuite.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from deltazip.compress import (  # noqa: E402
    SPARSITY_2_4, SPARSITY_NONE, CalibrationSet, CompressConfig, compress_model, compute_hessian,
    dequantize_layer, obs_compress_layer,
)
from deltazip.core import Rng, WeightStack, gaussian_matrix  # noqa: E402
from deltazip.inference import (  # noqa: E402
    BatchInput, DeltaHandle, TpLayout, forward_model, sbmm, tp_forward, tp_partition,
)

from make_golden import ld_arrays  # noqa: E402

CFG = CompressConfig(bits=4, sparsity=SPARSITY_2_4)  # test_inference.py CFG / acceptance CFG_4BIT


def obs(rows, cols, seed, scale=0.01):
    """test_inference.py `_layer_delta`: OBS-compressed gaussian delta, calibration from one Rng."""
    rng = Rng(seed)
    delta = gaussian_matrix(rng, rows, cols, scale)
    calib = CalibrationSet(gaussian_matrix(rng, cols, 2 * cols, 1.0))
    return obs_compress_layer(delta, compute_hessian(calib, 0.01), CFG)


def zero(rows, cols):
    """test_inference.py `_zero_delta`."""
    return obs_compress_layer(np.zeros((rows, cols)), np.eye(cols), CFG)


def paired(seed, layers=3, dim=12):
    """test_inference.py `_paired_stacks`: (fine-tuned, base) stacks."""
    rng = Rng(seed)
    std = 1.0 / np.sqrt(dim)
    base, fine = [], []
    for i in range(layers):
        w = gaussian_matrix(rng, dim, dim, std)
        d = gaussian_matrix(rng, dim, dim, 0.02 * std)
        base.append((f"l{i}", w))
        fine.append((f"l{i}", w + d))
    return WeightStack(fine), WeightStack(base)


def main():
    a: dict[str, np.ndarray] = {}

    def put_ld(key, ld):
        a.update(ld_arrays(f"{key}_", ld))

    # ---- TestDecoupledLinear ----------------------------------------------------------------
    rng = Rng(1)
    a["dl_zero_w"] = gaussian_matrix(rng, 8, 8, 1.0)
    a["dl_zero_x"] = gaussian_matrix(rng, 8, 3, 1.0)
    put_ld("dl_zero_ld", zero(8, 8))
    put_ld("dl_hand_ld", obs_compress_layer(np.array([[0.5, 0.0], [0.0, 0.0]]), np.eye(2),
                                            CompressConfig(bits=16, sparsity=SPARSITY_NONE)))
    for t in range(30):
        rng = Rng(100 + t)
        w = gaussian_matrix(rng, 12, 12, 0.5)
        ld = obs(12, 12, 200 + t)
        x = gaussian_matrix(rng, 12, 1, 1.0)[:, 0]
        a[f"dl_merged{t}_w"], a[f"dl_merged{t}_x"] = w, x
        a[f"dl_merged{t}_ref"] = (w + dequantize_layer(ld)) @ x
        put_ld(f"dl_merged{t}_ld", ld)
    # test_shape_error: the reference raises ShapeError already in _zero_delta(2, 2) (2:4 needs cols % 4)

    # ---- TestSbmm ---------------------------------------------------------------------------
    rng = Rng(30)
    a["sb_single_w"] = gaussian_matrix(rng, 8, 8, 0.5)
    put_ld("sb_single_ld", obs(8, 8, 31))
    a["sb_single_x"] = gaussian_matrix(rng, 8, 1, 1.0)[:, 0]
    rng = Rng(32)
    a["sb_multi_w"] = gaussian_matrix(rng, 8, 8, 0.5)
    deltas = {d: obs(8, 8, 40 + d) for d in range(3)}
    for d, ld in deltas.items():
        put_ld(f"sb_multi_d{d}", ld)
    rows = [(0, 0, 50), (1, 1, 51), (2, 2, 52), (3, 2, 53)]
    a["sb_multi_rows"] = np.array([(r, d) for r, d, _ in rows])
    a["sb_multi_x"] = np.stack([gaussian_matrix(Rng(s), 8, 1, 1.0)[:, 0] for _, _, s in rows])
    out = sbmm(a["sb_multi_w"], deltas, BatchInput([(r, d, x) for (r, d, _), x in zip(rows, a["sb_multi_x"])]))
    a["sb_multi_ref"] = np.stack([out[r] for r, _, _ in rows])
    put_ld("sb_zero4", zero(4, 4))
    rng = Rng(34)
    a["sb_order_w"] = gaussian_matrix(rng, 8, 8, 0.5)
    for d in range(2):
        put_ld(f"sb_order_d{d}", obs(8, 8, 60 + d))
    a["sb_order_x"] = np.stack([gaussian_matrix(Rng(70 + i), 8, 1, 1.0)[:, 0] for i in range(5)])

    # ---- TestTpForward ----------------------------------------------------------------------
    rng = Rng(80)
    a["tp_single_w"] = gaussian_matrix(rng, 8, 8, 0.5)
    ld = obs(8, 8, 81)
    put_ld("tp_single_ld", ld)
    a["tp_single_x"] = gaussian_matrix(rng, 8, 3, 1.0)
    for n in (1, 2, 4):
        rng = Rng(90 + n)
        w1, d1 = gaussian_matrix(rng, 8, 16, 0.4), gaussian_matrix(rng, 8, 16, 0.01)
        w2, d2 = gaussian_matrix(rng, 16, 8, 0.4), gaussian_matrix(rng, 16, 8, 0.01)
        x = gaussian_matrix(rng, 5, 8, 1.0)
        for k, v in dict(w1=w1, d1=d1, w2=w2, d2=d2, x=x, ref=(x @ (w1 + d1)) @ (w2 + d2)).items():
            a[f"tp_stack{n}_{k}"] = v
    rng = Rng(95)
    a["tp_zero_w"] = gaussian_matrix(rng, 6, 8, 0.4)
    a["tp_zero_x"] = gaussian_matrix(rng, 3, 6, 1.0)

    # ---- TestForwardModel -------------------------------------------------------------------
    def put_stack(key, ws):
        a[f"{key}_w"] = np.stack([w for _, w in ws.layers])

    _, base = paired(100)
    put_stack("fm_zero_base", base)
    put_ld("fm_zero_ld", zero(12, 12))
    a["fm_zero_x"] = gaussian_matrix(Rng(101), 12, 1, 1.0)[:, 0]
    a["fm_zero_ref"] = base.forward_tanh(a["fm_zero_x"].reshape(-1, 1))[:, 0]

    ft, base = paired(102)
    calib = CalibrationSet(gaussian_matrix(Rng(103), 12, 8, 1.0))
    cd = compress_model(ft, base, calib, CompressConfig(bits=16, sparsity=SPARSITY_NONE))
    put_stack("fm_lossless_base", base)
    for i, ld in enumerate(cd.layers):
        put_ld(f"fm_lossless_l{i}", ld)
    a["fm_lossless_x"] = gaussian_matrix(Rng(104), 12, 1, 1.0)[:, 0]
    a["fm_lossless_ref"] = ft.forward_tanh(a["fm_lossless_x"].reshape(-1, 1))[:, 0]

    _, base = paired(105)
    put_stack("fm_mixed_base", base)
    handles = {}
    for d in range(3):
        ftd, _ = paired(106 + d)
        calib = CalibrationSet(gaussian_matrix(Rng(120 + d), 12, 8, 1.0))
        cdd = compress_model(ftd, base, calib, CFG)
        handles[d] = DeltaHandle.from_compressed(d, cdd)
        for i, ld in enumerate(cdd.layers):
            put_ld(f"fm_mixed_d{d}_l{i}", ld)
    rows = [(i, i % 3, gaussian_matrix(Rng(130 + i), 12, 1, 1.0)[:, 0]) for i in range(6)]
    a["fm_mixed_x"] = np.stack([x for _, _, x in rows])
    out = forward_model(base, handles, BatchInput(rows))
    a["fm_mixed_ref"] = np.stack([out[r] for r, _, _ in rows])
    # duplicate request ids (inference.py:264-291): the reference's own semantics on this stack
    dup_rows = [(7, 2, rows[0][2]), (8, 0, rows[1][2]), (7, 0, rows[2][2]), (8, 1, rows[3][2]), (7, 1, rows[4][2])]
    a["fm_dup_rows"] = np.array([(r, d) for r, d, _ in dup_rows])
    a["fm_dup_x"] = np.stack([x for _, _, x in dup_rows])
    out = forward_model(base, handles, BatchInput(dup_rows))
    a["fm_dup_ref"] = np.stack([out[7], out[8]])
    out = sbmm(base.layers[0][1], {d: handles[d].layers[0] for d in range(3)}, BatchInput(dup_rows))
    a["sb_dup_ref"] = np.stack([out[7], out[8]])

    ft, base = paired(140, layers=2, dim=12)
    calib = CalibrationSet(gaussian_matrix(Rng(141), 12, 8, 1.0))
    cd = compress_model(ft, base, calib, CFG)
    put_stack("fm_tp_base", base)
    for i, ld in enumerate(cd.layers):
        put_ld(f"fm_tp_l{i}", ld)
    a["fm_tp_x"] = gaussian_matrix(Rng(142), 12, 1, 1.0)[:, 0]
    h = {0: DeltaHandle.from_compressed(0, cd)}
    batch = BatchInput([(0, 0, a["fm_tp_x"])])
    a["fm_tp_ref"] = forward_model(base, h, batch)[0]
    a["fm_tp_ref_tp2"] = forward_model(base, h, batch, layout=TpLayout(2, ("column", "row")))[0]

    # ---- acceptance criterion 5: 100 trials ------------------------------------------------
    for t in range(100):
        rng = Rng(5000 + t)
        n = 8 + 4 * (t % 3)
        a[f"acc5_{t}_base"] = gaussian_matrix(rng, n, n, 0.5)
        merged = []
        for d in range(3):
            delta = gaussian_matrix(rng, n, n, 0.01)
            calib = CalibrationSet(gaussian_matrix(rng, n, n, 1.0))
            ld = obs_compress_layer(delta, compute_hessian(calib, 0.01), CFG)
            put_ld(f"acc5_{t}_d{d}", ld)
            merged.append(a[f"acc5_{t}_base"] + dequantize_layer(ld))
        xs = [gaussian_matrix(rng, n, 1, 1.0)[:, 0] for _ in range(6)]
        a[f"acc5_{t}_x"] = np.stack(xs)
        a[f"acc5_{t}_merged"] = np.stack([merged[j % 3] @ xs[j] for j in range(6)])

    # ---- acceptance criterion 6: n in {1,2,4} x 10 trials -------------------------------------
    for n in (1, 2, 4):
        for t in range(10):
            rng = Rng(6000 + 10 * n + t)
            w1, d1 = gaussian_matrix(rng, 8, 16, 0.4), gaussian_matrix(rng, 8, 16, 0.01)
            w2, d2 = gaussian_matrix(rng, 16, 8, 0.4), gaussian_matrix(rng, 16, 8, 0.01)
            x = gaussian_matrix(rng, 4, 8, 1.0)
            y = tp_forward(tp_partition(w1, "column", n), tp_partition(d1, "column", n), x, "column")
            z = tp_forward(tp_partition(w2, "row", n), tp_partition(d2, "row", n), y, "row")
            for k, v in dict(w1=w1, d1=d1, w2=w2, d2=d2, x=x, ref=(x @ (w1 + d1)) @ (w2 + d2), z=z).items():
                a[f"acc6_{n}_{t}_{k}"] = v

    np.savez_compressed(os.path.join(HERE, "refsuite.npz"), **a)
    print(f"refsuite.npz: {len(a)} arrays")


if __name__ == "__main__":
    main()
