"""Generate golden fixtures by running the REFERENCE implementation itself.

Run once in the build container (the reference only exists there):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Writes `tests/golden/*.npz`. Each case stores the packed LayerDelta fields
exactly as the reference produced/consumed them plus the reference's own
outputs: `dequantize_layer` (compress.py:467-497) and, for SBMM cases,
`sbmm` (inference.py:126-154) on bf16-representable X / W_base. Nothing at
test time reads /root/reference; the fixtures travel with the repo.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from deltazip.compress import (  # noqa: E402
    SPARSITY_2_4, SPARSITY_NONE, CalibrationSet, CompressConfig, LayerDelta,
    compute_hessian, dequantize_layer, encode_mask_indices, obs_compress_layer, pack_codes,
)
from deltazip.core import Rng, gaussian_matrix  # noqa: E402
from deltazip.inference import BatchInput, group_by_delta, sbmm, tp_forward, tp_partition  # noqa: E402


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round f64 -> nearest-even bf16 -> f64 (so GPU inputs are exactly these values)."""
    f = np.asarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def obs_delta(rows, cols, bits, sparsity, gs, seed, scale=0.01):
    rng = Rng(seed)
    delta = gaussian_matrix(rng, rows, cols, scale)
    calib = CalibrationSet(gaussian_matrix(rng, cols, 2 * cols, 1.0))
    cfg = CompressConfig(bits=bits, sparsity=sparsity, group_size=gs,
                         block_size=4 * max(1, min(8, cols // 4)))
    return obs_compress_layer(delta, compute_hessian(calib, 0.01), cfg)


def rtn_delta(rows, cols, bits, gs, seed, scale=0.02):
    """magnitude 2:4 + RTN (pkg/tests/oracles.py:82-107 recipe), packed by the reference codec."""
    r = np.random.default_rng(seed)
    d = r.normal(0, scale, size=(rows, cols))
    q = (1 << (bits - 1)) - 1
    keep = np.ones((rows, cols), dtype=bool)
    for g0 in range(0, cols, 4):
        o = np.argsort(np.abs(d[:, g0:g0 + 4]), axis=1, kind="stable")
        keep[np.arange(rows), g0 + o[:, 0]] = False
        keep[np.arange(rows), g0 + o[:, 1]] = False
    ng = -(-cols // gs)
    scales = np.zeros((rows, ng))
    codes = np.zeros((rows, cols), dtype=np.int64)
    for g in range(ng):
        seg = d[:, g * gs:(g + 1) * gs]
        s = np.float64(np.float32(np.max(np.abs(seg), axis=1) / q))
        scales[:, g] = s
        codes[:, g * gs:(g + 1) * gs] = np.clip(np.rint(seg / s[:, None]), -q, q)
    return LayerDelta(name="rtn", rows=rows, cols=cols, packed_values=pack_codes(codes[keep], bits),
                      index_stream=encode_mask_indices(keep), scales=scales.astype("<f4").ravel(),
                      bits=bits, sparsity=SPARSITY_2_4, group_size=gs)


def random_delta(rows, cols, bits, gs, seed, sparse=True):
    """Raw random packed streams: every u in [0, 2^bits) including the unclamped one."""
    r = np.random.default_rng(seed)
    n = rows * cols // 2 if sparse else rows * cols
    per = 32 // bits
    nw = -(-n // per)
    words = r.integers(0, 2 ** 32, size=nw, dtype=np.uint64).astype("<u4")
    if n % per:
        words[-1] &= np.uint32((1 << ((n % per) * bits)) - 1)
    index = b""
    if sparse:
        nib = np.array([0x4, 0x8, 0xC, 0x9, 0xD, 0xE], dtype=np.uint8)[r.integers(0, 6, rows * (cols // 4))]
        if nib.size % 2:
            nib = np.concatenate([nib, np.zeros(1, np.uint8)])
        index = (nib[0::2] | (nib[1::2] << 4)).tobytes()
    ng = -(-cols // gs)
    scales = (np.abs(r.normal(0, 0.02, size=rows * ng)) / ((1 << (bits - 1)) - 1)).astype("<f4")
    return LayerDelta(name="rand", rows=rows, cols=cols, packed_values=words, index_stream=index,
                      scales=scales, bits=bits, sparsity=SPARSITY_2_4 if sparse else SPARSITY_NONE,
                      group_size=gs)


def ld_arrays(prefix, ld):
    return {
        f"{prefix}packed": np.asarray(ld.packed_values, dtype="<u4"),
        f"{prefix}index": np.frombuffer(ld.index_stream, dtype=np.uint8).copy(),
        f"{prefix}scales": np.asarray(ld.scales, dtype="<f4"),
        f"{prefix}meta": np.array([ld.rows, ld.cols, ld.bits, int(ld.sparsity == SPARSITY_2_4),
                                   ld.group_size], dtype=np.int64),
    }


def main():
    cases = {}
    # --- single-layer unpack cases: (name, LayerDelta) -----------------------------------
    unpack = [
        ("obs_8x8_b4", obs_delta(8, 8, 4, SPARSITY_2_4, 128, 31)),        # ref test shape
        ("obs_12x12_b4", obs_delta(12, 12, 4, SPARSITY_2_4, 128, 200)),   # rows not word aligned
        ("obs_16x64_b2", obs_delta(16, 64, 2, SPARSITY_2_4, 128, 5)),
        ("obs_16x32_b3", obs_delta(16, 32, 3, SPARSITY_2_4, 16, 6)),      # 3-bit, gs=16
        ("obs_8x32_b8_dense", obs_delta(8, 32, 8, SPARSITY_NONE, 128, 7)),
        ("obs_8x16_b16_dense", obs_delta(8, 16, 16, SPARSITY_NONE, 128, 8)),
        ("obs_8x16_b16_sparse", obs_delta(8, 16, 16, SPARSITY_2_4, 128, 9)),
        ("rtn_64x512_b4", rtn_delta(64, 512, 4, 128, 10)),
        ("rtn_48x384_b2", rtn_delta(48, 384, 2, 128, 11)),
        ("rtn_20x260_b4", rtn_delta(20, 260, 4, 128, 12)),                # cols/4 odd: nibbles straddle rows
        ("rand_24x136_b3", random_delta(24, 136, 3, 128, 13)),
        ("rand_32x256_b4_u15", random_delta(32, 256, 4, 128, 14)),        # includes unclamped u=15 -> code 8
        ("rand_16x256_b2", random_delta(16, 256, 2, 128, 15)),
        ("rand_16x128_b8", random_delta(16, 128, 8, 128, 16)),
        ("rand_8x64_b4_gs64", random_delta(8, 64, 4, 64, 17)),
        ("rand_8x96_b4_dense", random_delta(8, 96, 4, 128, 18, sparse=False)),
        ("rand_17x200_b4_gs48", random_delta(17, 200, 4, 48, 19)),
    ]
    for name, ld in unpack:
        arrs = ld_arrays("", ld)
        arrs["dequant"] = dequantize_layer(ld)
        np.savez_compressed(os.path.join(HERE, f"unpack_{name}.npz"), **arrs)
        cases[f"unpack_{name}"] = [ld.rows, ld.cols, ld.bits, ld.sparsity, ld.group_size]

    # --- SBMM cases: base + D deltas + T mixed tokens ------------------------------------
    sb = [
        ("cfg1_mini", 64, 256, 4, 4, 16, "rtn"),     # cfg1 in miniature (4 deltas, 16 tokens)
        ("b2_mixed", 48, 384, 2, 3, 9, "rtn"),
        ("ragged", 20, 260, 4, 3, 7, "rtn"),
        ("obs_12", 12, 12, 4, 3, 6, "obs"),          # acceptance-5 shape
        ("b3_rand", 24, 136, 3, 2, 5, "rand"),
        ("dense_b8", 16, 128, 8, 2, 4, "rand_dense"),
    ]
    for name, rows, cols, bits, D, T, kind in sb:
        r = np.random.default_rng(1000 + rows + cols + D)
        deltas = {}
        for d in range(D):
            seed = 7000 + 17 * d + rows
            if kind == "rtn":
                deltas[d] = rtn_delta(rows, cols, bits, 128, seed)
            elif kind == "obs":
                deltas[d] = obs_delta(rows, cols, bits, SPARSITY_2_4, 128, seed)
            elif kind == "rand":
                deltas[d] = random_delta(rows, cols, bits, 128, seed)
            else:
                deltas[d] = random_delta(rows, cols, bits, 128, seed, sparse=False)
        W = bf16_round(r.normal(0, 1 / np.sqrt(cols), size=(rows, cols)))
        X = bf16_round(r.normal(0, 1, size=(T, cols)))
        ids = r.permutation([i % D for i in range(T)]).astype(np.int64)
        rids = np.arange(100, 100 + T, dtype=np.int64)
        out = sbmm(W, deltas, BatchInput([(int(rids[i]), int(ids[i]), X[i]) for i in range(T)]))
        Y = np.stack([out[int(rid)] for rid in rids])
        perm, groups = group_by_delta(BatchInput([(int(rids[i]), int(ids[i]), X[i]) for i in range(T)]))
        arrs = {"W": W, "X": X, "ids": ids, "rids": rids, "Y": Y, "perm": np.array(perm, dtype=np.int64),
                "groups": np.array(groups, dtype=np.int64).reshape(-1, 3)}
        for d, ld in deltas.items():
            arrs.update(ld_arrays(f"d{d}_", ld))
        np.savez_compressed(os.path.join(HERE, f"sbmm_{name}.npz"), **arrs)
        cases[f"sbmm_{name}"] = [rows, cols, bits, D, T, kind]

    # --- TP case: column then row shards (inference.py:162-225) ---------------------------
    r = np.random.default_rng(77)
    w1 = bf16_round(r.normal(0, 0.4, (8, 16)))
    d1 = r.normal(0, 0.01, (8, 16))
    w2 = bf16_round(r.normal(0, 0.4, (16, 8)))
    d2 = r.normal(0, 0.01, (16, 8))
    x = bf16_round(r.normal(0, 1, (5, 8)))
    tp = {}
    for n in (1, 2, 4):
        y = tp_forward(tp_partition(w1, "column", n), tp_partition(d1, "column", n), x, "column")
        z = tp_forward(tp_partition(w2, "row", n), tp_partition(d2, "row", n), y, "row")
        tp[f"y{n}"] = y
        tp[f"z{n}"] = z
    np.savez_compressed(os.path.join(HERE, "tp_two_layer.npz"), w1=w1, d1=d1, w2=w2, d2=d2, x=x, **tp)
    cases["tp_two_layer"] = "w1 column, w2 row, n in 1,2,4"

    # --- KATs ----------------------------------------------------------------------------
    kat = {
        "pack_spec_word": [int(w) for w in pack_codes([-7, 0, 7, 1, 2, 3, -1, -2], 4)],
        "pack_zero_word": [int(w) for w in pack_codes([0] * 8, 4)],
    }
    keep = np.zeros((2, 8), dtype=bool)
    keep[0, [0, 1, 6, 7]] = True
    keep[1, [0, 3, 5, 6]] = True
    ld = LayerDelta(name="kat", rows=2, cols=8, packed_values=pack_codes([1, -2, 3, -7, 7, 0, -1, 2], 4),
                    index_stream=encode_mask_indices(keep), scales=np.array([0.5, 0.25], dtype="<f4"),
                    bits=4, sparsity=SPARSITY_2_4, group_size=128)
    kat["survey_index_hex"] = ld.index_stream.hex()
    kat["survey_packed"] = [int(w) for w in ld.packed_values]
    kat["survey_dequant"] = dequantize_layer(ld).tolist()
    b = BatchInput([(i, d, np.zeros(2)) for i, d in enumerate([2, 0, 2, 1])])
    perm, groups = group_by_delta(b)
    kat["group_by_delta_perm"] = perm
    kat["group_by_delta_groups"] = [list(g) for g in groups]
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat, f, indent=1)
    with open(os.path.join(HERE, "MANIFEST.json"), "w") as f:
        json.dump(cases, f, indent=1)
    print(f"wrote {len(cases)} cases")


if __name__ == "__main__":
    main()
