"""Golden fixtures for the GPU ΔCompress solver, produced by running the REFERENCE itself.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_obs.py

Each `obs_*.npz` holds one layer: the delta, the proxy Hessian (compute_hessian,
compress.py:178-186), the reference's inverse-Hessian factor U (_inverse_cholesky_factor,
compress.py:321-336), the config, and obs_compress_layer's outputs (compress.py:348-464): packed
words, index stream, scales, proxy loss, plus dequantize_layer of the result. `obs_model_*.npz`
holds a two-layer compress_model run (compress.py:508-548). Nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from deltazip.compress import (  # noqa: E402
    SPARSITY_2_4, SPARSITY_NONE, CalibrationSet, CompressConfig, _inverse_cholesky_factor,
    compress_model, compute_hessian, dequantize_layer, obs_compress_layer,
)
from deltazip.core import Rng, WeightStack, gaussian_matrix  # noqa: E402

CASES = [
    # name, rows, cols, bits, sparsity, group_size, block_size, seed
    ("obs_b4_single_48x32", 48, 32, 4, SPARSITY_2_4, 128, 32, 1),
    ("obs_b4_40x256", 40, 256, 4, SPARSITY_2_4, 128, 32, 2),
    ("obs_b2_64x384", 64, 384, 2, SPARSITY_2_4, 128, 32, 3),
    ("obs_b3_dense_24x200_bs16_gs64", 24, 200, 3, SPARSITY_NONE, 64, 16, 4),
    ("obs_b8_dense_17x100_gs48", 17, 100, 8, SPARSITY_NONE, 48, 32, 5),
    ("obs_b4_33x512_bs128", 33, 512, 4, SPARSITY_2_4, 128, 128, 6),
    ("obs_b4_gs40_20x160_bs8", 20, 160, 4, SPARSITY_2_4, 40, 8, 7),
    ("obs_b16_sparse_16x64", 16, 64, 16, SPARSITY_2_4, 128, 32, 8),
    ("obs_b16_dense_8x40", 8, 40, 16, SPARSITY_NONE, 128, 32, 9),
    # edge cases of the windowed schedule (window = group when block | group)
    ("obs_b16_sparse_16x320", 16, 320, 16, SPARSITY_2_4, 128, 32, 10),
    ("obs_b4_9x48_bs4_gs8", 9, 48, 4, SPARSITY_2_4, 8, 4, 11),
    ("obs_b2_dense_1x100_bs12_gs36", 1, 100, 2, SPARSITY_NONE, 36, 12, 12),
    ("obs_b8_70x264_gs64", 70, 264, 8, SPARSITY_2_4, 64, 32, 13),
]


def main():
    for name, r, c, bits, sp, gs, bs, seed in CASES:
        rng = Rng(seed)
        delta = gaussian_matrix(rng, r, c, 0.01)
        calib = CalibrationSet(gaussian_matrix(rng, c, 2 * c, 1.0))
        cfg = CompressConfig(bits=bits, sparsity=sp, group_size=gs, block_size=bs)
        h = compute_hessian(calib, cfg.damping)
        u = _inverse_cholesky_factor(h, name)
        ld = obs_compress_layer(delta, h, cfg, name=name)
        np.savez(os.path.join(HERE, name + ".npz"), delta=delta, hessian=h, u=u,
                 cfg=np.array([bits, 1 if sp == SPARSITY_2_4 else 0, gs, bs]),
                 packed=ld.packed_values, index=np.frombuffer(ld.index_stream, np.uint8),
                 scales=ld.scales, proxy_loss=np.float64(ld.proxy_loss), dequant=dequantize_layer(ld))
        print(name, ld.proxy_loss)

    # two-layer compress_model: 96 -> 64 -> 48, 4-bit 2:4, calibration 96 x 160
    rng = Rng(21)
    shapes = [(64, 96), (48, 64)]
    wb = WeightStack([(f"l{i}", gaussian_matrix(rng, o, n, 1 / np.sqrt(n))) for i, (o, n) in enumerate(shapes)])
    wf = WeightStack([(nm, w + gaussian_matrix(rng, *w.shape, 0.01)) for nm, w in wb.layers])
    calib = CalibrationSet(gaussian_matrix(rng, 96, 160, 1.0))
    cfg = CompressConfig(bits=4, sparsity=SPARSITY_2_4, group_size=32, block_size=16)
    cd = compress_model(wf, wb, calib, cfg, base_model_id="base")
    out = {"calib": calib.samples, "fingerprint": np.uint64(cd.calibration_fingerprint)}
    for i, ((nm, f), (_, b), ld) in enumerate(zip(wf.layers, wb.layers, cd.layers)):
        out.update({f"wf{i}": f, f"wb{i}": b, f"packed{i}": ld.packed_values,
                    f"index{i}": np.frombuffer(ld.index_stream, np.uint8), f"scales{i}": ld.scales,
                    f"loss{i}": np.float64(ld.proxy_loss), f"dequant{i}": dequantize_layer(ld)})
    np.savez(os.path.join(HERE, "obs_model_2layer.npz"), **out)
    print("obs_model_2layer", [ld.proxy_loss for ld in cd.layers])


if __name__ == "__main__":
    main()
