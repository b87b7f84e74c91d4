"""Generate DZDL container fixtures with the REFERENCE writer (formats.write_delta,
formats.py:60-99) from deltas the reference compressor produced (compress_model,
compress.py:511-548). Run once in the build container (the reference only exists there):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_dzdl.py

Writes tests/golden/dzdl_*.dzdl plus dzdl_*.npz with, per layer, the fields the reference's
read_delta returns and its dequantize_layer output, and a JSON sidecar of the header/config.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from deltazip.compress import (  # noqa: E402
    SPARSITY_2_4, SPARSITY_NONE, CalibrationSet, CompressConfig, compress_model, dequantize_layer,
)
from deltazip.core import Rng, WeightStack, gaussian_matrix  # noqa: E402
from deltazip.formats import inspect_delta, read_delta, write_delta  # noqa: E402


def compressed(seed, dims, bits, sparsity, lossless, gs=128):
    rng = Rng(seed)
    base, fine = [], []
    for i, (rows, cols) in enumerate(dims):
        w = gaussian_matrix(rng, rows, cols, 1.0 / np.sqrt(cols))
        d = gaussian_matrix(rng, rows, cols, 0.02 / np.sqrt(cols))
        base.append((f"layers.{i}.proj", w))
        fine.append((f"layers.{i}.proj", w + d))
    calib = CalibrationSet(gaussian_matrix(rng, dims[0][1], 16, 1.0))
    cfg = CompressConfig(bits=bits, sparsity=sparsity, group_size=gs, lossless=lossless)
    return compress_model(WeightStack(fine), WeightStack(base), calib, cfg, f"demo-base-{seed}")


CASES = {
    # name: (seed, layer dims (chain-compatible), bits, sparsity, lossless, group_size)
    "dzdl_b4": (1, [(128, 256), (64, 128)], 4, SPARSITY_2_4, "off", 128),
    "dzdl_b4_deflate": (2, [(128, 256), (64, 128)], 4, SPARSITY_2_4, "deflate", 128),
    "dzdl_b2": (3, [(64, 128)], 2, SPARSITY_2_4, "off", 128),
    "dzdl_b16_dense": (4, [(16, 16)], 16, SPARSITY_NONE, "off", 128),
}


def main():
    for name, (seed, dims, bits, sp, ll, gs) in CASES.items():
        cd = compressed(seed, dims, bits, sp, ll, gs)
        path = os.path.join(HERE, f"{name}.dzdl")
        write_delta(cd, path)
        again = read_delta(path)
        assert again == cd
        header, sizes, ratio = inspect_delta(path)
        arrays = {}
        for i, ld in enumerate(again.layers):
            arrays[f"l{i}_packed"] = np.asarray(ld.packed_values, dtype="<u4")
            arrays[f"l{i}_index"] = np.frombuffer(ld.index_stream, dtype=np.uint8)
            arrays[f"l{i}_scales"] = np.asarray(ld.scales, dtype="<f4")
            arrays[f"l{i}_dequant"] = dequantize_layer(ld)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
        meta = {"header": header, "ratio": ratio,
                "layers": [{"name": ld.name, "rows": ld.rows, "cols": ld.cols} for ld in again.layers],
                "sizes": [[s.scales_bytes, s.index_bytes, s.payload_bytes] for s in sizes],
                "file_bytes": os.path.getsize(path)}
        with open(os.path.join(HERE, f"{name}.json"), "w") as f:
            json.dump(meta, f, indent=1, sort_keys=True)
        print(name, os.path.getsize(path), "bytes", len(again.layers), "layers")


if __name__ == "__main__":
    main()
