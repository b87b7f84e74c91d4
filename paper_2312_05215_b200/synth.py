"""Synthetic Llama-shaped workloads generated on the device (no datasets or checkpoints here).

Deltas follow SURVEY §8(d): reference-layout packed streams with uniform codes
u in [0, 2^bits) (including the unclamped code), index nibbles uniform over the six valid 2:4
patterns, scales |N(0, 0.02/sqrt(in))|*(3/qmax) as f32. They go through the real upload path
(`dz_repack_sparse`, which validates every nibble) into native blocks. Base weights are
N(0, 1/sqrt(in)) in bf16 (cli.py:142 convention).
"""

from __future__ import annotations

import math

import torch

from . import _lib as L
from .device import ErrFlag, stream_ptr
from .engine import NativeDelta

_NIBS = torch.tensor([0x4, 0x8, 0xC, 0x9, 0xD, 0xE], dtype=torch.uint8)

LLAMA_SHAPES = {
    "7b": dict(hidden=4096, inter=11008, layers=32, kv=4096),
    "13b": dict(hidden=5120, inter=13824, layers=40, kv=5120),
    "70b": dict(hidden=8192, inter=28672, layers=80, kv=1024),
    # test-sized Llama layer: GQA-style kv, intermediate of 11 native blocks (uneven at TP 2/4)
    "tiny": dict(hidden=1024, inter=1408, layers=2, kv=512),
}


def llama_linears(model: str) -> list[tuple[str, int, int]]:
    """(name, out, in) of one decoder layer's seven linears."""
    s = LLAMA_SHAPES[model]
    h, i, kv = s["hidden"], s["inter"], s["kv"]
    return [("q", h, h), ("k", kv, h), ("v", kv, h), ("o", h, h), ("gate", i, h), ("up", i, h), ("down", h, i)]


def random_ref_delta_device(rows: int, cols: int, bits: int, gen: torch.Generator, device, group_size: int = 128):
    """Random reference-layout LayerDelta bytes, directly in device memory. Returns (struct, keepalive)."""
    n = rows * cols // 2
    per = 32 // bits
    nw = -(-n // per)
    packed = torch.randint(-(2 ** 31), 2 ** 31 - 1, (nw + 4,), dtype=torch.int32, device=device, generator=gen)
    ng = rows * (cols // 4)
    nb = -(-ng // 2)
    nibs = _NIBS.to(device)
    lo = nibs[torch.randint(0, 6, (nb,), device=device, generator=gen)]
    hi = nibs[torch.randint(0, 6, (nb,), device=device, generator=gen)]
    index = lo | (hi << 4)
    n_groups = math.ceil(cols / group_size)
    qmax = (1 << (bits - 1)) - 1
    scales = (torch.randn(rows * n_groups, device=device, generator=gen).abs_()
              .mul_(0.02 / math.sqrt(cols) * 3.0 / qmax)).float()
    st = L.DzRefDelta(packed.data_ptr(), nw, index.data_ptr(), nb, scales.data_ptr(), rows * n_groups,
                      rows, cols, bits, 1, group_size, 0)
    return st, (packed, index, scales)


def random_native_delta(rows: int, cols: int, bits: int, gen: torch.Generator, device,
                        err: ErrFlag | None = None, keep_ref: list | None = None) -> NativeDelta:
    """keep_ref: a list that receives (DzRefDelta, tensors) — the reference-layout bytes the
    native blocks were built from (parity tests dequantise them with K1 as the reference does)."""
    st, keep = random_ref_delta_device(rows, cols, bits, gen, device)
    if keep_ref is not None:
        keep_ref.append((st, keep))
    lib = L.lib()
    nbytes = lib.dz_native_sparse_bytes(rows, cols, bits)
    blocks = torch.empty(nbytes, dtype=torch.uint8, device=device)
    err = err or ErrFlag(device)
    L.check(lib.dz_repack_sparse(st, blocks.data_ptr(), err.ptr, stream_ptr()), "synthetic delta upload")
    del keep, st
    kind = {2: L.DZ_KIND_SPARSE2, 3: L.DZ_KIND_SPARSE3, 4: L.DZ_KIND_SPARSE4}[bits]
    return NativeDelta(kind, (1 << (bits - 1)) - 1, rows, cols, blocks, bits)


def random_base(rows: int, cols: int, gen: torch.Generator, device) -> torch.Tensor:
    return (torch.randn(rows, cols, device=device, generator=gen) / math.sqrt(cols)).to(torch.bfloat16)


def delta_algorithmic_bytes(rows: int, cols: int, bits: int, group_size: int = 128) -> int:
    """4*ceil(n_kept*bits/32) + ceil(rows*cols/8) + 4*rows*ceil(cols/gs)."""
    n = rows * cols // 2
    per = 32 // bits
    return 4 * (-(-n // per)) + (-(-rows * cols // 8)) + 4 * rows * math.ceil(cols / group_size)


def linear_algorithmic_bytes(rows: int, cols: int, bits: int, n_distinct: int, T: int) -> int:
    """B = 2*out*in + sum_d delta bytes + 2*T*in + 2*T*out + 4*T."""
    return 2 * rows * cols + n_distinct * delta_algorithmic_bytes(rows, cols, bits) + 2 * T * cols + 2 * T * rows + 4 * T
