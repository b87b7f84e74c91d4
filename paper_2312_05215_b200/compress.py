"""ΔCompress packed-delta format and its GPU unpack (K1).

`LayerDelta` is field-for-field the reference container (compress.py:101-143), so a caller's
existing objects (or the reference's own) are accepted as-is. `dequantize_layer` runs the K1
CUDA kernel and returns exactly the reference's float64 matrix (the product code*scale is
formed in f64 on the GPU, as the reference does on the CPU, compress.py:467-497).
The offline ΔCompress solver (compress.py:348-548) is out of scope.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .device import ErrFlag, RefDeltaDevice, require_cuda, stream_ptr
from .errors import EncodingError

SPARSITY_NONE = "none"
SPARSITY_2_4 = "two_of_four"
VALID_BITS = (2, 3, 4, 8, 16)


@dataclass
class LayerDelta:
    """Packed compressed delta for one layer (reference compress.py:101-143)."""

    name: str
    rows: int
    cols: int
    packed_values: np.ndarray
    index_stream: bytes
    scales: np.ndarray
    bits: int
    sparsity: str
    group_size: int
    proxy_loss: float = field(default=0.0, compare=False)

    def __post_init__(self):
        self.packed_values = np.ascontiguousarray(self.packed_values, dtype="<u4")
        self.scales = np.ascontiguousarray(self.scales, dtype="<f4")

    def __eq__(self, other) -> bool:
        if not isinstance(other, LayerDelta):
            return NotImplemented
        return (self.name == other.name and self.rows == other.rows and self.cols == other.cols
                and self.bits == other.bits and self.sparsity == other.sparsity
                and self.group_size == other.group_size
                and np.array_equal(self.packed_values, other.packed_values)
                and bytes(self.index_stream) == bytes(other.index_stream)
                and np.array_equal(self.scales, other.scales))

    @property
    def n_groups(self) -> int:
        return math.ceil(self.cols / self.group_size)


# ------------------------------------------------------------------------------ producer side
# (pack side of the codec; used to build LayerDeltas, never on the serving path)


def pack_codes(codes, bits: int) -> np.ndarray:
    """Signed codes -> little-endian u32 words (format definition: compress.py:243-262)."""
    if not 2 <= bits <= 16:
        raise ValueError(f"bits must be in [2, 16], got {bits}")
    c = np.asarray(codes, dtype=np.int64).ravel()
    q = (1 << (bits - 1)) - 1
    if c.size and (int(c.min()) < -q or int(c.max()) > q):
        raise EncodingError(f"codes out of range [-{q}, {q}] for {bits}-bit packing")
    per = 32 // bits
    nw = -(-c.size // per)
    u = np.zeros(nw * per, dtype=np.uint64)
    u[: c.size] = (c + q).astype(np.uint64)
    u = u.reshape(nw, per) << (np.arange(per, dtype=np.uint64) * np.uint64(bits))
    return np.bitwise_or.reduce(u, axis=1).astype(np.uint64).astype("<u4") if nw else np.zeros(0, "<u4")


def encode_mask_indices(keep: np.ndarray) -> bytes:
    """Bool 2:4 keep-mask -> nibble stream (format definition: compress.py:280-292)."""
    keep = np.asarray(keep, dtype=bool)
    pos = np.argwhere(keep.reshape(-1, 4))[:, 1].reshape(-1, 2)
    nib = (pos[:, 0] | (pos[:, 1] << 2)).astype(np.uint8)
    if nib.size % 2:
        nib = np.concatenate([nib, np.zeros(1, np.uint8)])
    return (nib[0::2] | (nib[1::2] << 4)).astype(np.uint8).tobytes()


# ------------------------------------------------------------------------------ GPU unpack (K1)


def unpack_codes(words, bits: int, count: int) -> np.ndarray:
    """GPU inverse of pack_codes (compress.py:265-277): `count` signed codes, no clamping."""
    if not 2 <= bits <= 16:
        raise ValueError(f"bits must be in [2, 16], got {bits}")
    dev = require_cuda()
    w = np.ascontiguousarray(words, dtype="<u4")
    wd = torch.from_numpy(np.concatenate([w, np.zeros(1, "<u4")]).view(np.int32)).to(dev)
    out = torch.empty(max(count, 1), dtype=torch.int32, device=dev)
    L.check(L.lib().dz_unpack_codes(wd.data_ptr(), w.size, bits, count, out.data_ptr(), stream_ptr()),
            "unpack_codes")
    return out[:count].cpu().numpy().astype(np.int64)


def decode_mask_indices(data: bytes, rows: int, cols: int) -> np.ndarray:
    """GPU decode of the 2-bit index stream into the bool keep-mask (compress.py:295-314)."""
    dev = require_cuda()
    raw = np.frombuffer(bytes(data), dtype=np.uint8)
    d = torch.zeros(raw.size + 16, dtype=torch.uint8, device=dev)
    if raw.size:
        d[: raw.size].copy_(torch.from_numpy(raw.copy()))
    keep = torch.zeros(max(rows * cols, 4), dtype=torch.uint8, device=dev)
    err = ErrFlag(dev)
    L.check(L.lib().dz_decode_index(d.data_ptr(), raw.size, rows, cols, keep.data_ptr(), err.ptr, stream_ptr()),
            "decode_mask_indices")
    err.raise_if_set("corrupt index stream: kept positions not strictly increasing")
    return keep[: rows * cols].cpu().numpy().astype(bool).reshape(rows, cols)


def dequantize_layer_device(ld, dtype: torch.dtype = torch.float32, ref: RefDeltaDevice | None = None,
                            check: bool = True) -> torch.Tensor:
    """K1 on the device: dense ΔW [rows, cols] as float64 / float32 / bfloat16.

    f64 is bit-identical to the reference's dequantize_layer; f32 to np.float32 of it; bf16 to
    torch's .to(bfloat16) of it."""
    dev = require_cuda()
    code = {torch.float64: L.DZ_F64, torch.float32: L.DZ_F32, torch.bfloat16: L.DZ_BF16}[dtype]
    ref = ref or RefDeltaDevice(ld, dev)
    out = torch.empty(ref.rows, ref.cols, dtype=dtype, device=dev)
    err = ErrFlag(dev)
    L.check(L.lib().dz_unpack(ref.struct, code, out.data_ptr(), ref.cols, err.ptr, stream_ptr()),
            "dequantize_layer")
    if check:
        err.raise_if_set("corrupt index stream: kept positions not strictly increasing")
    return out


def dequantize_layer(ld) -> np.ndarray:
    """Reconstruct the dense float64 delta (reference compress.py:467-497) on the GPU."""
    return dequantize_layer_device(ld, torch.float64).cpu().numpy()
