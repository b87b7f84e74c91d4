"""DZDL delta containers -> device-resident deltas (the swap-in path).

Reference: formats.py:60-169 (write_delta / read_delta / inspect_delta), compress.py:560-564
(zlib lossless codec). The container is parsed in place by the native parser
(`dz_dzdl_parse_header` / `dz_dzdl_parse_layers`, dz_dzdl.cpp) over an mmap of the file, deflate
payloads are inflated by `dz_inflate`, and `load_delta` stages every layer through pinned host
memory with asynchronous copies before the upload-time re-layout (`dz_repack_sparse`), which
validates every index nibble (FormatError at load time, not at first use).

`read_delta` / `inspect_delta` keep the reference signatures and error contract (FormatError
with the byte offset of truncations, bad magic, unsupported version, trailing bytes) for host
callers; `DeltaPool` is the serving-side store of resident deltas with tensor-parallel
resharding of the packed format (stack.shard_sub).
"""

from __future__ import annotations

import ctypes as C
import json
import mmap
import os
import traceback
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .compress import SPARSITY_2_4, LayerDelta
from .errors import FormatError

DELTA_MAGIC = b"DZDL"
LOSSLESS_OFF, LOSSLESS_DEFLATE = "off", "deflate"


@dataclass(frozen=True)
class CompressConfig:
    """The configuration fields a DZDL header carries (reference compress.py:44-69)."""

    bits: int = 4
    sparsity: str = SPARSITY_2_4
    group_size: int = 128
    damping: float = 0.01
    block_size: int = 32
    lossless: str = LOSSLESS_OFF
    solver: str = "obs"

    def __post_init__(self):  # reference compress.py:52-69
        if self.solver != "obs":
            raise ValueError(f"solver {self.solver!r} is not implemented")
        if self.bits not in (2, 3, 4, 8, 16):
            raise ValueError(f"bits must be one of (2, 3, 4, 8, 16), got {self.bits}")
        if self.sparsity not in ("none", SPARSITY_2_4):
            raise ValueError(f"unknown sparsity {self.sparsity!r}")
        if self.group_size < 1:
            raise ValueError("group_size must be >= 1")
        if self.block_size < 1:
            raise ValueError("block_size must be >= 1")
        if self.sparsity == SPARSITY_2_4 and self.block_size % 4 != 0:
            raise ValueError("block_size must be a multiple of 4 for 2:4 sparsity")
        if self.damping < 0:
            raise ValueError("damping must be nonnegative")
        if self.lossless not in (LOSSLESS_OFF, LOSSLESS_DEFLATE):
            raise ValueError(f"unknown lossless codec {self.lossless!r}")

    @property
    def is_passthrough(self) -> bool:
        return self.bits == 16


@dataclass
class CompressedDelta:
    """reference compress.py:147-161"""

    base_model_id: str
    layers: list
    config: CompressConfig
    calibration_fingerprint: int

    def __eq__(self, other) -> bool:
        if not isinstance(other, CompressedDelta):
            return NotImplemented
        return (self.base_model_id == other.base_model_id and self.config == other.config
                and self.calibration_fingerprint == other.calibration_fingerprint and self.layers == other.layers)


@dataclass
class LayerSizes:
    """reference formats.py:172-186"""

    name: str
    rows: int
    cols: int
    scales_bytes: int
    index_bytes: int
    payload_bytes: int

    @property
    def total_bytes(self) -> int:
        return self.scales_bytes + self.index_bytes + self.payload_bytes

    @property
    def dense16_bytes(self) -> int:
        return self.rows * self.cols * 2


@dataclass
class _Parsed:
    data: object  # bytes-like (mmap or bytes)
    header: dict
    config: CompressConfig
    layers: list = field(default_factory=list)  # DzDzdlLayer records


def _buf_ptr(data) -> tuple[int, object]:
    arr = np.frombuffer(data, dtype=np.uint8)
    return arr.ctypes.data, arr


def _parse(data, strict_header: bool = True) -> _Parsed:
    lib = L.lib()
    ptr, keep = _buf_ptr(data)
    n = len(data)
    info = L.DzDzdlInfo()
    off = C.c_int64(0)
    st = lib.dz_dzdl_parse_header(ptr, n, C.byref(info), C.byref(off))
    if st == L.DZ_E_FORMAT:
        if n >= 4 and bytes(data[:4]) != DELTA_MAGIC:
            raise FormatError(f"bad magic {bytes(data[:4])!r}, expected {DELTA_MAGIC!r}", offset=0)
        raise FormatError("truncated file while reading the container header", offset=off.value)
    if st == L.DZ_E_UNSUPPORTED:
        raise FormatError(f"unsupported version {info.version}", offset=4)
    L.check(st, "dzdl header")
    try:
        header = json.loads(bytes(data[info.header_off: info.header_off + info.header_len]).decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise FormatError(f"bad header json: {exc}", offset=12) from exc
    try:
        cfg = CompressConfig(bits=int(header["bits"]), sparsity=header["sparsity"], group_size=int(header["group_size"]),
                             damping=header.get("damping", 0.01), block_size=header.get("block_size", 32),
                             lossless=LOSSLESS_DEFLATE if info.lossless else LOSSLESS_OFF)
        count = int(header["layer_count"])
        header["base_model_id"], header["calibration_fingerprint"]  # noqa: B018 (required keys)
    except (KeyError, ValueError, TypeError) as exc:
        raise FormatError(f"invalid header: {exc}", offset=12) from exc
    recs = (L.DzDzdlLayer * max(count, 1))()
    st = lib.dz_dzdl_parse_layers(ptr, n, info.layers_off, count, recs, C.byref(off))
    if st == L.DZ_E_FORMAT:
        raise FormatError("truncated file while reading a layer record", offset=off.value)
    if st == L.DZ_E_VALUE and strict_header:
        raise FormatError(f"{n - off.value} trailing bytes after last layer", offset=off.value)
    if st not in (L.DZ_OK, L.DZ_E_VALUE):
        L.check(st, "dzdl layers")
    del keep
    return _Parsed(data, header, cfg, list(recs)[:count])


def _inflate(src: np.ndarray, rows: int, cols: int, cfg: CompressConfig) -> np.ndarray:
    """zlib payload -> uint8 array (compress.py:560-564, FormatError on a corrupt stream)."""
    lib = L.lib()
    n_vals = rows * cols // 2 if cfg.sparsity == SPARSITY_2_4 else rows * cols
    guess = 8 * n_vals if cfg.bits == 16 else 4 * (-(-n_vals * cfg.bits // 32)) + 64
    out = np.empty(max(guess, 16), dtype=np.uint8)
    got = C.c_int64(0)
    st = lib.dz_inflate(src.ctypes.data, src.size, out.ctypes.data, out.size, C.byref(got))
    if st == L.DZ_E_ENCODING:
        out = np.empty(got.value, dtype=np.uint8)
        st = lib.dz_inflate(src.ctypes.data, src.size, out.ctypes.data, out.size, C.byref(got))
    if st == L.DZ_E_FORMAT:
        raise FormatError("corrupt lossless stream")
    L.check(st, "inflate")
    return out[: got.value]


def _layer_arrays(p: _Parsed, rec) -> tuple[str, np.ndarray, bytes, np.ndarray]:
    buf = np.frombuffer(p.data, dtype=np.uint8)
    name = bytes(buf[rec.name_off: rec.name_off + rec.name_len]).decode("utf-8")
    scales = buf[rec.scales_off: rec.scales_off + rec.scales_len]
    index = buf[rec.index_off: rec.index_off + rec.index_len]
    payload = buf[rec.payload_off: rec.payload_off + rec.payload_len]
    if p.config.lossless == LOSSLESS_DEFLATE:
        payload = _inflate(np.ascontiguousarray(payload), rec.rows, rec.cols, p.config)
    if payload.size % 4:
        raise FormatError("payload not a whole number of 32-bit words", offset=int(rec.payload_off + rec.payload_len))
    return name, payload, index, scales


def write_delta(cd: CompressedDelta, path) -> None:
    """Write a DZDL container (reference formats.py:60-97), byte-identical to the reference's
    writer: the producer side of the swap path, used after `solver.compress_model`."""
    import struct
    import zlib
    lossless = cd.config.lossless == LOSSLESS_DEFLATE
    header = {"base_model_id": cd.base_model_id, "bits": cd.config.bits, "sparsity": cd.config.sparsity,
              "group_size": cd.config.group_size, "layer_count": len(cd.layers),
              "calibration_fingerprint": cd.calibration_fingerprint, "damping": cd.config.damping,
              "block_size": cd.config.block_size, "codec": LOSSLESS_DEFLATE if lossless else LOSSLESS_OFF}
    hb = json.dumps(header, sort_keys=True).encode("utf-8")
    parts = [DELTA_MAGIC, struct.pack("<HHI", 1, 0x1 if lossless else 0, len(hb)), hb]
    for ld in cd.layers:
        name = ld.name.encode("utf-8")
        sc = np.ascontiguousarray(ld.scales, dtype="<f4").tobytes()
        idx = bytes(ld.index_stream)
        payload = np.ascontiguousarray(ld.packed_values, dtype="<u4").tobytes()
        if lossless:
            payload = zlib.compress(payload, 6)  # compress.py:556-557
        parts += [struct.pack("<H", len(name)), name, struct.pack("<III", ld.rows, ld.cols, len(sc)), sc,
                  struct.pack("<I", len(idx)), idx, struct.pack("<I", len(payload)), payload]
    with open(path, "wb") as f:
        f.write(b"".join(parts))


def read_delta(path) -> CompressedDelta:
    """Reference formats.read_delta (formats.py:102-169): host LayerDeltas of a DZDL file."""
    with open(path, "rb") as f:
        data = f.read()
    p = _parse(data)
    layers = []
    for rec in p.layers:
        name, payload, index, scales = _layer_arrays(p, rec)
        layers.append(LayerDelta(name=name, rows=int(rec.rows), cols=int(rec.cols),
                                 packed_values=payload.view("<u4").copy(), index_stream=index.tobytes(),
                                 scales=scales.view("<f4").copy(), bits=p.config.bits, sparsity=p.config.sparsity,
                                 group_size=p.config.group_size))
    return CompressedDelta(base_model_id=p.header["base_model_id"], layers=layers, config=p.config,
                           calibration_fingerprint=p.header["calibration_fingerprint"])


def inspect_delta(path) -> tuple[dict, list[LayerSizes], float]:
    """Reference formats.inspect_delta (formats.py:189-218): lenient like the reference — only the
    magic and truncation are checked (FormatError with the offset); the version, the configuration
    values and trailing bytes are not, and a bad JSON header raises json's own error."""
    import struct
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 4:
        raise FormatError("truncated file while reading magic", offset=0)
    if data[:4] != DELTA_MAGIC:
        raise FormatError("bad magic", offset=0)
    if len(data) < 12:
        raise FormatError("truncated file while reading the container header", offset=min(len(data), 8))
    (hlen,) = struct.unpack_from("<I", data, 8)
    if 12 + hlen > len(data):
        raise FormatError("truncated file while reading header", offset=12)
    header = json.loads(data[12:12 + hlen].decode("utf-8"))
    count = header["layer_count"]
    lib = L.lib()
    ptr, keep = _buf_ptr(data)
    recs = (L.DzDzdlLayer * max(count, 1))()
    off = C.c_int64(0)
    st = lib.dz_dzdl_parse_layers(ptr, len(data), 12 + hlen, count, recs, C.byref(off))
    if st == L.DZ_E_FORMAT:
        raise FormatError("truncated file while reading a layer record", offset=off.value)
    if st not in (L.DZ_OK, L.DZ_E_VALUE):  # DZ_E_VALUE = trailing bytes: ignored, as the reference does
        L.check(st, "dzdl layers")
    del keep
    sizes = []
    for rec in list(recs)[:count]:
        name = data[rec.name_off: rec.name_off + rec.name_len].decode("utf-8")
        sizes.append(LayerSizes(name, int(rec.rows), int(rec.cols), int(rec.scales_len), int(rec.index_len),
                                int(rec.payload_len)))
    dense = sum(s.dense16_bytes for s in sizes)
    return header, sizes, (dense / len(data) if data else 0.0)


class _PinnedLayer:
    """One layer's reference-layout bytes staged in pinned host memory and copied to the device
    asynchronously (the copy overlaps the parsing of the next layer)."""

    def __init__(self, ld_fields, device):
        from .device import RefDeltaDevice
        name, payload, index, scales, rows, cols, cfg = ld_fields
        self.ld = LayerDelta(name=name, rows=rows, cols=cols, packed_values=np.zeros(0, "<u4"), index_stream=b"",
                             scales=np.zeros(0, "<f4"), bits=cfg.bits, sparsity=cfg.sparsity,
                             group_size=cfg.group_size)
        pin = torch.empty(payload.size + index.size + scales.size + 48, dtype=torch.uint8).pin_memory()
        hv = pin.numpy()
        o1, o2 = payload.size, payload.size + index.size
        hv[:o1] = payload
        hv[o1:o2] = index
        hv[o2:o2 + scales.size] = scales
        self.pin = pin
        self.dev = RefDeltaDevice.from_pinned(self.ld, pin, (0, o1), (o1, o2), (o2, o2 + scales.size), device)


def load_delta(path, device=None):
    """Parse a DZDL file (mmap), inflate deflate payloads, stage each layer through pinned memory
    with async H2D copies, and re-lay it out on the GPU (nibbles validated). Returns
    (CompressedDelta metadata with empty host arrays, list of NativeDelta)."""
    from .device import require_cuda
    from .engine import NativeDelta
    dev = device or require_cuda()
    with open(path, "rb") as f:
        mm = mmap.mmap(f.fileno(), 0, access=mmap.ACCESS_READ) if os.path.getsize(path) else b""
    try:
        meta, staged = _stage_layers(mm, dev)  # every layer copied out of the mapping
    except BaseException as e:
        # the traceback's frames hold numpy views of the mapping: drop them so it can close, and the
        # caller sees the parser's own FormatError / EncodingError (formats.py:102-169)
        traceback.clear_frames(e.__traceback__)
        if isinstance(mm, mmap.mmap):
            mm.close()
        raise
    if isinstance(mm, mmap.mmap):
        mm.close()
    natives = [NativeDelta.from_ref_device(s.dev, s.ld) for s in staged]
    torch.cuda.current_stream(dev).synchronize()  # pinned staging buffers may be released now
    return meta, natives


def _stage_layers(buf, dev):
    """Parse a DZDL buffer and stage every layer in pinned host memory (async H2D started)."""
    p = _parse(buf)
    staged = []
    for rec in p.layers:
        name, payload, index, scales = _layer_arrays(p, rec)
        staged.append(_PinnedLayer((name, payload, index, scales, int(rec.rows), int(rec.cols), p.config), dev))
        del payload, index, scales  # views into the mapping: released before it closes
    meta = CompressedDelta(base_model_id=p.header["base_model_id"], layers=[s.ld for s in staged],
                           config=p.config, calibration_fingerprint=p.header["calibration_fingerprint"])
    return meta, staged


class DeltaPool:
    """Device-resident deltas of the served models: delta id -> one NativeDelta per layer.

    `load` swaps a DZDL file in (optionally as this rank's tensor-parallel shard: per-layer axes,
    "column" splits W's output rows, "row" its input columns, on native-block edges like
    stack.tp_bounds); `table(layer, ids)` builds the device table one fused launch routes to."""

    def __init__(self, device=None):
        from .device import require_cuda
        self.device = device or require_cuda()
        self.deltas: dict[int, list] = {}

    def load(self, delta_id: int, path, rank: int = 0, world: int = 1, axes=None) -> None:
        from .stack import shard_sub, split_units
        _, natives = load_delta(path, self.device)
        if world > 1:
            out = []
            for i, nat in enumerate(natives):
                ax = (axes or ["column"] * len(natives))[i]
                if ax == "column":
                    r0, r1 = split_units(nat.rows, world, 16)[rank]
                    out.append(shard_sub(nat, r0, r1, 0, nat.cols))
                else:
                    c0, c1 = split_units(nat.cols, world, 128)[rank]
                    out.append(shard_sub(nat, 0, nat.rows, c0, c1))
            natives = out
        self.deltas[int(delta_id)] = natives

    def evict(self, delta_id: int) -> None:
        self.deltas.pop(int(delta_id), None)

    def table(self, layer: int, ids):
        from .engine import DeltaTable
        nats = [self.deltas[int(d)][layer] for d in ids]
        return DeltaTable(nats, nats[0].rows, nats[0].cols)

    @property
    def nbytes(self) -> int:
        return sum(n.nbytes for v in self.deltas.values() for n in v)
