"""Device plumbing: CUDA availability, streams, uploads of reference-layout deltas."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .errors import CudaError


_CUDA_OK = False  # set once the library loaded and a device was seen (checked on every call until then)


def require_cuda() -> torch.device:
    """The product path has no CPU fallback: fail loudly without a GPU or the extension."""
    global _CUDA_OK
    if not _CUDA_OK:
        L.lib()
        if not torch.cuda.is_available():
            raise CudaError("no CUDA device: the DeltaZip B200 path has no CPU fallback")
        _CUDA_OK = True
    return torch.device("cuda", torch.cuda.current_device())


_NVTX = [False]  # NVTX ranges around launches / layers / API calls (nsys, ncu --nvtx); off by default


def set_nvtx(on: bool = True) -> None:
    """Annotate launches (`dz_sbmm <out>x<in> T=<T>`), stack layers and drop-in API calls with NVTX
    ranges, for nsys timelines and `ncu --nvtx --nvtx-include`. Off: one list lookup per call."""
    _NVTX[0] = bool(on)


def nvtx_push(name: str) -> None:
    if _NVTX[0]:
        torch.cuda.nvtx.range_push(name)


def nvtx_pop() -> None:
    if _NVTX[0]:
        torch.cuda.nvtx.range_pop()


def stream_ptr() -> int:
    """cudaStream_t of the current stream (the raw handle; torch.cuda.current_stream() builds a
    Python Stream object per call, a measurable share of a small drop-in call)."""
    return torch._C._cuda_getCurrentRawStream(torch.cuda.current_device())


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def bf16_from_numpy(a, device) -> torch.Tensor:
    """f64/f32 host array -> bf16 device tensor (round-to-nearest-even, via f32 like torch)."""
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))
    return t.to(device=device, non_blocking=False).to(torch.bfloat16).contiguous()


class ErrFlag:
    """A device int the kernels set on a data error (e.g. corrupt index nibble)."""

    def __init__(self, device):
        self.t = torch.zeros(1, dtype=torch.int32, device=device)

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    def raise_if_set(self, what: str) -> None:
        code = int(self.t.item())  # host sync: upload/validation time only, never per forward
        if code:
            self.t.zero_()
            L.check(code, what)


class RefDeltaDevice:
    """A LayerDelta's reference-layout bytes resident in device memory (verbatim copy)."""

    def __init__(self, ld, device):
        self.rows, self.cols, self.bits = int(ld.rows), int(ld.cols), int(ld.bits)
        self.sparse = ld.sparsity == "two_of_four"
        self.group_size = int(ld.group_size)
        pv = np.ascontiguousarray(ld.packed_values, dtype="<u4")
        idx = np.frombuffer(bytes(ld.index_stream), dtype=np.uint8)
        sc = np.ascontiguousarray(ld.scales, dtype="<f4")
        # +16 bytes slack so empty arrays still have a valid device pointer
        self.packed = torch.zeros(pv.size + 4, dtype=torch.int32, device=device)
        self.index = torch.zeros(idx.size + 16, dtype=torch.uint8, device=device)
        self.scales = torch.zeros(sc.size + 4, dtype=torch.float32, device=device)
        if pv.size:
            self.packed[: pv.size].copy_(torch.from_numpy(pv.view(np.int32)))
        if idx.size:
            self.index[: idx.size].copy_(torch.from_numpy(idx.copy()))
        if sc.size:
            self.scales[: sc.size].copy_(torch.from_numpy(sc))
        self.struct = L.DzRefDelta(
            self.packed.data_ptr(), pv.size, self.index.data_ptr(), idx.size,
            self.scales.data_ptr(), sc.size, self.rows, self.cols, self.bits,
            1 if self.sparse else 0, self.group_size, 0)

    @classmethod
    def from_pinned(cls, ld, pin: torch.Tensor, r_packed, r_index, r_scales, device) -> "RefDeltaDevice":
        """Same device layout, filled by asynchronous copies from slices of a pinned host buffer
        (the DZDL loader's staging; the caller keeps `pin` alive until the stream syncs)."""
        self = cls.__new__(cls)
        self.rows, self.cols, self.bits = int(ld.rows), int(ld.cols), int(ld.bits)
        self.sparse = ld.sparsity == "two_of_four"
        self.group_size = int(ld.group_size)
        npk = (r_packed[1] - r_packed[0]) // 4
        nix = r_index[1] - r_index[0]
        nsc = (r_scales[1] - r_scales[0]) // 4
        self.packed = torch.zeros(npk + 4, dtype=torch.int32, device=device)
        self.index = torch.zeros(nix + 16, dtype=torch.uint8, device=device)
        self.scales = torch.zeros(nsc + 4, dtype=torch.float32, device=device)
        if npk:
            self.packed.view(torch.uint8)[: 4 * npk].copy_(pin[r_packed[0]: r_packed[1]], non_blocking=True)
        if nix:
            self.index[:nix].copy_(pin[r_index[0]: r_index[1]], non_blocking=True)
        if nsc:
            self.scales.view(torch.uint8)[: 4 * nsc].copy_(pin[r_scales[0]: r_scales[1]], non_blocking=True)
        self.struct = L.DzRefDelta(
            self.packed.data_ptr(), npk, self.index.data_ptr(), nix, self.scales.data_ptr(), nsc,
            self.rows, self.cols, self.bits, 1 if self.sparse else 0, self.group_size, 0)
        return self
