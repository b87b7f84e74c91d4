"""GPU ΔCompress: the producer of packed layer deltas.

Reference: compress.py:178-186 (compute_hessian), :321-336 (_inverse_cholesky_factor),
:348-464 (obs_compress_layer), :508-548 (compress_model). Same names, arguments and errors.

Split of work:
  * the proxy Hessian H = X X^T + damping * mean(diag) * I (one cuBLAS DSYRK) and the
    propagation X <- (W_b + ΔW~) X (a plain f64 GEMM through torch);
  * the inverse-Hessian factor U (upper, H^-1 = U^T U) is one f64 Cholesky of the reversed H and
    a triangular inverse (cuSOLVER / cuBLAS through torch.linalg); the reference uses LAPACK;
  * the OBS column solver, the 2:4 mask choice, the RTN grid, the proxy loss and the packing
    into the reference layout are the `dz_obs_compress` kernels (csrc/dz_obs.cu).
Given the same U the solver reproduces the reference's codes, masks and scales bit for bit
(tests/test_gpu_obs.py); end to end, cuSOLVER's U differs from LAPACK's in the last bits, so
results agree to the tolerance those bits allow (a rare flipped rounding or mask decision).
"""

from __future__ import annotations

import ctypes as C
import hashlib
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .compress import SPARSITY_2_4, LayerDelta
from .core import WeightStack, as_matrix
from .device import require_cuda, stream_ptr
from .errors import CalibrationError, NumericDomainError, ShapeError
from .formats import CompressConfig, CompressedDelta


@dataclass
class CalibrationSet:
    """Per-sample input vectors, one column per sample (reference compress.py:76-99)."""

    samples: np.ndarray

    def __post_init__(self):
        self.samples = as_matrix(self.samples, "calibration samples")

    @property
    def input_dim(self) -> int:
        return self.samples.shape[0]

    @property
    def n_samples(self) -> int:
        return self.samples.shape[1]

    def fingerprint(self) -> int:
        h = hashlib.sha256()
        h.update(np.asarray(self.samples.shape, dtype="<i8").tobytes())
        h.update(np.ascontiguousarray(self.samples, dtype="<f8").tobytes())
        return int.from_bytes(h.digest()[:8], "little")


def _dev_f64(a, device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(device)


_CUBLAS = None


def _cublas():
    """torch's own cuBLAS (already loaded in the process), for DSYRK."""
    global _CUBLAS
    if _CUBLAS is None:
        import glob
        import os
        cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cublas", "lib",
                                       "libcublas.so.*")) + ["libcublas.so.12", "libcublas.so"]
        for c in cands:
            try:
                lib = C.CDLL(c)
                lib.cublasDsyrk_v2.restype = C.c_int
                _CUBLAS = lib
                break
            except OSError:
                continue
        if _CUBLAS is None:
            _CUBLAS = False
    return _CUBLAS


def hessian_device(x: torch.Tensor, damping: float) -> torch.Tensor:
    """H = X X^T + damping * mean(diag(X X^T)) * I on the device (compress.py:178-186).

    X X^T is symmetric, so it is one cuBLAS DSYRK (half the flops of the GEMM the reference
    runs) on torch's handle and stream, mirrored into the full matrix."""
    if damping < 0:
        raise ValueError("damping must be nonnegative")
    n, k = x.shape
    lib = _cublas()
    h = None
    if lib:
        x = x.contiguous()
        h = torch.zeros(n, n, dtype=torch.float64, device=x.device)
        one, zero = C.c_double(1.0), C.c_double(0.0)
        # column-major view: A = X^T (k x n, lda = k); C = A^T A, FILL_MODE_LOWER (0) = row-major upper
        st = lib.cublasDsyrk_v2(C.c_void_p(torch.cuda.current_blas_handle()), 0, 1, n, k, C.byref(one),
                                C.c_void_p(x.data_ptr()), k, C.byref(zero), C.c_void_p(h.data_ptr()), n)
        if st != 0:
            h = None
        else:
            h = torch.triu(h) + torch.triu(h, 1).T
    if h is None:  # cuBLAS without the symbol: the plain GEMM
        h = x @ x.T
    d = torch.diagonal(h)
    d += damping * torch.mean(d)
    return h


def compute_hessian(calib: CalibrationSet, damping: float) -> np.ndarray:
    """Reference signature (compress.py:178): the proxy Hessian as a host f64 matrix."""
    dev = require_cuda()
    return hessian_device(_dev_f64(calib.samples, dev), damping).cpu().numpy()


def inverse_cholesky_factor(h: torch.Tensor, name: str = "layer") -> torch.Tensor:
    """Upper U with H^-1 = U^T U (compress.py:321-336), f64 on the device.

    The reference factors H, inverts it and factors the inverse (LAPACK potrf, potrs, potrf).
    The same unique factor comes from one Cholesky and one triangular inverse: with J the
    reversal permutation and J H J = L L^T, U = J L^-1 J is upper triangular with a positive
    diagonal and U^T U = J (J H J)^-1 J = H^-1. That is 2 cuSOLVER/cuBLAS calls instead of 3
    and about half the flops."""
    if not bool(torch.isfinite(h).all()):
        raise NumericDomainError(f"hessian for layer {name!r} is not positive definite")
    lo, info = torch.linalg.cholesky_ex(torch.flip(h, (0, 1)))
    if int(info.item()) != 0:
        raise NumericDomainError(f"hessian for layer {name!r} is not positive definite")
    eye = torch.eye(h.shape[0], dtype=h.dtype, device=h.device)
    linv = torch.linalg.solve_triangular(lo, eye, upper=False)
    return torch.flip(linv, (0, 1)).contiguous()


@dataclass
class ObsResult:
    """Device outputs of one layer solve; `quantized` is the dense f64 ΔW~ (= dequantize_layer)."""

    packed: torch.Tensor
    index: torch.Tensor
    scales: torch.Tensor
    loss: torch.Tensor
    quantized: torch.Tensor


def _n_words(rows: int, cols: int, cfg: CompressConfig) -> int:
    n = rows * cols // 2 if cfg.sparsity == SPARSITY_2_4 else rows * cols
    if cfg.is_passthrough:
        return 2 * n
    per = 32 // cfg.bits
    return -(-n // per)


def obs_solve_device(delta: torch.Tensor, u: torch.Tensor | None, cfg: CompressConfig) -> ObsResult:
    """Run the GPU solver on a device f64 delta (consumed: it becomes the quantized delta)."""
    dev = delta.device
    rows, cols = delta.shape
    sparse = cfg.sparsity == SPARSITY_2_4
    if sparse and cols % 4 != 0:
        raise ShapeError(f"2:4 sparsity needs cols divisible by 4, got {cols}")
    c = L.DzObsCfg(cfg.bits, 1 if sparse else 0, cfg.group_size, cfg.block_size)
    lib = L.lib()
    packed = torch.empty(_n_words(rows, cols, cfg), dtype=torch.int32, device=dev)
    index = torch.empty(rows * cols // 8 + (1 if (rows * cols // 4) % 2 else 0) if sparse else 0,
                        dtype=torch.uint8, device=dev)
    ng = math.ceil(cols / cfg.group_size)
    scales = torch.empty(0 if cfg.is_passthrough else rows * ng, dtype=torch.float32, device=dev)
    loss = torch.zeros(1, dtype=torch.float64, device=dev)
    ws_bytes = lib.dz_obs_workspace_bytes(rows, cols, C.byref(c))
    if ws_bytes == 0:
        raise ValueError("dz_obs_compress: invalid configuration")
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    uptr = u.data_ptr() if u is not None else delta.data_ptr()  # U unused for the dense identity case
    L.check(lib.dz_obs_compress(delta.data_ptr(), uptr, rows, cols, C.byref(c), packed.data_ptr(),
                                index.data_ptr() if sparse else None,
                                scales.data_ptr() if scales.numel() else None, loss.data_ptr(),
                                ws.data_ptr(), ws_bytes, stream_ptr()), "obs_compress_layer")
    return ObsResult(packed, index, scales, loss, delta)


def _to_layer_delta(res: ObsResult, name: str, rows: int, cols: int, cfg: CompressConfig) -> LayerDelta:
    return LayerDelta(name=name, rows=rows, cols=cols,
                      packed_values=res.packed.cpu().numpy().view("<u4"),
                      index_stream=res.index.cpu().numpy().tobytes(),
                      scales=res.scales.cpu().numpy(), bits=cfg.bits, sparsity=cfg.sparsity,
                      group_size=cfg.group_size, proxy_loss=float(res.loss.item()))


def obs_compress_layer(delta, hessian, cfg: CompressConfig, name: str = "layer", u=None) -> LayerDelta:
    """Greedy OBS column compression of one layer delta on the GPU (compress.py:348-464).

    `u` (optional, host or device f64 [cols, cols]) supplies the inverse-Hessian factor instead
    of factoring `hessian` on the device."""
    delta = as_matrix(delta, "delta")
    hessian = as_matrix(hessian, "hessian")
    r, c = delta.shape
    if hessian.shape != (c, c):
        raise ShapeError(f"hessian shape {hessian.shape} does not match delta cols {c}")
    if cfg.sparsity == SPARSITY_2_4 and c % 4 != 0:
        raise ShapeError(f"layer {name!r}: 2:4 sparsity needs cols divisible by 4, got {c}")
    dev = require_cuda()
    d = _dev_f64(delta, dev)
    ut = None
    if not (cfg.is_passthrough and cfg.sparsity != SPARSITY_2_4):
        ut = _dev_f64(u, dev) if u is not None else inverse_cholesky_factor(_dev_f64(hessian, dev), name)
    return _to_layer_delta(obs_solve_device(d, ut, cfg), name, r, c, cfg)


def compress_model(w_f: WeightStack, w_b: WeightStack, calib: CalibrationSet, cfg: CompressConfig,
                   base_model_id: str = "base") -> CompressedDelta:
    """Compress every layer delta, propagating the calibration inputs through the reconstructed
    (base + ΔW~) weights (compress.py:508-548); the whole pass stays on the device."""
    if len(w_f) != len(w_b):
        raise ShapeError(f"stack depth mismatch: {len(w_f)} vs {len(w_b)}")
    for (nf, wf), (nb, wb) in zip(w_f.layers, w_b.layers):
        if wf.shape != wb.shape:
            raise ShapeError(f"layer {nf!r}/{nb!r} shape mismatch {wf.shape} vs {wb.shape}")
    if calib.input_dim != w_b.layers[0][1].shape[1]:
        raise ShapeError(f"calibration dim {calib.input_dim} does not match layer 0 input "
                         f"dim {w_b.layers[0][1].shape[1]}")
    dev = require_cuda()
    x = _dev_f64(calib.samples, dev)
    layers = []
    for (name, wf), (_, wb) in zip(w_f.layers, w_b.layers):
        if not bool(torch.any(x != 0)):
            raise CalibrationError(f"calibration inputs vanished at layer {name!r}")
        wb_t = _dev_f64(wb, dev)
        delta = _dev_f64(wf, dev) - wb_t
        ut = None
        if not (cfg.is_passthrough and cfg.sparsity != SPARSITY_2_4):
            ut = inverse_cholesky_factor(hessian_device(x, cfg.damping), name)
        res = obs_solve_device(delta, ut, cfg)
        layers.append(_to_layer_delta(res, name, wb.shape[0], wb.shape[1], cfg))
        x = (res.quantized + wb_t) @ x
    return CompressedDelta(base_model_id=base_model_id, layers=layers, config=cfg,
                           calibration_fingerprint=calib.fingerprint())
