"""ctypes binding of the C ABI in `include/dz_b200.h` (library `_dz_b200.so`, built in-tree).

There is no CPU fallback: if the library is missing every entry point raises CudaError.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import (
    CudaError, EncodingError, FormatError, PartitionError, ShapeError, UnknownDeltaError,
)

LIB_PATH = os.environ.get("DZ_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_dz_b200.so")

DZ_OK, DZ_E_SHAPE, DZ_E_ENCODING, DZ_E_FORMAT, DZ_E_PARTITION = 0, 1, 2, 3, 4
DZ_E_UNKNOWN, DZ_E_VALUE, DZ_E_UNSUPPORTED, DZ_E_CUDA = 5, 6, 7, 8
DZ_F32, DZ_BF16, DZ_F64 = 0, 1, 2
DZ_ACT_NONE, DZ_ACT_TANH = 0, 1
DZ_KIND_SPARSE4, DZ_KIND_SPARSE2, DZ_KIND_DENSE, DZ_KIND_SPARSE3 = 1, 2, 3, 4


class DzRefDelta(C.Structure):
    _fields_ = [
        ("packed", C.c_void_p), ("n_words", C.c_int64),
        ("index", C.c_void_p), ("index_bytes", C.c_int64),
        ("scales", C.c_void_p), ("n_scales", C.c_int64),
        ("rows", C.c_int32), ("cols", C.c_int32), ("bits", C.c_int32),
        ("sparse", C.c_int32), ("group_size", C.c_int32), ("_pad", C.c_int32),
    ]


class DzNativeDelta(C.Structure):
    _fields_ = [("blocks", C.c_void_p), ("kind", C.c_int32), ("qmax", C.c_int32),
                ("rows", C.c_int32), ("cols", C.c_int32), ("_reserved", C.c_uint8 * 40),
                ("tmap", C.c_uint64 * 16)]


class DzObsCfg(C.Structure):
    _fields_ = [("bits", C.c_int32), ("sparse", C.c_int32), ("group_size", C.c_int32), ("block_size", C.c_int32)]


class DzJob(C.Structure):
    _fields_ = [("slot", C.c_int32), ("tok_begin", C.c_int32), ("tok_count", C.c_int32),
                ("kind", C.c_int32)]


class DzSbmmArgs(C.Structure):
    _fields_ = [
        ("X", C.c_void_p), ("ldx", C.c_int64),
        ("Y", C.c_void_p), ("ldy", C.c_int64),
        ("y_dtype", C.c_int32), ("act", C.c_int32),
        ("T", C.c_int32), ("out", C.c_int32), ("in_", C.c_int32),
        ("base", C.c_void_p),
        ("table", C.c_void_p), ("n_slots", C.c_int32),
        ("order", C.c_void_p),
        ("jobs", C.c_void_p), ("n_jobs", C.c_int32),
        ("workspace", C.c_void_p),
        ("grid", C.c_int32), ("debug", C.c_int32),
        ("perm", C.c_void_p), ("xs", C.c_void_p),
        ("n_pf_jobs", C.c_int32), ("t_pf", C.c_int32),
        ("ldxs", C.c_int64),
        ("base_splits", C.c_int32), ("delta_splits", C.c_int32),
        ("tp", C.c_void_p),
        ("n_jobs_dev", C.c_void_p),
        ("keep_planes", C.c_int32), ("prefill_variant", C.c_int32),
        ("fused_merge", C.c_int32), ("mixed_parts", C.c_int32),
        ("next", C.c_void_p),
        ("pf_counts_dev", C.c_void_p),
        ("sparse_job_tokens", C.c_int32), ("_pad6", C.c_int32),
    ]


class DzTpCtx(C.Structure):
    _fields_ = [("peer_R", C.c_void_p), ("peer_flags", C.c_void_p), ("sync", C.c_void_p),
                ("max_elems", C.c_int64), ("rank", C.c_int32), ("world", C.c_int32)]


class DzDzdlInfo(C.Structure):
    _fields_ = [("version", C.c_int32), ("flags", C.c_int32), ("lossless", C.c_int32), ("_pad", C.c_int32),
                ("header_off", C.c_int64), ("header_len", C.c_int64), ("layers_off", C.c_int64)]


class DzDzdlLayer(C.Structure):
    _fields_ = [("name_off", C.c_int64), ("name_len", C.c_int32), ("rows", C.c_int32), ("cols", C.c_int32),
                ("_pad", C.c_int32), ("scales_off", C.c_int64), ("scales_len", C.c_int64),
                ("index_off", C.c_int64), ("index_len", C.c_int64), ("payload_off", C.c_int64),
                ("payload_len", C.c_int64)]


# symbol -> (restype, argtypes); every symbol include/dz_b200.h declares
SIGNATURES = {
    "dz_version": (C.c_char_p, []),
    "dz_strerror": (C.c_char_p, [C.c_int]),
    "dz_unpack": (C.c_int, [C.POINTER(DzRefDelta), C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "dz_unpack_codes": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p]),
    "dz_decode_index": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                  C.c_void_p]),
    "dz_native_sparse_bytes": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32]),
    "dz_repack_sparse": (C.c_int, [C.POINTER(DzRefDelta), C.c_void_p, C.c_void_p, C.c_void_p]),
    "dz_unpack_native": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                   C.c_int64, C.c_void_p]),
    "dz_native_dense_bytes": (C.c_int64, [C.c_int32, C.c_int32]),
    "dz_pack_dense_bf16": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "dz_base_init": (C.c_int, [C.POINTER(DzNativeDelta), C.c_void_p, C.c_int64, C.c_int32, C.c_int32]),
    "dz_native_delta_init": (C.c_int, [C.POINTER(DzNativeDelta), C.c_void_p, C.c_int32, C.c_int32, C.c_int32]),
    "dz_pad_x": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p]),
    "dz_plan_max_jobs": (C.c_int32, [C.c_int32]),
    "dz_plan": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                          C.c_int32, C.POINTER(C.c_int32), C.c_int32]),
    "dz_plan_mixed": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                C.POINTER(C.c_int32), C.c_int32]),
    "dz_sbmm_workspace_bytes": (C.c_size_t, [C.c_int32, C.c_int32]),
    "dz_sbmm_chain_desc_bytes": (C.c_size_t, [C.c_int32]),
    "dz_sbmm_chain_encode": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_size_t, C.POINTER(C.c_int32)]),
    "dz_sbmm_chain": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
    "dz_sbmm_prefill": (C.c_int, [C.POINTER(DzSbmmArgs), C.c_void_p]),
    "dz_gather_rows": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int64,
                                 C.c_void_p]),
    "dz_sbmm": (C.c_int, [C.POINTER(DzSbmmArgs), C.c_void_p]),
    "dz_sbmm_ctas_per_sm": (C.c_int, []),
    "dz_dzdl_parse_header": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(DzDzdlInfo), C.POINTER(C.c_int64)]),
    "dz_dzdl_parse_layers": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int32, C.c_void_p,
                                       C.POINTER(C.c_int64)]),
    "dz_inflate": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]),
    "dz_plan_device": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                 C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "dz_plan_mixed_device": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                       C.c_void_p]),
    "dz_admit_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "dz_obs_workspace_bytes": (C.c_size_t, [C.c_int32, C.c_int32, C.POINTER(DzObsCfg)]),
    "dz_obs_compress": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.POINTER(DzObsCfg), C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "dz_peer_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "dz_peer_free": (C.c_int, [C.c_void_p]),
    "dz_ipc_handle": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dz_ipc_open": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "dz_ipc_close": (C.c_int, [C.c_void_p]),
}

_lib = None


def lib():
    """Load (once) and return the CDLL. Raises CudaError when the extension is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CudaError(f"CUDA extension not built: {LIB_PATH} missing (run __graft_entry__.build())")
        try:
            L = C.CDLL(LIB_PATH)
        except OSError as e:  # pragma: no cover
            raise CudaError(f"cannot load {LIB_PATH}: {e}") from e
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int, what: str = "") -> None:
    """Map a DZ_* status to the reference exception class."""
    if status == DZ_OK:
        return
    msg = lib().dz_strerror(status).decode()
    if what:
        msg = f"{what}: {msg}"
    if status == DZ_E_SHAPE:
        raise ShapeError(msg)
    if status == DZ_E_ENCODING:
        raise EncodingError(msg)
    if status == DZ_E_FORMAT:
        raise FormatError(msg)
    if status == DZ_E_PARTITION:
        raise PartitionError(msg)
    if status == DZ_E_UNKNOWN:
        raise UnknownDeltaError(msg)
    if status in (DZ_E_VALUE, DZ_E_UNSUPPORTED):
        raise ValueError(msg)
    raise CudaError(msg)
