"""DeltaZip serving hot path, B200-native (sm_100a CUDA behind a C ABI).

Drop-in for the reference package `deltazip` on the serving path: the same public names
(`__init__.py:3-32` of the reference) for the decoupled linear, SBMM, TP and the packed-delta
format, plus the device-resident throughput API in `engine`.
"""

from .compress import (
    SPARSITY_2_4,
    SPARSITY_NONE,
    LayerDelta,
    decode_mask_indices,
    dequantize_layer,
    dequantize_layer_device,
    encode_mask_indices,
    pack_codes,
    unpack_codes,
)
from .core import AXIS_COLUMN, AXIS_ROW, Matrix, WeightStack, as_matrix
from .errors import (
    CalibrationError,
    CudaError,
    DeltaZipError,
    EncodingError,
    FormatError,
    NumericDomainError,
    PartitionError,
    ShapeError,
    TraceError,
    UnknownDeltaError,
)
from .inference import (
    BatchInput,
    DeltaHandle,
    TpLayout,
    decoupled_linear,
    forward_model,
    group_by_delta,
    sbmm,
    tp_forward,
    tp_partition,
)

from .device import set_nvtx
from .resident import clear as clear_resident_cache, invalidate as invalidate_resident
from .formats import CompressConfig, CompressedDelta, inspect_delta, read_delta, write_delta
from .solver import CalibrationSet, compress_model, compute_hessian, obs_compress_layer

__version__ = "0.1.0"
