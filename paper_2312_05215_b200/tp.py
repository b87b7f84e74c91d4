"""Tensor parallelism for the decoupled linear (inference.py:162-243, §5.3).

The delta is partitioned exactly like its base (`_tp_grouped_linear`
inference.py:233-243): a column-parallel layer splits W's output rows (no collective), a
row-parallel layer splits W's input columns and sums the partial outputs (an all-reduce).

Packed-format sharding is exact and needs no dequantisation when the cut points fall on native
block edges (rows multiple of 16, columns multiple of 128 — every 70B shard at TP 2/4/8): the
shard is a sub-grid of the native 16x128 blocks (scales live inside the blocks). Other cut
points fall back to a GPU-dequantised bf16 shard (K1), still on the device.

`TpLinear` is one rank's shard of a linear with an NCCL all-reduce after row-parallel layers
(`torch.distributed`, one process per GPU).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .compress import dequantize_layer_device
from .core import AXIS_COLUMN, AXIS_ROW
from .device import bf16_from_numpy, require_cuda
from .engine import BLK_COLS, BLK_ROWS, DeltaTable, NativeBase, NativeDelta, Plan, sbmm_forward
from .errors import PartitionError


def _check_div(rows: int, cols: int, axis: str, n: int) -> None:
    if n < 1:
        raise PartitionError("worker count must be >= 1")
    if axis == AXIS_COLUMN:  # splits W's output rows (tp_partition(w.T, "column") divides w.T cols)
        if rows % n:
            raise PartitionError(f"{rows} columns not divisible by {n} workers")
    elif axis == AXIS_ROW:
        if cols % n:
            raise PartitionError(f"{cols} rows not divisible by {n} workers")
    else:
        raise PartitionError(f"unknown partition axis {axis!r}")


def shard_bounds(rows: int, cols: int, axis: str, n: int, i: int) -> tuple[int, int, int, int]:
    """(r0, r1, c0, c1) of shard i of W (out=rows, in=cols)."""
    _check_div(rows, cols, axis, n)
    if axis == AXIS_COLUMN:
        s = rows // n
        return i * s, (i + 1) * s, 0, cols
    s = cols // n
    return 0, rows, i * s, (i + 1) * s


def shard_native(nat: NativeDelta, axis: str, n: int, i: int, source_ld=None) -> NativeDelta:
    """Shard i of a resident delta, partitioned like its base."""
    r0, r1, c0, c1 = shard_bounds(nat.rows, nat.cols, axis, n, i)
    aligned = r0 % BLK_ROWS == 0 and c0 % BLK_COLS == 0 and (r1 % BLK_ROWS == 0 or r1 == nat.rows) \
        and (c1 % BLK_COLS == 0 or c1 == nat.cols)
    if nat.kind != L.DZ_KIND_DENSE and aligned:
        n16, nkb = -(-nat.rows // BLK_ROWS), -(-nat.cols // BLK_COLS)
        grid = nat.blocks.view(n16, nkb, -1)
        sub = grid[r0 // BLK_ROWS: -(-r1 // BLK_ROWS), c0 // BLK_COLS: -(-c1 // BLK_COLS)].contiguous()
        return NativeDelta(nat.kind, nat.qmax, r1 - r0, c1 - c0, sub.view(-1), nat.bits)
    if source_ld is None:
        raise PartitionError("unaligned shard of a native delta needs its source LayerDelta")
    dense = dequantize_layer_device(source_ld, torch.bfloat16)
    return NativeDelta.from_dense_bf16(dense[r0:r1, c0:c1].contiguous(), bits=nat.bits)


def tp_layer_forward(w: np.ndarray, lds: list, slots: np.ndarray, X: torch.Tensor, axis: str, n: int,
                     act: int = L.DZ_ACT_NONE) -> torch.Tensor:
    """One layer through n shards on this GPU (forward_model's TP branch, inference.py:267-283)."""
    dev = require_cuda()
    rows, cols = w.shape
    _check_div(rows, cols, axis, n)
    natives = [NativeDelta.from_layer_delta(ld, dev) for ld in lds]
    parts = []
    for i in range(n):
        r0, r1, c0, c1 = shard_bounds(rows, cols, axis, n, i)
        base = NativeBase(bf16_from_numpy(w[r0:r1, c0:c1], dev))
        table = DeltaTable([shard_native(nt, axis, n, i, ld) for nt, ld in zip(natives, lds)], r1 - r0, c1 - c0)
        plan = Plan(slots, table.kinds, len(table), device=dev)
        Xi = X if axis == AXIS_COLUMN else X[:, c0:c1].contiguous()
        parts.append(sbmm_forward(Xi, plan, base, table, y_dtype=torch.float32,
                                  act=act if axis == AXIS_COLUMN else L.DZ_ACT_NONE))
    if axis == AXIS_COLUMN:
        return torch.cat(parts, dim=1)
    y = parts[0]
    for p in parts[1:]:
        y = y + p  # shard order, like the reference's simulated all-reduce (inference.py:216-223)
    return torch.tanh(y) if act == L.DZ_ACT_TANH else y


class TpLinear:
    """This rank's shard of one decoupled linear; row-parallel outputs are all-reduced (NCCL).

    W (full, bf16) and the resident deltas are sharded here once at load time."""

    def __init__(self, W: torch.Tensor, natives: list[NativeDelta], axis: str, rank: int, world: int,
                 sources: list | None = None, group=None):
        rows, cols = int(W.shape[0]), int(W.shape[1])
        self.axis, self.rank, self.world, self.group = axis, rank, world, group
        r0, r1, c0, c1 = shard_bounds(rows, cols, axis, world, rank)
        self.c0, self.c1 = c0, c1
        self.base = NativeBase(W[r0:r1, c0:c1].contiguous())
        srcs = sources or [None] * len(natives)
        self.table = DeltaTable([shard_native(nt, axis, world, rank, s) for nt, s in zip(natives, srcs)],
                                r1 - r0, c1 - c0)

    def forward(self, X: torch.Tensor, plan: Plan, y_dtype=torch.bfloat16) -> torch.Tensor:
        """column: X is the full activation, returns this rank's output slice.
        row: X is this rank's input slice (the column-parallel output), returns the full sum."""
        Y = sbmm_forward(X, plan, self.base, self.table, y_dtype=y_dtype)
        if self.axis == AXIS_ROW and self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(Y, op=dist.ReduceOp.SUM, group=self.group)
        return Y
