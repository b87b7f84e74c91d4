"""Device-resident serving objects and the throughput API over the fused SBMM kernel (K2).

- `NativeDelta`  one layer delta uploaded once: the reference bytes are copied to HBM, every index
                 nibble is validated (FormatError here, at load time), and 2:4 deltas with 2/3/4-bit
                 codes are re-laid out into mma.sp-native 16x128 blocks (same bytes per parameter).
                 Other variants (dense, 8/16-bit, odd group sizes) are dequantised on the GPU (K1)
                 to bf16 and stored as dense native blocks — still GPU, never a CPU path.
- `NativeBase`   the shared base weight W [out, in] in dense native blocks.
- `DeltaTable`   the device table of NativeDeltas one linear layer can route tokens to.
- `Plan`         the batch plan (group_by_delta, inference.py:106-123) for one token->slot map;
                 shared by every linear of a decode step.
- `sbmm_forward` Y = X W^T + SBMM(X, ΔW_slot) in one persistent launch.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _lib as L
from .compress import SPARSITY_2_4, dequantize_layer_device
from .device import _NVTX, ErrFlag, RefDeltaDevice, nvtx_pop, nvtx_push, require_cuda, stream_ptr
from .errors import ShapeError, UnknownDeltaError

BLK_ROWS, BLK_COLS = 16, 128


def _ceil(a: int, b: int) -> int:
    return -(-a // b)


class NativeDelta:
    """One LayerDelta resident on the GPU in kernel-native form."""

    def __init__(self, kind: int, qmax: int, rows: int, cols: int, blocks: torch.Tensor, bits: int):
        self.kind, self.qmax, self.rows, self.cols, self.blocks, self.bits = kind, qmax, rows, cols, blocks, bits

    @property
    def nbytes(self) -> int:
        return self.blocks.numel()

    @staticmethod
    def sparse_native_ok(ld) -> bool:
        ng = _ceil(int(ld.cols), int(ld.group_size))
        return (ld.sparsity == SPARSITY_2_4 and int(ld.bits) in (2, 3, 4)
                and (int(ld.group_size) % BLK_COLS == 0 or ng == 1))

    @classmethod
    def from_layer_delta(cls, ld, device=None) -> "NativeDelta":
        dev = device or require_cuda()
        return cls.from_ref_device(RefDeltaDevice(ld, dev), ld)

    @classmethod
    def from_ref_device(cls, ref: RefDeltaDevice, ld) -> "NativeDelta":
        """Upload-time re-layout of reference-layout bytes already on the device (`ld` supplies
        the configuration: sparsity, bits, group size)."""
        dev = ref.packed.device
        lib = L.lib()
        err = ErrFlag(dev)
        if cls.sparse_native_ok(ld):
            nbytes = lib.dz_native_sparse_bytes(ref.rows, ref.cols, ref.bits)
            blocks = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            L.check(lib.dz_repack_sparse(ref.struct, blocks.data_ptr(), err.ptr, stream_ptr()), "upload delta")
            err.raise_if_set("corrupt index stream: kept positions not strictly increasing")
            kind = {2: L.DZ_KIND_SPARSE2, 3: L.DZ_KIND_SPARSE3, 4: L.DZ_KIND_SPARSE4}[ref.bits]
            return cls(kind, (1 << (ref.bits - 1)) - 1, ref.rows, ref.cols, blocks, ref.bits)
        dense = dequantize_layer_device(ld, torch.bfloat16, ref=ref)  # raises FormatError / EncodingError
        return cls.from_dense_bf16(dense, bits=ref.bits)

    @classmethod
    def from_dense_bf16(cls, W: torch.Tensor, bits: int = 16) -> "NativeDelta":
        blocks = pack_dense(W)
        return cls(L.DZ_KIND_DENSE, 0, W.shape[0], W.shape[1], blocks, bits)

    def to_dense_f32(self) -> torch.Tensor:
        """Inverse view (parity check of the re-layout)."""
        out = torch.empty(self.rows, self.cols, dtype=torch.float32, device=self.blocks.device)
        if self.kind == L.DZ_KIND_DENSE:
            raise ValueError("dense native deltas are already bf16 matrices")
        L.check(L.lib().dz_unpack_native(self.blocks.data_ptr(), self.rows, self.cols, self.bits, self.qmax,
                                         out.data_ptr(), self.cols, stream_ptr()), "unpack_native")
        return out


def pack_dense(W: torch.Tensor) -> torch.Tensor:
    if W.dim() != 2 or W.dtype != torch.bfloat16 or not W.is_cuda:
        raise ShapeError("pack_dense expects a 2-D bf16 CUDA tensor")
    W = W.contiguous()
    rows, cols = W.shape
    nbytes = L.lib().dz_native_dense_bytes(rows, cols)
    blocks = torch.empty(nbytes, dtype=torch.uint8, device=W.device)
    L.check(L.lib().dz_pack_dense_bf16(W.data_ptr(), W.stride(0), rows, cols, blocks.data_ptr(), stream_ptr()),
            "pack base")
    return blocks


def table_bytes(deltas: list[NativeDelta]) -> np.ndarray:
    """Host-encoded dz_native_delta entries (192 B each, with their TMA descriptors)."""
    n = max(1, len(deltas))
    arr = (L.DzNativeDelta * n)()
    for i, d in enumerate(deltas):
        L.check(L.lib().dz_native_delta_init(C.byref(arr[i]), d.blocks.data_ptr(), d.kind, d.rows, d.cols),
                "table entry")
    return np.frombuffer(C.string_at(C.addressof(arr), C.sizeof(arr)), dtype=np.uint8).copy()


class NativeBase:
    """Shared base weight W_base [out, in] (bf16), kept in its natural row-major layout: the fused
    kernel streams it with 128B-swizzled TMA tiles straight into tcgen05 MMAs. Rows are padded to
    a 16-byte multiple only when `in` is not a multiple of 8 (TMA row-stride rule)."""

    def __init__(self, W: torch.Tensor):
        if W.dim() != 2 or W.dtype != torch.bfloat16 or not W.is_cuda:
            raise ShapeError("base weight must be a 2-D bf16 CUDA tensor")
        self.out, self.inp = int(W.shape[0]), int(W.shape[1])
        if W.stride(1) != 1 or W.stride(0) % 8 or W.data_ptr() % 16:
            ld = _ceil(self.inp, 8) * 8
            Wp = torch.zeros(self.out, ld, dtype=torch.bfloat16, device=W.device)
            Wp[:, : self.inp] = W
            W = Wp
        self.W = W
        e = L.DzNativeDelta()
        L.check(L.lib().dz_base_init(C.byref(e), W.data_ptr(), W.stride(0), self.out, self.inp), "base entry")
        raw = np.frombuffer(C.string_at(C.addressof(e), C.sizeof(e)), dtype=np.uint8).copy()
        self.entry = torch.from_numpy(raw).to(W.device)

    @property
    def nbytes(self) -> int:
        return self.out * self.inp * 2


class DeltaTable:
    """Device table of the deltas one linear layer serves (slot i -> deltas[i])."""

    def __init__(self, deltas: list[NativeDelta], out: int, inp: int):
        for d in deltas:
            if (d.rows, d.cols) != (out, inp):
                raise ShapeError(f"delta shape ({d.rows}, {d.cols}) != base ({out}, {inp})")
        self.deltas = list(deltas)
        self.out, self.inp = out, inp
        dev = deltas[0].blocks.device if deltas else require_cuda()
        self.dev = torch.from_numpy(table_bytes(deltas)).to(dev)
        self.kinds = np.array([d.kind for d in deltas] or [L.DZ_KIND_SPARSE4], dtype=np.int32)

    def __len__(self) -> int:
        return len(self.deltas)


PF_MIN = int(os.environ.get("DZ_PF_MIN", "192"))  # tokens per delta group routed to the prefill kernel
# (7B stacks: one 128-token group is faster on the decode kernel, one 256-token group on K3;
#  profiles/r01_ab_pf_min.txt)


class Plan:
    """Batch plan (group_by_delta, inference.py:106-123), uploaded to the device.

    Decode plan (no group reaches `pf_min` tokens): stable sort of tokens by slot + job list
    (dz_plan). Mixed plan: groups of >= pf_min tokens become prefill jobs for K3 over a staged
    (permuted) copy of X and the remaining tokens are planned for K2 (dz_plan_mixed)."""

    def __init__(self, slots, kinds: np.ndarray, n_slots: int, with_base: bool = True, device=None,
                 upload: bool = True, pf_min: int | None = None, sparse_job_tokens: int | None = None):
        s = np.ascontiguousarray(np.asarray(slots, dtype=np.int32).ravel())
        self.T = int(s.size)
        lib = L.lib()
        if sparse_job_tokens is None:  # 16-token 2:4 jobs (decode each chunk once per 16 tokens) when
            # some group is wider than 8 tokens; results do not depend on the width
            cnt = np.bincount(s, minlength=max(n_slots, 1)) if s.size and s.min() >= 0 else np.zeros(1, int)
            sparse_job_tokens = 16 if cnt.max(initial=0) > 8 else 8
        self.sparse_job_tokens = int(sparse_job_tokens)
        maxj = lib.dz_plan_max_jobs(self.T)
        order = np.zeros(max(self.T, 1), dtype=np.int32)
        perm = np.zeros(max(self.T, 1), dtype=np.int32)
        jobs = (L.DzJob * max(maxj, 1))()
        nj, npf, tpf = C.c_int32(0), C.c_int32(0), C.c_int32(0)
        kinds = np.ascontiguousarray(kinds, dtype=np.int32)
        self.pf_min = PF_MIN if pf_min is None else int(pf_min)
        st = lib.dz_plan_mixed(s.ctypes.data, self.T, kinds.ctypes.data, n_slots, 1 if with_base else 0,
                               self.pf_min, perm.ctypes.data, order.ctypes.data, jobs, maxj, C.byref(nj),
                               C.byref(npf), C.byref(tpf), self.sparse_job_tokens)
        if st == L.DZ_E_UNKNOWN:
            raise UnknownDeltaError("a token references a slot outside the delta table")
        L.check(st, "plan")
        self.n_jobs, self.n_pf_jobs, self.t_pf = int(nj.value), int(npf.value), int(tpf.value)
        self.order_host = order[: self.T].copy()
        self.perm_host = perm[: self.T].copy() if self.t_pf > 0 else None
        self.jobs_host = np.frombuffer(C.string_at(C.addressof(jobs), C.sizeof(L.DzJob) * max(self.n_jobs, 1)),
                                       dtype=np.int32).reshape(-1, 4)[: self.n_jobs].copy()
        self.jobs_bytes = np.frombuffer(C.string_at(C.addressof(jobs), C.sizeof(L.DzJob) * max(maxj, 1)),
                                        dtype=np.uint8).copy()
        self.with_base = with_base
        self.order = self.jobs = self.perm = None
        if upload:
            dev = device or require_cuda()
            self.order = torch.from_numpy(order).to(dev)
            self.jobs = torch.from_numpy(self.jobs_bytes).to(dev)
            if self.t_pf > 0:
                self.perm = torch.from_numpy(perm).to(dev)


class DevicePlan:
    """On-device plan: the token -> slot map stays on the GPU and each `update`
    enqueues one planner CTA, so a serving loop (or a captured CUDA graph of it) needs no host
    round trip.

    mixed=False (default): dz_plan_device — the decode plan (same stable group_by_delta and job cut
    as `Plan` with pf_min=0). mixed=True: dz_plan_mixed_device — `Plan`'s mixed plan: groups of
    >= pf_min tokens staged for the tensor-core prefill kernel (K3), the rest planned for K2; the
    counts (prefill jobs, decode jobs, staged prefill rows) stay on the device."""

    def __init__(self, T: int, kinds: np.ndarray, n_slots: int, with_base: bool = True, device=None,
                 mixed: bool = False, pf_min: int | None = None, sparse_job_tokens: int = 16):
        dev = device or require_cuda()
        lib = L.lib()
        self.T, self.n_slots, self.with_base, self.mixed = int(T), int(n_slots), with_base, mixed
        self.sparse_job_tokens = int(sparse_job_tokens)  # 8: the narrow kernel, for decode-only batches
        self.pf_min = (PF_MIN if pf_min is None else int(pf_min)) if mixed else 0
        self.kinds_dev = torch.from_numpy(np.ascontiguousarray(kinds, dtype=np.int32)).to(dev)
        self.max_jobs = int(lib.dz_plan_max_jobs(self.T))
        pf_cap = self.T if mixed else 0  # prefill region of the job list (decode jobs start at jobs[T])
        self.n_jobs = pf_cap + self.max_jobs  # capacity: the kernels read the device counts
        self.order = torch.zeros(max(self.T, 1), dtype=torch.int32, device=dev)
        self.jobs = torch.zeros(max(self.n_jobs, 1) * C.sizeof(L.DzJob), dtype=torch.uint8, device=dev)
        self.n_jobs_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        self.counts = torch.zeros(3, dtype=torch.int32, device=dev)  # mixed: prefill jobs, decode jobs, t_pf
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.t_pf, self.n_pf_jobs = 0, pf_cap
        self.perm = torch.zeros(max(self.T, 1), dtype=torch.int32, device=dev) if mixed else None

    def update(self, slots_dev: torch.Tensor) -> "DevicePlan":
        if slots_dev.numel() != self.T or slots_dev.dtype != torch.int32 or not slots_dev.is_cuda:
            raise ShapeError("slots must be an int32 CUDA tensor of T entries")
        lib = L.lib()
        if self.mixed:
            L.check(lib.dz_plan_mixed_device(slots_dev.data_ptr(), self.T, self.kinds_dev.data_ptr(), self.n_slots,
                                             1 if self.with_base else 0, self.pf_min, self.perm.data_ptr(),
                                             self.order.data_ptr(), self.jobs.data_ptr(), self.counts.data_ptr(),
                                             self.err.data_ptr(), self.sparse_job_tokens, stream_ptr()),
                    "device mixed plan")
        else:
            L.check(lib.dz_plan_device(slots_dev.data_ptr(), self.T, self.kinds_dev.data_ptr(), self.n_slots,
                                       1 if self.with_base else 0, self.order.data_ptr(), self.jobs.data_ptr(),
                                       self.max_jobs, self.n_jobs_dev.data_ptr(), self.err.data_ptr(),
                                       self.sparse_job_tokens, stream_ptr()), "device plan")
        return self

    def check(self) -> None:
        """Host sync: raise the reference's error for a slot outside the table (inference.py:135-137)."""
        code = int(self.err.item())
        if code == L.DZ_E_UNKNOWN:
            raise UnknownDeltaError("a token references a slot outside the delta table")
        L.check(code, "device plan")


class Workspace:
    """Per-(T, out) scratch for the fused kernel: scheduler + tile counters (zeroed once; the
    kernel resets them itself) and the fp32 partial buffers."""

    def __init__(self):
        self._bufs: dict[tuple, torch.Tensor] = {}

    def get(self, T: int, out: int, device) -> torch.Tensor:
        need = int(L.lib().dz_sbmm_workspace_bytes(T, out))
        device = torch.device(device)
        key = (device.type, device.index if device.index is not None else torch.cuda.current_device())
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < need:
            buf = torch.zeros(max(need, 256), dtype=torch.uint8, device=device)
            self._bufs[key] = buf
        return buf


_default_ws = Workspace()


def prepare_x(X: torch.Tensor) -> torch.Tensor:
    """Kernel contract: bf16, row stride >= ceil128(in), zero columns in..ceil128(in), 16 B aligned."""
    if X.dim() != 2 or X.dtype != torch.bfloat16 or not X.is_cuda:
        raise ShapeError("X must be a 2-D bf16 CUDA tensor [T, in]")
    T, inp = X.shape
    ldp = _ceil(inp, BLK_COLS) * BLK_COLS
    if ldp == inp and X.stride(1) == 1 and X.stride(0) % 8 == 0 and X.data_ptr() % 16 == 0:
        return X
    Xp = torch.empty(T, ldp, dtype=torch.bfloat16, device=X.device)
    L.check(L.lib().dz_pad_x(X.data_ptr(), X.stride(0), T, inp, Xp.data_ptr(), ldp, stream_ptr()), "pad x")
    return Xp


def sbmm_forward(X: torch.Tensor, plan: Plan, base: NativeBase | None, table: DeltaTable,
                 y_dtype: torch.dtype = torch.bfloat16, act: int = L.DZ_ACT_NONE, Y: torch.Tensor | None = None,
                 workspace: Workspace | None = None, grid: int = 0, debug: int = 0,
                 base_splits: int = 0, tp=None, delta_splits: int = 0, next_args: int = 0,
                 prefill_variant: int = 0, fused_merge: bool = False, overlap_sms: int | None = None) -> torch.Tensor:
    """Y[T, out] = X W_base^T + ΔW_{slot(t)} x_t for all t, one fused launch (inference.py:126-154).

    next_args: device address of the next linear's dz_sbmm_args (see `sbmm_args`), or 0; CTAs that
    run out of work then warm L2 with that launch's first weight stages.
    prefill_variant: K3's delta product for mixed plans (0 = 2:4-sparse tcgen05; 1 / 2 = the
    dense-dequantised variant with 128- / 256-row items, for A/B runs and equivalence tests).
    fused_merge: write Y inside the SBMM kernel (combiner warp) instead of a k_finalize launch.
    overlap_sms: mixed plans only — SMs given to the prefill kernel (K3) while the decode kernel
    (K2) runs on the rest, concurrently on a second stream (None / 0: one after the other, the
    default: both kernels need every SM — K3 its tensor cores, K2 its decode warps — so a split
    measured 2-19% slower on cfg3, profiles/r02_ab_cfg3_overlap.txt; -1: the split from
    `split_sms`)."""
    if _NVTX[0]:
        nvtx_push(f"dz_sbmm {table.out}x{table.inp} T={X.shape[0]}")
        try:
            return _sbmm_forward(X, plan, base, table, y_dtype, act, Y, workspace, grid, debug, base_splits, tp,
                                 delta_splits, next_args, prefill_variant, fused_merge, overlap_sms)
        finally:
            nvtx_pop()
    return _sbmm_forward(X, plan, base, table, y_dtype, act, Y, workspace, grid, debug, base_splits, tp,
                         delta_splits, next_args, prefill_variant, fused_merge, overlap_sms)


def _sbmm_forward(X, plan, base, table, y_dtype, act, Y, workspace, grid, debug, base_splits, tp, delta_splits,
                  next_args, prefill_variant, fused_merge, overlap_sms) -> torch.Tensor:
    a, Y, keep = sbmm_args(X, plan, base, table, y_dtype, act, Y, workspace, grid, debug, base_splits, tp,
                           delta_splits)
    a.prefill_variant = prefill_variant
    a.fused_merge = 1 if fused_merge else 0
    a.next = next_args or None
    lib = L.lib()
    sms = _sm_count(X.device)
    pf_sms = 0
    if plan.perm is not None and grid == 0 and plan.n_pf_jobs > 0 and plan.n_jobs > plan.n_pf_jobs:
        pf_sms = 0 if not overlap_sms else split_sms(plan, table, X.shape[1], sms) if overlap_sms < 0 else overlap_sms
    if pf_sms <= 0 or pf_sms >= sms:
        L.check(lib.dz_sbmm(C.byref(a), stream_ptr()), "sbmm")
        return Y
    # stage X once, then K3 on an auxiliary stream with pf_sms SMs while K2 runs on the rest: a
    # tensor-bound and an HBM-bound kernel share the machine (graph-capturable fork / join)
    main = torch.cuda.current_stream(X.device)
    aux = _aux_stream(X.device)
    a.mixed_parts = 1
    L.check(lib.dz_sbmm(C.byref(a), main.cuda_stream), "sbmm stage")
    aux.wait_stream(main)
    a.mixed_parts, a.grid = 2, pf_sms
    L.check(lib.dz_sbmm(C.byref(a), aux.cuda_stream), "sbmm prefill")
    a.mixed_parts, a.grid = 4, sms - pf_sms
    L.check(lib.dz_sbmm(C.byref(a), main.cuda_stream), "sbmm decode")
    main.wait_stream(aux)
    return Y


_AUX: dict = {}
_SMS: dict = {}


def _aux_stream(device) -> torch.cuda.Stream:
    key = torch.device(device).index
    if key not in _AUX:
        _AUX[key] = torch.cuda.Stream(device=device)
    return _AUX[key]


def _sm_count(device) -> int:
    key = torch.device(device).index
    if key not in _SMS:
        _SMS[key] = torch.cuda.get_device_properties(device).multi_processor_count
    return _SMS[key]


def split_sms(plan, table, inp: int, sms: int) -> int:
    """SMs for K3 when K3 and K2 of a mixed plan run concurrently: balance the prefill part's tensor
    time (3 flops per staged token per weight: base GEMM + kept 2:4 delta MACs, at ~6.5 TFLOP/s per
    SM sustained by K3) against the decode part's HBM time (base + the decode groups' deltas at
    ~45 GB/s per SM, capped by ~6 TB/s)."""
    out = table.out
    if isinstance(plan, Plan):
        t_pf = plan.t_pf
        dec_slots = {int(s) for s, _, _, k in plan.jobs_host[plan.n_pf_jobs:] if k != 0}
    else:  # device mixed plan: counts unknown on the host, assume half the tokens prefill
        t_pf = plan.T // 2
        dec_slots = set(range(len(table)))
    flops = 3.0 * t_pf * out * inp
    nbytes = 2.0 * out * inp + sum(table.deltas[s].nbytes for s in dec_slots)
    best, best_t = 0, float("inf")
    for s in range(8, sms - 8, 4):
        t = max(flops / (s * 6.5e12), nbytes / min((sms - s) * 45e9, 6.0e12))
        if t < best_t:
            best, best_t = s, t
    return best


def sbmm_args(X: torch.Tensor, plan: Plan, base: NativeBase | None, table: DeltaTable,
              y_dtype: torch.dtype = torch.bfloat16, act: int = L.DZ_ACT_NONE, Y: torch.Tensor | None = None,
              workspace: Workspace | None = None, grid: int = 0, debug: int = 0,
              base_splits: int = 0, tp=None, delta_splits: int = 0):
    """The dz_sbmm_args of one launch (plus Y and the tensors the args point to)."""
    T, inp = int(X.shape[0]), int(X.shape[1])
    out = table.out if base is None else base.out
    if base is not None and (base.out, base.inp) != (table.out, table.inp):
        raise ShapeError("base / delta table shape mismatch")
    if inp != table.inp:
        raise ShapeError(f"input dim {inp} != layer in {table.inp}")
    if T != plan.T:
        raise ShapeError("plan built for a different batch")
    Xp = prepare_x(X)
    if Y is None:
        Y = torch.empty(T, out, dtype=y_dtype, device=X.device)
    ws = (workspace or _default_ws).get(T, out, X.device)
    a = L.DzSbmmArgs()
    a.X, a.ldx = Xp.data_ptr(), Xp.stride(0)
    a.Y, a.ldy = Y.data_ptr(), Y.stride(0)
    a.y_dtype = L.DZ_F32 if Y.dtype == torch.float32 else L.DZ_BF16
    a.act = act
    a.T, a.out, a.in_ = T, out, inp
    a.base = base.entry.data_ptr() if base is not None else None
    a.table, a.n_slots = table.dev.data_ptr(), len(table)
    a.order = plan.order.data_ptr()
    a.jobs, a.n_jobs = plan.jobs.data_ptr(), plan.n_jobs
    a.workspace = ws.data_ptr()
    a.grid = grid
    a.debug = debug
    a.sparse_job_tokens = plan.sparse_job_tokens  # selects the kernel instantiation (X stage size)
    a.base_splits = base_splits  # 0 = by shape (batch-independent); 1..4 = explicit K-splits of the base
    a.delta_splits = delta_splits  # 0 = by shape; 1..2 = explicit K-splits of each decode delta job
    if tp is not None:  # peer.PeerGroup: row-parallel shard, reduced over peer memory by the finalize
        a.tp = C.addressof(tp.ctx)
    if isinstance(plan, DevicePlan):
        if plan.mixed:
            a.pf_counts_dev = plan.counts.data_ptr()
        else:
            a.n_jobs_dev = plan.n_jobs_dev.data_ptr()
    xs = None
    if plan.perm is not None:  # mixed plan: staged (permuted) copy of X, compact padded rows
        ldxs = _ceil(inp, BLK_COLS) * BLK_COLS
        xs = torch.empty(T, ldxs, dtype=torch.bfloat16, device=X.device)
        a.perm, a.xs, a.ldxs = plan.perm.data_ptr(), xs.data_ptr(), ldxs
        a.n_pf_jobs, a.t_pf = plan.n_pf_jobs, plan.t_pf
    return a, Y, (Xp, xs, ws)


def args_to_device(args: list, device) -> torch.Tensor:
    """Device copy of a list of dz_sbmm_args (for `next_args` chains)."""
    raw = b"".join(C.string_at(C.addressof(a), C.sizeof(a)) for a in args)
    return torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(device)


def concat_rows(parts: list[NativeDelta]) -> NativeDelta:
    """Row-concatenate resident deltas of linears that share an input (QKV, gate/up fusion).

    Exact and copy-only: native blocks are row-group-major ([16-row group][K block]), so the
    concatenation of [ΔW_q; ΔW_k; ΔW_v] is the concatenation of their block buffers, provided every
    part but the last has rows % 16 == 0 and all parts share cols and kind."""
    if not parts:
        raise ShapeError("nothing to concatenate")
    kind, cols = parts[0].kind, parts[0].cols
    for p in parts:
        if p.kind != kind or p.cols != cols or p.qmax != parts[0].qmax:
            raise ShapeError("concat_rows needs deltas of one kind and one input width")
    for p in parts[:-1]:
        if p.rows % BLK_ROWS:
            raise ShapeError("concat_rows needs rows % 16 == 0 for all but the last part")
    blocks = torch.cat([p.blocks for p in parts])
    return NativeDelta(kind, parts[0].qmax, sum(p.rows for p in parts), cols, blocks, parts[0].bits)
