"""Llama decoder-stack driver over the fused SBMM kernels (the forward_model
equivalent for Llama-shaped layers, inference.py:246-291 / PAPER.md §5.3).

Per decoder layer the seven linears run as four launches: QKV and gate/up are row-fused (they
read the same input; the concatenation of native blocks is exact, `engine.concat_rows`), o and
down run alone. Attention, norms and the SwiGLU product are outside the reference hot path
(SPEC.md:324): o consumes the q slice of the QKV output (the attention output has its width)
and down the up slice of the gate/up output, so every byte of every linear is streamed exactly
as in a real decode step.

Tensor parallelism (Megatron, the delta partitioned exactly like its base):
q, k, v, gate, up are column-parallel (this rank's output rows, no collective); o and down are
row-parallel (this rank's input columns) followed by an NCCL all-reduce of the bf16 output. The
shared dimensions are cut on native-block edges — 128 columns for the row-parallel input,
which fixes the matching 16-row-aligned column-parallel output — so every shard of a resident
delta is a sub-grid of its native blocks (`tp.shard_native`), unevenly where the dimension is
not divisible (7B intermediate 11008 = 86 x 128 at TP 4: 22,22,21,21 blocks).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .device import ErrFlag, nvtx_pop, nvtx_push
from .engine import DeltaTable, NativeBase, NativeDelta, Plan, Workspace, concat_rows, sbmm_forward
from .synth import delta_algorithmic_bytes, llama_linears, random_base, random_native_delta

FUSED = {"qkv": ("q", "k", "v"), "o": ("o",), "gate_up": ("gate", "up"), "down": ("down",)}
C_SIZEOF_ARGS = __import__("ctypes").sizeof(L.DzSbmmArgs)
STEP_ORDER = (("qkv", "h"), ("o", "v"), ("gate_up", "h"), ("down", "up"))
ROW_PARALLEL = ("o", "down")


def split_units(n: int, world: int, unit: int) -> list[tuple[int, int]]:
    """Contiguous [start, end) parts of range(n), each a whole number of `unit`s (the last part
    may end at n), as even as possible."""
    nb = -(-n // unit)
    if nb < world:
        raise ValueError(f"{n} cannot be split into {world} parts of {unit}")
    q, r = divmod(nb, world)
    bounds, s = [], 0
    for i in range(world):
        e = min(n, s + (q + (1 if i < r else 0)) * unit)
        bounds.append((s, e))
        s = e
    return bounds


def tp_bounds(model: str, rank: int, world: int) -> tuple[tuple[int, int], tuple[int, int], tuple[int, int]]:
    """This rank's [start, end) of the hidden, kv and intermediate dimensions: the row-parallel
    inputs (o: hidden, down: intermediate) are cut on 128-column native-block edges and the
    column-parallel outputs (q: hidden, k/v: kv, gate/up: intermediate) use the same cuts."""
    shapes = {n: (o, i) for n, o, i in llama_linears(model)}
    hid, inter, kv = shapes["q"][1], shapes["gate"][0], shapes["k"][0]
    return (split_units(hid, world, 128)[rank], split_units(kv, world, 128)[rank],
            split_units(inter, world, 128)[rank])


def shard_sub(nat: NativeDelta, r0: int, r1: int, c0: int, c1: int) -> NativeDelta:
    """Sub-grid of a resident native delta (rows on 16-row, columns on 128-column block edges)."""
    from .engine import BLK_COLS, BLK_ROWS
    if r0 == 0 and c0 == 0 and r1 == nat.rows and c1 == nat.cols:
        return nat
    assert r0 % BLK_ROWS == 0 and c0 % BLK_COLS == 0
    assert (r1 % BLK_ROWS == 0 or r1 == nat.rows) and (c1 % BLK_COLS == 0 or c1 == nat.cols)
    n16, nkb = -(-nat.rows // BLK_ROWS), -(-nat.cols // BLK_COLS)
    grid = nat.blocks.view(n16, nkb, -1)
    sub = grid[r0 // BLK_ROWS: -(-r1 // BLK_ROWS), c0 // BLK_COLS: -(-c1 // BLK_COLS)].contiguous()
    return NativeDelta(nat.kind, nat.qmax, r1 - r0, c1 - c0, sub.view(-1), nat.bits)


class FusedLinear:
    """This rank's shard of one (possibly row-fused) linear: base entry + delta table."""

    def __init__(self, name: str, W: torch.Tensor, natives: list[NativeDelta], row_parallel: bool):
        self.name, self.row_parallel = name, row_parallel
        self.out, self.inp = int(W.shape[0]), int(W.shape[1])
        self.base = NativeBase(W)
        self.table = DeltaTable(natives, self.out, self.inp)


class LlamaStack:
    """Synthetic Llama-shaped decoder stack with `n_deltas` resident deltas per linear.

    Weights and deltas are generated per ORIGINAL linear from fixed seeds (identical on every
    rank, so the shards of all ranks partition one model), then sharded and row-fused."""

    def __init__(self, model: str, layers: int, n_deltas: int, bits: int, device, rank: int = 0, world: int = 1,
                 seed: int = 10_000, group=None, keep_refs: bool = False):
        """keep_refs: also keep every ORIGINAL (unsharded, unfused) linear's bf16 base weight in
        `base_full[(layer, name)]` and its deltas' reference-layout bytes in `refs[(layer, name, d)]`
        (the parity tests rebuild each linear's reference output from them)."""
        self.model, self.layers, self.n_deltas, self.bits = model, layers, n_deltas, bits
        self.rank, self.world, self.group, self.device = rank, world, group, device
        shapes = {n: (o, i) for n, o, i in llama_linears(model)}
        self.shapes = shapes
        self.h_b, self.kv_b, self.i_b = tp_bounds(model, rank, world)
        out_rows = {"q": self.h_b, "k": self.kv_b, "v": self.kv_b, "gate": self.i_b, "up": self.i_b}
        in_cols = {"o": self.h_b, "down": self.i_b}
        names = [n for n, _, _ in llama_linears(model)]
        gen = torch.Generator(device=device)
        err = ErrFlag(device)
        self.stack: list[dict[str, FusedLinear]] = []
        self.base_full: dict = {}
        self.refs: dict = {}
        for l in range(layers):
            lin = {}
            for fname, members in FUSED.items():
                Ws, per_delta = [], [[] for _ in range(n_deltas)]
                for m in members:
                    out, inp = shapes[m]
                    r0, r1 = out_rows.get(m, (0, out))
                    c0, c1 = in_cols.get(m, (0, inp))
                    gen.manual_seed(seed + 7 * l + names.index(m))
                    Wf = random_base(out, inp, gen, device)
                    Ws.append(Wf[r0:r1, c0:c1].contiguous())
                    if keep_refs:
                        self.base_full[(l, m)] = Wf
                    del Wf
                    for d in range(n_deltas):
                        kr = [] if keep_refs else None
                        nat = random_native_delta(out, inp, bits, gen, device, err, keep_ref=kr)
                        if keep_refs:
                            self.refs[(l, m, d)] = kr[0]
                        per_delta[d].append(shard_sub(nat, r0, r1, c0, c1))
                W = torch.cat(Ws) if len(Ws) > 1 else Ws[0]
                nats = [concat_rows(p) if len(p) > 1 else p[0] for p in per_delta]
                lin[fname] = FusedLinear(fname, W, nats, fname in ROW_PARALLEL)
                del W, Ws, per_delta
            self.stack.append(lin)
            torch.cuda.synchronize(device)
        err.raise_if_set("synthetic delta upload")
        self.ws = Workspace()

    # ------------------------------------------------------------------ activations / one step
    def buffers(self, T: int) -> dict[str, torch.Tensor]:
        l0 = self.stack[0]
        mk = lambda c: torch.zeros(T, c, dtype=torch.bfloat16, device=self.device)  # noqa: E731
        hid = self.shapes["q"][1]
        b = {"x": mk(hid), "qkv": mk(l0["qkv"].out), "o": mk(hid), "gate_up": mk(l0["gate_up"].out), "down": mk(hid)}
        hq = self.h_b[1] - self.h_b[0]
        b["v"] = b["qkv"][:, :hq]  # stand-in for the attention output: the q slice has its width
        b["up"] = b["gate_up"][:, l0["gate_up"].out // 2:]
        assert b["v"].shape[1] == l0["o"].inp and b["up"].shape[1] == l0["down"].inp
        return b

    def enable_fused_tp(self, max_tokens: int) -> None:
        """Row-parallel outputs reduced by the finalize kernel over peer memory (dz_tp.cu) instead
        of an NCCL all-reduce: every rank reads the peers' fp32 partial sums in rank order."""
        import sys

        from .errors import CudaError
        from .peer import PeerGroup
        out = max(lin[f].out for lin in self.stack[:1] for f in ROW_PARALLEL)
        try:
            self.peers = PeerGroup(self.rank, self.world, max_tokens * out, self.device, self.group)
        except CudaError as e:  # e.g. no CUDA IPC between the ranks' devices: keep the NCCL all-reduce
            self.peers = None
            print(f"[dz] fused TP reduction unavailable ({e}); using the NCCL all-reduce", file=sys.stderr)

    def linear(self, lin: FusedLinear, plan: Plan, X: torch.Tensor, Y: torch.Tensor, next_args: int = 0) -> None:
        fused = lin.row_parallel and self.world > 1 and getattr(self, "peers", None) is not None \
            and plan.perm is None
        sbmm_forward(X, plan, lin.base, lin.table, Y=Y, workspace=self.ws, tp=self.peers if fused else None,
                     base_splits=getattr(self, "base_splits", 0), next_args=next_args,
                     overlap_sms=getattr(self, "overlap_sms", None),
                     fused_merge=getattr(self, "fused_merge", False),
                     prefill_variant=getattr(self, "prefill_variant", 0))
        if lin.row_parallel and self.world > 1 and not fused:
            import torch.distributed as dist
            dist.all_reduce(Y, op=dist.ReduceOp.SUM, group=self.group)

    def prepare_chain(self, plan: Plan, bufs: dict[str, torch.Tensor]) -> None:
        """Device copies of every launch's args in step order, so each launch can point its tail
        prefetch at the next one (`sbmm_forward(next_args=...)`). Single GPU, decode plans."""
        from .engine import args_to_device, sbmm_args
        args, h = [], bufs["x"]
        for lin in self.stack:
            src = {"h": h, "v": bufs["v"], "up": bufs["up"]}
            for f, s_ in STEP_ORDER:
                a, _, _ = sbmm_args(src[s_], plan, lin[f].base, lin[f].table, Y=bufs[f], workspace=self.ws,
                                    base_splits=getattr(self, "base_splits", 0))
                args.append(a)
            h = bufs["down"]
        if not hasattr(self, "chains"):
            self.chains = {}
        self.chains[(id(plan), bufs["x"].data_ptr())] = (plan, args_to_device(args, self.device))

    def prepare_step_kernel(self, plan: Plan, bufs: dict[str, torch.Tensor]) -> None:
        """Encode the whole decode step (every layer's four launches) for ONE chained launch
        (`dz_sbmm_chain`): no launch boundaries between linears, Y merged in-kernel. Single GPU,
        decode plans; the device descriptors stay valid while `bufs`, `plan` and the stack live."""
        import ctypes as C
        from .engine import sbmm_args
        # one workspace for the whole chain, sized for the widest linear before any args point to it
        self.ws.get(plan.T, max(lin[f].out for lin in self.stack for f in FUSED), self.device)
        args, h = [], bufs["x"]
        for lin in self.stack:
            src = {"h": h, "v": bufs["v"], "up": bufs["up"]}
            for f, s_ in STEP_ORDER:
                a, _, _ = sbmm_args(src[s_], plan, lin[f].base, lin[f].table, Y=bufs[f], workspace=self.ws,
                                    base_splits=getattr(self, "base_splits", 0))
                args.append(a)
            h = bufs["down"]
        lib = L.lib()
        n = len(args)
        arr = (L.DzSbmmArgs * n)(*args)
        nbytes = int(lib.dz_sbmm_chain_desc_bytes(n))
        host = torch.empty(nbytes + 64, dtype=torch.uint8)
        off = (-host.data_ptr()) % 64
        narrow = C.c_int32(0)
        L.check(lib.dz_sbmm_chain_encode(arr, n, host.data_ptr() + off, nbytes, C.byref(narrow)), "chain encode")
        dev = torch.empty(nbytes + 64, dtype=torch.uint8, device=self.device)
        doff = (-dev.data_ptr()) % 64
        dev[doff:doff + nbytes].copy_(host[off:off + nbytes])
        self.step_kernel = (plan, bufs["x"].data_ptr(), dev, doff, n, int(narrow.value))

    def step_chained(self, plan: Plan, bufs: dict[str, torch.Tensor]) -> torch.Tensor:
        """One decode step as ONE chained launch (see prepare_step_kernel)."""
        from .device import stream_ptr
        pk = getattr(self, "step_kernel", None)
        if pk is None or pk[0] is not plan or pk[1] != bufs["x"].data_ptr():
            self.prepare_step_kernel(plan, bufs)
            pk = self.step_kernel
        _, _, dev, doff, n, narrow = pk
        per = getattr(self, "chain_len", 0) or n  # linears per launch (A/B: 1 = the chain kernel per linear)
        esz = int(L.lib().dz_sbmm_chain_desc_bytes(1))
        for l0 in range(0, n, per):
            L.check(L.lib().dz_sbmm_chain(dev.data_ptr() + doff + l0 * esz, min(per, n - l0), narrow, 0,
                                          stream_ptr()), "chain")
        return bufs["down"]

    def step(self, plan: Plan, bufs: dict[str, torch.Tensor], record=None) -> torch.Tensor:
        """One decode step through every layer; returns the last layer's output buffer."""
        chain = getattr(self, "chains", {}).get((id(plan), bufs["x"].data_ptr()))
        use_chain = chain is not None and chain[0] is plan and self.world == 1
        n_lin = len(self.stack) * len(STEP_ORDER)
        h, k = bufs["x"], 0
        for li, lin in enumerate(self.stack):
            nvtx_push(f"layer {li}")
            src = {"h": h, "v": bufs["v"], "up": bufs["up"]}
            for f, s_ in STEP_ORDER:
                if record is not None:
                    record(f, "begin")
                nxt = chain[1].data_ptr() + (k + 1) * C_SIZEOF_ARGS if use_chain and k + 1 < n_lin else 0
                self.linear(lin[f], plan, src[s_], bufs[f], next_args=nxt)
                if record is not None:
                    record(f, "end")
                k += 1
            h = bufs["down"]
            nvtx_pop()
        return h

    # ------------------------------------------------------------------ bytes
    def launch_bytes(self, T: int, n_distinct: int) -> dict[str, int]:
        """Algorithmic HBM bytes of one launch of each fused linear on this rank: base + every
        distinct routed delta (per original linear) + X read once + Y written once + slot ids."""
        l0 = self.stack[0]
        out = {}
        for fname, members in FUSED.items():
            lin = l0[fname]
            if fname in ROW_PARALLEL:
                parts = [(lin.out, lin.inp)]
            else:
                rows = {"q": self.h_b, "k": self.kv_b, "v": self.kv_b, "gate": self.i_b, "up": self.i_b}
                parts = [(rows[m][1] - rows[m][0], lin.inp) for m in members]
            b = sum(2 * o * i + n_distinct * delta_algorithmic_bytes(o, i, self.bits) for o, i in parts)
            out[fname] = b + 2 * T * lin.inp + 2 * T * lin.out + 4 * T
        return out

    @property
    def kinds(self) -> np.ndarray:
        return np.array([L.DZ_KIND_SPARSE2 if self.bits == 2 else L.DZ_KIND_SPARSE3 if self.bits == 3
                         else L.DZ_KIND_SPARSE4] * self.n_deltas, dtype=np.int32)
