#!/usr/bin/env python3
"""Benchmark: decode tokens/s of the fused base-GEMM + SBMM hot path on a Llama-2-7B-shaped
decoder stack with 32 concurrent 4-bit 2:4 deltas, decode batch 64 (BASELINE.json configs[1]).

One step = one decode step through all 32 layers x 7 linears (q,k,v,o 4096x4096; gate/up
11008x4096; down 4096x11008): 224 fused SBMM launches, each reading the bf16 base weight once and
every delta of the 32 routed deltas once (97.5 GB per step, far larger than L2 — no L2 flush
needed). Attention/norm/activation are out of scope (the reference hot path is the decoupled
linear): o consumes the q slice of the QKV output, down the up slice of the gate/up
output, the next layer down's output (paper_2312_05215_b200/stack.py). The step is captured in
one CUDA graph.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 (torchrun): Megatron tensor parallelism of the same stack (strong scaling) — q,k,v,gate,up
column-parallel, o,down row-parallel, reduced by the finalize kernel over peer memory (CUDA IPC,
NVLink; DZ_TP_FUSED=0 falls back to an NCCL all-reduce); shared dimensions cut on 128-column
native-block edges (7B intermediate 11008 = 86 blocks, uneven at TP 4/8).

--impl reference: the reference's own sbmm (`deltazip.inference.sbmm` from baseline/_ref, installed
from /root/reference/pkg; the oracle port when absent) on the host cores, one process per core over
the active deltas, plus one real cfg1 call as the anchor of the extrapolation.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MODEL = "7b"
D_DELTAS = 32
T_TOKENS = 64
BITS = 4
ID_SEED = 12


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--layers", type=int, default=32, help="decoder layers (32 = full 7B stack)")
    p.add_argument("--no-graph", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--quick", action="store_true", help="skip clocks sampler / cpu baseline (profiling runs)")
    p.add_argument("--fused-merge", action="store_true", help="Y written inside k_sbmm (no k_finalize launch)")
    p.add_argument("--chain", action="store_true", help="the whole step as ONE chained launch (dz_sbmm_chain)")
    p.add_argument("--chain-len", type=int, default=0, help="with --chain: linears per chained launch (0 = all)")
    return p.parse_args()


METRIC = "decode tokens/s (Llama-2-7B-shaped stack, 32 x 4-bit 2:4 deltas, batch 64)"
WORKLOAD = ("llama2-7b decoder stack, {layers} layers x 7 linears (q,k,v,o,gate,up,down; QKV and gate/up row-fused "
            "into one launch each), D=32 4-bit 2:4 deltas (gs=128), T=64 decode tokens, ids=perm(i%32)")


def token_ids():
    rng = np.random.default_rng(ID_SEED)
    return rng.permutation([i % D_DELTAS for i in range(T_TOKENS)]).astype(np.int32)


# ----------------------------------------------------------------------------- CPU reference arm


def _reference_pkg():
    """The reference package itself (`deltazip`, installed once from /root/reference/pkg into
    baseline/_ref, git-ignored; it travels to the GPU box with the snapshot), or None — then the
    CPU arm times the oracle port of the same algorithm instead."""
    p = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(p, "deltazip")):
        return None
    if p not in sys.path:
        sys.path.insert(0, p)
    try:
        import deltazip.compress  # noqa: F401
        import deltazip.inference  # noqa: F401
        return sys.modules["deltazip"]
    except Exception:  # pragma: no cover
        return None


def _ref_delta(dz, o):
    """A reference LayerDelta (compress.py:101-143) holding the oracle-generated packed fields."""
    return dz.compress.LayerDelta(name="bench", rows=o.rows, cols=o.cols, packed_values=o.packed_values,
                                  index_stream=o.index_stream, scales=o.scales, bits=o.bits, sparsity=o.sparsity,
                                  group_size=o.group_size)


def _delta_task(args):
    """One active delta of sbmm on one linear shape (dequantise + the routed tokens' products,
    inference.py:140-153): the reference's own `deltazip.inference.sbmm` when installed, else the
    oracle port. Runs in a worker process; times only the call."""
    out, inp, seed, tokens = args
    import oracle as O
    rng = np.random.default_rng(seed)
    W = rng.normal(0, 1 / math.sqrt(inp), (out, inp)).astype(np.float32).astype(np.float64)
    ld = O.random_packed_delta(rng, out, inp, BITS)
    X = rng.normal(0, 1, (tokens, inp))
    dz = _reference_pkg()
    if dz is not None:
        batch = dz.inference.BatchInput([(i, 0, X[i]) for i in range(tokens)])
        rd = {0: _ref_delta(dz, ld)}
        t0 = time.perf_counter()
        dz.inference.sbmm(W, rd, batch)
    else:
        t0 = time.perf_counter()
        O.sbmm_matrix(W, {0: ld}, np.zeros(tokens, np.int64), X)
    return time.perf_counter() - t0


def _worker_init():
    """One BLAS thread per worker process: the pool already puts one process on every core
    (otherwise each forked numpy would start a full OpenBLAS pool and oversubscribe the host)."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except ImportError:  # pragma: no cover
        pass


def _base_task(args):
    out, inp, seed = args
    rng = np.random.default_rng(seed)
    W = rng.normal(0, 1 / math.sqrt(inp), (out, inp))
    X = rng.normal(0, 1, (T_TOKENS, inp))
    t0 = time.perf_counter()
    _ = X @ W.T
    return time.perf_counter() - t0


def cfg1_anchor():
    """One real call of the reference's sbmm at BASELINE configs[0] (4096x4096, 4 deltas 4-bit
    2:4, 16 tokens ids perm(i%4)), single process: the measured point the extrapolated step rests on."""
    dz = _reference_pkg()
    if dz is None:
        return None
    import oracle as O
    rng = np.random.default_rng(11)
    n = 4096
    W = rng.normal(0, 1 / math.sqrt(n), (n, n)).astype(np.float32).astype(np.float64)
    lds = {d: _ref_delta(dz, O.random_packed_delta(rng, n, n, 4)) for d in range(4)}
    ids = rng.permutation(np.arange(16) % 4)
    batch = dz.inference.BatchInput([(i, int(ids[i]), rng.normal(0, 1, n)) for i in range(16)])
    t0 = time.perf_counter()
    dz.inference.sbmm(W, lds, batch)
    dt = time.perf_counter() - t0
    return {"config": "cfg1: 4096x4096, 4 x 4-bit 2:4 deltas, T=16", "seconds_per_call": dt, "tokens_per_s": 16 / dt,
            "impl": "deltazip.inference.sbmm (baseline/_ref)"}


class CpuReference:
    """The reference's sbmm on the host cores: `deltazip.inference.sbmm` itself (baseline/_ref)
    when installed, else the oracle port (numpy f64).

    The reference's cost is one dequantise + GEMV per ACTIVE delta per linear (inference.py:
    140-153, single-threaded numpy masked gathers), so the step parallelises over deltas: a pool
    of `cores` processes runs one active delta each, concurrently, per distinct 7B linear shape.
    A sample = one such round per shape (cores deltas x 2 tokens) + the 64-token base GEMM;
    the step time is extrapolated to 32 active deltas x 32 layers."""

    def __init__(self, cores: int | None = None):
        import multiprocessing as mp
        from paper_2312_05215_b200.synth import llama_linears
        self.cores = cores or min(os.cpu_count() or 1, 32)  # ~1.5 GB of numpy temporaries per worker
        self.kind = "reference" if _reference_pkg() is not None else "port"
        self.pool = mp.get_context("fork").Pool(self.cores, initializer=_worker_init)
        self.shapes = {}
        for name, out, inp in llama_linears(MODEL):
            self.shapes.setdefault((out, inp), []).append(name)
        self.round = 0

    def sample(self):
        per_shape, work = {}, 0.0
        for k, ((out, inp), names) in enumerate(self.shapes.items()):
            seeds = [(out, inp, 1000 * self.round + 31 * k + c, T_TOKENS // D_DELTAS) for c in range(self.cores)]
            # each task times only its own sbmm (inputs are generated before its clock starts);
            # the tasks run concurrently, one per core, so `cores` deltas take max(times)
            times = self.pool.map(_delta_task, seeds, chunksize=1)
            tb = _base_task((out, inp, k))
            work += max(times) + tb
            per_delta = max(times) / self.cores
            per_shape[(out, inp)] = (D_DELTAS * per_delta + tb, len(names))
        self.round += 1
        step_s = 32 * sum(t * n for t, n in per_shape.values())
        impl = ("deltazip.inference.sbmm (the reference package, baseline/_ref)" if self.kind == "reference"
                else "oracle port of inference.sbmm (numpy f64)")
        desc = (f"{impl}: per distinct 7B linear shape, {self.cores} active deltas x {T_TOKENS // D_DELTAS} tokens "
                f"on {self.cores} processes (one delta each) + the 64-token base GEMM; extrapolated to {D_DELTAS} "
                f"active deltas x 32 layers ({work:.1f} s wall per sample)")
        return T_TOKENS / step_s, work, desc

    def close(self):
        self.pool.terminate()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ref = CpuReference()
    for _ in range(min(args.warmup, 1)):
        ref.sample()  # forks warm (numpy imported, pages touched)
    vals = []
    for _ in range(max(1, args.steps)):
        v, w, desc = ref.sample()
        vals.append(v)
    ref.close()
    anchor = cfg1_anchor()
    v = float(np.median(vals))
    line = {
        "impl": "reference", "metric": METRIC,
        "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * T_TOKENS / v, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD.format(layers=32), "global_batch": T_TOKENS, "parallelism": "cpu"},
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": ref.cores, "kind": ref.kind, "sample": desc,
                         "cfg1_anchor": anchor},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_traffic():
    """Per-launch DRAM bytes (read + write) of the fused kernel from the committed ncu --set full
    capture (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as f:
        d = json.load(f)
    return float(d["mean_dram_bytes_per_launch"]), float(d["mean_algorithmic_bytes_per_launch"])


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # DZ_BENCH_SHARE_GPU=1 (testing the N>1 path on a one-GPU box): every rank on cuda:0 and the
    # collective over gloo (NCCL refuses two ranks on one device); gloo cannot be graph-captured.
    share = world > 1 and os.environ.get("DZ_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
        args.no_graph = True
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=device)

    from paper_2312_05215_b200.engine import Plan
    from paper_2312_05215_b200.stack import STEP_ORDER, LlamaStack

    t_build = time.time()
    st = LlamaStack(MODEL, args.layers, D_DELTAS, BITS, device, rank=rank, world=world)
    st.fused_merge = args.fused_merge
    fused_tp = world > 1 and os.environ.get("DZ_TP_FUSED", "1") == "1"
    if fused_tp:  # row-parallel outputs reduced over peer memory by the finalize kernel (no NCCL)
        st.enable_fused_tp(T_TOKENS)
        flag = torch.tensor([0 if st.peers is None else 1], device=device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)  # every rank must take the same path
        if int(flag.item()) == 0:
            st.peers, fused_tp = None, False
    t_build = time.time() - t_build

    ids = token_ids()
    kinds = st.kinds
    plan = Plan(ids, kinds, D_DELTAS, device=device)
    assert plan.t_pf == 0  # 2 tokens per delta: pure decode plan
    bufs = st.buffers(T_TOKENS)
    # random token activations (N(0, 1), bf16): the stack's buffers start at zero, and an all-zero
    # step draws less power and clocks ~3% higher under the power cap than real data
    # (profiles/r02_e2e_zero_inputs.txt)
    gen_x = torch.Generator(device=device)
    gen_x.manual_seed(1234 + rank)
    bufs["x"].copy_(torch.randn(T_TOKENS, bufs["x"].shape[1], generator=gen_x, device=device).to(torch.bfloat16))
    tail_pf = world == 1 and os.environ.get("DZ_TAIL_PREFETCH", "1") != "0"
    if tail_pf:  # each launch warms L2 with the next launch's first weight stages at its tail
        st.prepare_chain(plan, bufs)
    stream = torch.cuda.current_stream()
    chained = args.chain and world == 1
    st.chain_len = args.chain_len
    step_fn = (lambda p_: st.step_chained(p_, bufs)) if chained else (lambda p_: st.step(p_, bufs))

    step_fn(plan)  # eager warm-up (sets kernel attributes, NCCL communicators)
    torch.cuda.synchronize()
    graph = None
    if not args.no_graph:
        s_ = torch.cuda.Stream()
        s_.wait_stream(stream)
        with torch.cuda.stream(s_):
            step_fn(plan)
        stream.wait_stream(s_)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step_fn(plan)
        torch.cuda.synchronize()

    def run_step():
        if graph is not None:
            graph.replay()
        else:
            step_fn(plan)

    for _ in range(args.warmup):
        run_step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local) if not args.quick else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
        time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall0 = time.time()
    e0.record(stream)
    for _ in range(args.steps):
        run_step()
    e1.record(stream)
    torch.cuda.synchronize()
    wall = time.time() - wall0
    if world > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["not sampled"]}
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---- per-launch kernel durations: eager step with events around every fused launch (the
    # events bracket the kernel(s) of one linear on the launching stream; TP adds the all-reduce
    # of o/down, which is excluded by bracketing sbmm_forward only)
    lin_bytes = st.launch_bytes(T_TOKENS, D_DELTAS)
    evs, order = [], []
    h = bufs["x"]
    torch.cuda.synchronize()
    from paper_2312_05215_b200.engine import sbmm_forward
    for lin in st.stack:
        src = {"h": h, "v": bufs["v"], "up": bufs["up"]}
        for f, s_ in STEP_ORDER:
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            sbmm_forward(src[s_], plan, lin[f].base, lin[f].table, Y=bufs[f], workspace=st.ws)
            b_.record(stream)
            evs.append((a_, b_))
            order.append(f)
        h = bufs["down"]
    torch.cuda.synchronize()
    durs = np.array([a_.elapsed_time(b_) for a_, b_ in evs])  # ms
    per_name = {}
    for n, d in zip(order, durs):
        per_name.setdefault(n, []).append(d)
    kern_bytes = sum(lin_bytes[n] for n in order)
    kern_ms = float(durs.sum())
    achieved = kern_bytes / (kern_ms * 1e-3) / 1e9
    peak, peak_kind = measured_peaks()
    step_bytes = args.layers * sum(lin_bytes.values())
    tokens_per_s = T_TOKENS / (ms * 1e-3)  # TP: the step serves T tokens across all ranks
    traffic, traffic_alg = ncu_traffic() if world == 1 and args.layers == 32 else (None, None)

    # ---- e2e through the public API: pinned host X -> host plan (group_by_delta, dz_plan) ->
    # H2D of X + plan -> step -> D2H of the step's output, all inside the timed region.
    e2e = None
    if not args.no_e2e:
        # Two pinned input/output sets used alternately, each with its own captured graph of
        # [H2D slots + X, on-device plan (dz_plan_device), the step, D2H Y], so the host can write
        # step k+1's tokens and delta ids while step k runs without racing the in-flight copies.
        from paper_2312_05215_b200.engine import DevicePlan
        hid = bufs["x"].shape[1]
        # decode batches of a few tokens per delta: 8-token 2:4 jobs (the narrow kernel instantiation;
        # a token's result does not depend on the job width)
        dplan = DevicePlan(T_TOKENS, kinds, D_DELTAS, device=device, sparse_job_tokens=8)
        slots_dev = torch.zeros(T_TOKENS, dtype=torch.int32, device=device)
        if tail_pf:
            st.prepare_chain(dplan, bufs)
        sets = []
        for _ in range(2):
            io = {"x": torch.randn(T_TOKENS, hid).to(torch.bfloat16).pin_memory(),
                  "y": torch.empty(T_TOKENS, hid, dtype=torch.bfloat16).pin_memory(),
                  "slots": torch.zeros(T_TOKENS, dtype=torch.int32).pin_memory(),
                  "done": torch.cuda.Event()}
            sets.append(io)

        def e2e_body(io):
            slots_dev.copy_(io["slots"], non_blocking=True)
            bufs["x"].copy_(io["x"], non_blocking=True)
            dplan.update(slots_dev)  # group_by_delta on the device
            st.step(dplan, bufs)
            io["y"].copy_(bufs["down"], non_blocking=True)

        def host_plan(io):
            io["slots"].copy_(torch.from_numpy(ids))  # this step's token -> delta map

        graphs = []
        if graph is not None:
            for io in sets:
                host_plan(io)
                g2 = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g2):
                    e2e_body(io)
                graphs.append(g2)
        torch.cuda.synchronize()

        def e2e_step(k):
            io = sets[k % 2]
            io["done"].synchronize()  # this set's previous copies finished: safe to overwrite
            host_plan(io)
            if graphs:
                graphs[k % 2].replay()
            else:
                e2e_body(io)
            io["done"].record(stream)

        for k in range(2):  # warm: first-call host overheads outside the timed region
            e2e_step(k)
        torch.cuda.synchronize()
        # the same starting point as the `value` block: the GPU idles briefly after the warm-up steps
        # (a block that starts right after another runs a few percent lower under the power cap)
        time.sleep(float(os.environ.get("DZ_BENCH_E2E_GAP", "1.0")))
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for k in range(args.steps):
            e2e_step(k)
        f1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = f0.elapsed_time(f1) / args.steps
        if world > 1:
            t = torch.tensor([e2e_ms], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        dplan.check()
        io = sets[0]
        h2d = io["x"].numel() * 2 + io["slots"].numel() * 4
        d2h = io["y"].numel() * 2
        e2e = {"value": T_TOKENS / (e2e_ms * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms,
               "path": "pinned H2D (delta ids, X) + on-device group_by_delta (dz_plan_device) + step + D2H (Y), "
                       "one CUDA graph per step"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.quick:
        ref = CpuReference()
        v, wsec, desc = ref.sample()
        ref.close()
        cpu = {"value": v, "unit": "tokens/s", "cores": ref.cores, "kind": ref.kind, "sample": desc,
               "cfg1_anchor": cfg1_anchor()}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": tokens_per_s, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random bf16 base, random reference-layout 4-bit 2:4 deltas uploaded via dz_repack_sparse, "
                    "random N(0,1) bf16 token activations)",
            "config": {"workload": WORKLOAD.format(layers=args.layers),
                       "global_batch": T_TOKENS,
                       "parallelism": (f"tp{world}" + ("+peer-memory reduce" if fused_tp else "+nccl all-reduce"))
                       if world > 1 else "single",
                       "l2": "inputs > L2 (97.5 GB streamed per step at N=1)", "cuda_graph": graph is not None,
                       "step_bytes_rank0": step_bytes,
                       "output_rms": float(bufs["down"].float().pow(2).mean().sqrt()),
                       "output_finite": bool(torch.isfinite(bufs["down"]).all())},
            "gpu_launches": (1 if args.fused_merge else 2) * len(order) * args.steps,  # k_sbmm (+ k_finalize) per fused linear
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "traffic_algorithmic": traffic_alg, "peak_kind": peak_kind,
                         "kernel": "k_sbmm (fused base GEMM + SBMM), all 4 x layers launches of one step (QKV, o, "
                                   "gate/up, down); achieved = algorithmic bytes / summed launch time; traffic = "
                                   "mean DRAM bytes per launch (k_sbmm + k_finalize) from ncu --set full (profiles/r02_ncu_full.md)",
                         "per_launch_us": {n: float(np.mean(v) * 1e3) for n, v in per_name.items()},
                         "step_GBps": step_bytes / (ms * 1e-3) / 1e9},
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "build_s": round(t_build, 1),
            "wall_s_timed": round(wall, 3),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
