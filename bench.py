#!/usr/bin/env python3
"""Benchmark: decode tokens/s of the fused base-GEMM + SBMM hot path on a Llama-2-7B-shaped
decoder stack with 32 concurrent 4-bit 2:4 deltas, decode batch 64 (BASELINE.json configs[1]).

One step = one decode step through all 32 layers x 7 linears (q,k,v,o 4096x4096; gate/up
11008x4096; down 4096x11008): 224 fused SBMM launches, each reading the bf16 base weight once and
every delta of the 32 routed deltas once (97.5 GB per step, far larger than L2 — no L2 flush
needed). Attention/norm/activation are out of scope (the reference hot path is the decoupled
linear): o consumes v's output, down consumes up's output, the next layer consumes
down's output. The step is captured in one CUDA graph.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 (torchrun): Megatron tensor parallelism of the same stack — q,k,v,gate,up column-parallel,
o,down row-parallel + NCCL all-reduce; intermediate (11008) sharded in 128-column blocks.
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
    return p.parse_args()


def token_ids():
    rng = np.random.default_rng(ID_SEED)
    return rng.permutation([i % D_DELTAS for i in range(T_TOKENS)]).astype(np.int32)


# ----------------------------------------------------------------------------- CPU reference arm


def cpu_reference_sample(model: str = MODEL, deltas_per_shape: int = 1, tokens: int = 4):
    """Time the oracle port (numpy f64, the reference's algorithm) on a bounded sample of the
    same workload: per distinct linear shape, sbmm over `deltas_per_shape` deltas and `tokens`
    tokens; extrapolate linearly in active deltas (cost per active delta is the dequantise,
    inference.py:145-153) to the full step. Returns (tokens_per_s, seconds_of_work, desc)."""
    import oracle as O
    from paper_2312_05215_b200.synth import llama_linears

    rng = np.random.default_rng(0)
    t_work = 0.0
    per_shape = {}
    shapes = {}
    for name, out, inp in llama_linears(model):
        shapes.setdefault((out, inp), []).append(name)
    for (out, inp), names in shapes.items():
        W = rng.normal(0, 1 / math.sqrt(inp), (out, inp)).astype(np.float32).astype(np.float64)
        ds = {d: O.random_packed_delta(rng, out, inp, BITS) for d in range(deltas_per_shape)}
        X = rng.normal(0, 1, (tokens, inp))
        ids = np.arange(tokens) % deltas_per_shape
        t0 = time.perf_counter()
        O.sbmm_matrix(W, ds, ids, X)
        dt = time.perf_counter() - t0
        t_work += dt
        # base GEMM for the full batch (64 tokens) measured too
        X64 = rng.normal(0, 1, (T_TOKENS, inp))
        t1 = time.perf_counter()
        _ = X64 @ W.T
        tb = time.perf_counter() - t1
        t_work += tb
        per_delta = dt / deltas_per_shape
        per_shape[(out, inp)] = (D_DELTAS * per_delta + tb, len(names))
    layers = 32
    step_s = layers * sum(t * n for t, n in per_shape.values())
    desc = (f"oracle sbmm (numpy f64) per distinct 7B linear shape with {deltas_per_shape} delta(s) x "
            f"{tokens} tokens + 64-token base GEMM, extrapolated x{D_DELTAS} active deltas x{layers} layers")
    return T_TOKENS / step_s, t_work, desc


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count()
    for _ in range(args.warmup):
        pass  # the sample has no warm state worth warming beyond numpy import
    vals, work = [], 0.0
    for _ in range(max(1, args.steps)):
        v, w, desc = cpu_reference_sample()
        vals.append(v)
        work += w
    v = float(np.median(vals))
    line = {
        "impl": "reference", "metric": "decode tokens/s (Llama-2-7B-shaped stack, 32 x 4-bit 2:4 deltas, batch 64)",
        "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * T_TOKENS / v, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "llama2-7b decoder stack, 32 layers x 7 linears, D=32 4-bit 2:4 deltas, T=64 decode",
                   "parallelism": "cpu"},
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "port", "sample": desc},
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


FUSED = {"qkv": ("q", "k", "v"), "o": ("o",), "gate_up": ("gate", "up"), "down": ("down",)}


def build_stack(layers, rank, world, device):
    """Per layer 4 fused linears (QKV and gate/up row-concatenated: they read the same input),
    each = (base W, delta table of 32 natives). Deltas are generated per original linear and
    concatenated, so bytes and math are exactly those of the 7 separate linears."""
    import torch
    from paper_2312_05215_b200.device import ErrFlag
    from paper_2312_05215_b200.engine import DeltaTable, NativeBase, concat_rows
    from paper_2312_05215_b200.synth import llama_linears, random_base, random_native_delta
    from paper_2312_05215_b200.tp import TpLinear

    gen = torch.Generator(device=device)
    err = ErrFlag(device)
    shapes = {n: (o, i) for n, o, i in llama_linears(MODEL)}
    names = [n for n, _, _ in llama_linears(MODEL)]
    stack = []
    for l in range(layers):
        lin = {}
        for fname, members in FUSED.items():
            Ws, per_delta = [], [[] for _ in range(D_DELTAS)]
            for m in members:
                out, inp = shapes[m]
                gen.manual_seed(10_000 + 7 * l + names.index(m))
                Ws.append(random_base(out, inp, gen, device))
                for d in range(D_DELTAS):
                    per_delta[d].append(random_native_delta(out, inp, BITS, gen, device, err))
            W = torch.cat(Ws) if len(Ws) > 1 else Ws[0]
            nats = [concat_rows(p) if len(p) > 1 else p[0] for p in per_delta]
            out, inp = int(W.shape[0]), int(W.shape[1])
            if world == 1:
                lin[fname] = (NativeBase(W), DeltaTable(nats, out, inp), out, inp)
            else:
                axis = "row" if fname in ("o", "down") else "column"
                lin[fname] = TpLinear(W, nats, axis, rank, world)
            del W, Ws, per_delta
        stack.append(lin)
        torch.cuda.synchronize()
    err.raise_if_set("synthetic delta upload")
    return stack


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
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)

    from paper_2312_05215_b200 import _lib as L
    from paper_2312_05215_b200.engine import Plan, Workspace, sbmm_forward
    from paper_2312_05215_b200.synth import linear_algorithmic_bytes, llama_linears

    t_build = time.time()
    stack = build_stack(args.layers, rank, world, device)
    t_build = time.time() - t_build

    ids = token_ids()
    kinds = np.full(D_DELTAS, L.DZ_KIND_SPARSE4, dtype=np.int32)
    plan = Plan(ids, kinds, D_DELTAS, device=device)
    ws = Workspace()
    shapes = dict((n, (o, i)) for n, o, i in llama_linears(MODEL))
    hid, inter = shapes["q"][1], shapes["gate"][0]

    # activation buffers (static addresses for graph capture). Attention is out of scope: o reads
    # the v slice of the fused QKV output, down reads the up slice of the fused gate/up output.
    def buf(cols):
        return torch.zeros(T_TOKENS, cols, dtype=torch.bfloat16, device=device)

    fshape = {f: (sum(shapes[m][0] for m in ms), shapes[ms[0]][1]) for f, ms in FUSED.items()}
    x_in = buf(hid)
    if world == 1:
        outs = {f: buf(fshape[f][0]) for f in FUSED}
        v_in = outs["qkv"][:, shapes["q"][0] + shapes["k"][0]:]
        up_in = outs["gate_up"][:, shapes["gate"][0]:]
    else:
        outs = {f: buf(stack[0][f].table.out if f in ("qkv", "gate_up") else hid) for f in FUSED}
        v_in = outs["qkv"][:, 2 * outs["qkv"].shape[1] // 3:]
        up_in = outs["gate_up"][:, outs["gate_up"].shape[1] // 2:]

    def linear(lin, name, X, Y):
        if world == 1:
            base, table, _, _ = lin
            sbmm_forward(X, plan, base, table, Y=Y, workspace=ws)
        else:
            Yl = lin.forward(X, plan)
            Y.copy_(Yl) if Yl.data_ptr() != Y.data_ptr() else None

    step_order = [("qkv", "h"), ("o", "v"), ("gate_up", "h"), ("down", "up")]

    def step():
        h = x_in
        for lin in stack:
            src = {"h": h, "v": v_in, "up": up_in}
            for f, s_ in step_order:
                linear(lin[f], f, src[s_], outs[f])
                src = {"h": h, "v": v_in, "up": up_in}
            h = outs["down"]
        return h

    stream = torch.cuda.current_stream()
    # eager warm-up (sets kernel attributes, checks the path), then capture
    step()
    torch.cuda.synchronize()
    graph = None
    if not args.no_graph:
        s = torch.cuda.Stream()
        s.wait_stream(stream)
        with torch.cuda.stream(s):
            step()
        stream.wait_stream(s)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        torch.cuda.synchronize()

    def run_step():
        if graph is not None:
            graph.replay()
        else:
            step()

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

    # ---- per-launch kernel durations (eager, events between consecutive launches on the stream)
    lin_bytes = {n: linear_algorithmic_bytes(o, i, BITS, D_DELTAS, T_TOKENS) for n, (o, i) in shapes.items()}
    f_bytes = {f: sum(lin_bytes[m] for m in ms) - (len(ms) - 1) * (2 * T_TOKENS * fshape[f][1] + 4 * T_TOKENS)
               for f, ms in FUSED.items()}  # the shared input x is read once per fused launch
    if world > 1:
        f_bytes = {n: b // world for n, b in f_bytes.items()}
    evs = []
    torch.cuda.synchronize()
    h = x_in
    order = []
    for lin in stack:
        src = {"h": h, "v": v_in, "up": up_in}
        for f, s_ in step_order:
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            linear(lin[f], f, src[s_], outs[f])
            b_.record(stream)
            evs.append((a_, b_))
            order.append(f)
        h = outs["down"]
    torch.cuda.synchronize()
    durs = np.array([a_.elapsed_time(b_) for a_, b_ in evs])  # ms
    per_name = {}
    for n, d in zip(order, durs):
        per_name.setdefault(n, []).append(d)
    lin_bytes = f_bytes
    kern_bytes = sum(lin_bytes[n] for n in order)
    kern_ms = float(durs.sum())
    achieved = kern_bytes / (kern_ms * 1e-3) / 1e9
    peak, peak_kind = measured_peaks()
    step_bytes = args.layers * sum(lin_bytes.values())
    tokens_per_s = T_TOKENS / (ms * 1e-3)  # TP: the step serves T tokens across all ranks

    # ---- e2e through the public API: host X (pinned) -> plan on host -> H2D -> step -> D2H
    e2e = None
    if not args.no_e2e:
        # e2e through the public API: pinned host X -> host plan (group_by_delta, dz_plan) ->
        # H2D of X + plan -> step -> D2H of the step's output, all inside the timed region.
        xh = torch.randn(T_TOKENS, hid).to(torch.bfloat16).pin_memory()
        yh = torch.empty(T_TOKENS, hid, dtype=torch.bfloat16).pin_memory()
        order_pin = torch.empty(plan.order.numel(), dtype=torch.int32).pin_memory()
        jobs_pin = torch.empty(plan.jobs.numel(), dtype=torch.uint8).pin_memory()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            hp = Plan(ids, kinds, D_DELTAS, upload=False)
            order_pin[: hp.T].copy_(torch.from_numpy(hp.order_host))
            jobs_pin[: hp.jobs_bytes.size].copy_(torch.from_numpy(hp.jobs_bytes))
            x_in.copy_(xh, non_blocking=True)
            plan.order.copy_(order_pin, non_blocking=True)
            plan.jobs.copy_(jobs_pin, non_blocking=True)
            run_step()
            yh.copy_(outs["down"], non_blocking=True)
        f1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = f0.elapsed_time(f1) / args.steps
        if world > 1:
            t = torch.tensor([e2e_ms], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        h2d = xh.numel() * 2 + order_pin.numel() * 4 + jobs_pin.numel()
        d2h = yh.numel() * 2
        e2e = {"value": T_TOKENS / (e2e_ms * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.quick:
        v, wsec, desc = cpu_reference_sample()
        cpu = {"value": v, "unit": "tokens/s", "cores": 1, "kind": "port",
               "sample": desc + f" ({wsec:.1f} s of CPU work; numpy dequant is single-threaded)"}

    if rank == 0:
        line = {
            "metric": "decode tokens/s (Llama-2-7B-shaped stack, 32 x 4-bit 2:4 deltas, batch 64)",
            "value": tokens_per_s, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random bf16 base, random reference-layout 4-bit 2:4 deltas uploaded via dz_repack_sparse)",
            "config": {"workload": f"llama2-7b decoder stack, {args.layers} layers x 7 linears (q,k,v,o,gate,up,down; "
                                   f"QKV and gate/up row-fused into one launch each), "
                                   f"D={D_DELTAS} 4-bit 2:4 deltas (gs=128), T={T_TOKENS} decode tokens, ids=perm(i%32)",
                       "global_batch": T_TOKENS, "parallelism": f"tp{world}" if world > 1 else "single",
                       "l2": "inputs > L2 (97.5 GB streamed per step)", "cuda_graph": graph is not None,
                       "step_bytes": step_bytes},
            "gpu_launches": len(order) * args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": None, "peak_kind": peak_kind,
                         "kernel": "k_sbmm (fused base GEMM + SBMM), all 4 x layers launches of one step (QKV, o, gate/up, down)",
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
