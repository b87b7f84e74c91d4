#!/usr/bin/env python3
"""Kernel bench of the prefill path (K3) at BASELINE cfg3 shapes (Llama-2-13B linears, 2-bit 2:4
deltas): 8 requests x 256 prefill tokens on 8 distinct deltas (+ optional decode tokens).

Prints per shape: time per launch (CUDA events, L2 flushed between launches), algorithmic
TFLOP/s (base 2·T·out·in + kept delta MACs 2·T_d·out·in/2), the executed tensor
TFLOP/s (the delta tile is dequantised to dense bf16: 2·T·out·in per product) and the fraction
of the measured bf16 peak (MEASURED_PEAKS.json)."""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2312_05215_b200.device import ErrFlag  # noqa: E402
from paper_2312_05215_b200.engine import DeltaTable, NativeBase, Plan, sbmm_forward  # noqa: E402
from paper_2312_05215_b200.synth import random_base, random_native_delta  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--bits", type=int, default=2)
p.add_argument("--prefill", type=int, default=8, help="prefill requests (one delta each)")
p.add_argument("--ptok", type=int, default=256, help="tokens per prefill request")
p.add_argument("--decode", type=int, default=0, help="extra decode tokens (spread over other deltas)")
p.add_argument("--iters", type=int, default=20)
p.add_argument("--shapes", default="5120x5120,13824x5120,5120x13824")
p.add_argument("--pf-min", type=int, default=64)
args = p.parse_args()

dev = torch.device("cuda", 0)
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 2250.0}
peak = float(peaks["bf16_tflops"])
gen = torch.Generator(device=dev)
gen.manual_seed(14)
err = ErrFlag(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
D = args.prefill + (8 if args.decode else 0)
for shp in args.shapes.split(","):
    out, inp = map(int, shp.split("x"))
    W = random_base(out, inp, gen, dev)
    nats = [random_native_delta(out, inp, args.bits, gen, dev, err) for _ in range(D)]
    table = DeltaTable(nats, out, inp)
    base = NativeBase(W)
    ids = np.concatenate([np.full(args.ptok, d, np.int32) for d in range(args.prefill)] +
                         [args.prefill + (np.arange(args.decode) % 8).astype(np.int32)])
    T = ids.size
    X = torch.randn(T, inp, device=dev, generator=gen).to(torch.bfloat16)
    plan = Plan(ids, table.kinds, D, device=dev, pf_min=args.pf_min)
    Y = torch.empty(T, out, dtype=torch.bfloat16, device=dev)
    for _ in range(3):
        sbmm_forward(X, plan, base, table, Y=Y)
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.iters):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sbmm_forward(X, plan, base, table, Y=Y)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    t = float(np.median(ts))
    Tp = args.prefill * args.ptok
    f_alg = 2.0 * T * out * inp + 2.0 * T * out * inp / 2
    f_exec_pf = 2.0 * Tp * out * inp * 2  # base + dense-dequantised delta on the prefill rows
    print(json.dumps({"shape": shp, "T": T, "t_pf": plan.t_pf, "n_pf_jobs": plan.n_pf_jobs, "us": t * 1e6,
                      "alg_tflops": f_alg / t / 1e12, "exec_pf_tflops": f_exec_pf / t / 1e12,
                      "exec_frac_of_peak": f_exec_pf / t / 1e12 / peak, "peak_tflops": peak}), flush=True)
    del nats, table, base, W
    torch.cuda.empty_cache()
err.raise_if_set("synthetic upload")
