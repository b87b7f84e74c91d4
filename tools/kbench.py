"""Micro-benchmarks of the fused SBMM kernel on one linear shape (isolates base / delta paths).

  python tools/kbench.py [--out 4096] [--in 4096] [--deltas 32] [--tokens 64]
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2312_05215_b200 import _lib as L  # noqa: E402
from paper_2312_05215_b200.engine import DeltaTable, NativeBase, Plan, Workspace, sbmm_forward  # noqa: E402
from paper_2312_05215_b200.synth import delta_algorithmic_bytes, random_base, random_native_delta  # noqa: E402


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3  # us


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out", type=int, default=4096)
    p.add_argument("--in", dest="inp", type=int, default=4096)
    p.add_argument("--deltas", type=int, default=32)
    p.add_argument("--tokens", type=int, default=64)
    p.add_argument("--bits", type=int, default=4)
    p.add_argument("--grid", type=int, default=0)
    p.add_argument("--case", default="")
    p.add_argument("--debug", type=int, default=0)
    args = p.parse_args()
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    out, inp, D, T = args.out, args.inp, args.deltas, args.tokens
    base = NativeBase(random_base(out, inp, gen, dev))
    nats = [random_native_delta(out, inp, args.bits, gen, dev) for _ in range(D)]
    table = DeltaTable(nats, out, inp)
    X = torch.randn(T, inp, device=dev).to(torch.bfloat16)
    ws = Workspace()
    ids = np.random.default_rng(12).permutation([i % D for i in range(T)]).astype(np.int32)
    res = {}
    dbytes = delta_algorithmic_bytes(out, inp, args.bits)
    cases = {
        "full": (ids, True, D * dbytes + 2 * out * inp),
        "deltas_only": (ids, False, D * dbytes),
        "base_plus_1delta": (np.zeros(T, np.int32), True, dbytes + 2 * out * inp),
        "1delta_only": (np.zeros(T, np.int32), False, dbytes),
        "base_only": (ids, True, 2 * out * inp),  # run with --debug 2 (delta items dropped)
    }
    for name, (sl, wb, nbytes) in cases.items():
        if args.case and name != args.case:
            continue
        plan = Plan(sl, table.kinds, D, with_base=wb)
        us = timeit(lambda: sbmm_forward(X, plan, base if wb else None, table, workspace=ws, grid=args.grid, debug=args.debug))
        res[name] = {"us": round(us, 1), "GBps": round(nbytes / us / 1e3, 1), "n_jobs": plan.n_jobs}
    print(json.dumps({"shape": [out, inp], "D": D, "T": T, **res}))


if __name__ == "__main__":
    main()
