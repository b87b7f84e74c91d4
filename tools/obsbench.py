#!/usr/bin/env python3
"""Time the GPU ΔCompress solver on a Llama-shaped layer (default 4096 x 4096, 4-bit 2:4, gs 128,
block 32) and the oracle restatement of the reference solver on a row sample of the same layer.

Prints one JSON line: factor (cuSOLVER) and solver (dz_obs_compress) times from CUDA events, the
solver's f64 flop rate for the trailing updates (rows * cols^2 * ~1 flops... counted exactly),
and the CPU reference time scaled from the row sample (rows are independent given U)."""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2312_05215_b200.formats import CompressConfig  # noqa: E402
from paper_2312_05215_b200.solver import hessian_device, inverse_cholesky_factor, obs_solve_device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=4096)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--block", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cpu-rows", type=int, default=64)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    r, c = a.rows, a.cols
    cfg = CompressConfig(bits=a.bits, block_size=a.block)
    x = torch.randn(c, 2 * c, generator=g, device=dev, dtype=torch.float64)
    delta0 = torch.randn(r, c, generator=g, device=dev, dtype=torch.float64) * 0.01

    def ev():
        return torch.cuda.Event(enable_timing=True)

    t_h, t_u, t_s = [], [], []
    for i in range(a.reps + 1):
        e0, e1, e2, e3 = ev(), ev(), ev(), ev()
        d = delta0.clone()
        e0.record()
        h = hessian_device(x, cfg.damping)
        e1.record()
        u = inverse_cholesky_factor(h)
        e2.record()
        res = obs_solve_device(d, u, cfg)
        e3.record()
        torch.cuda.synchronize()
        if i:
            t_h.append(e0.elapsed_time(e1))
            t_u.append(e1.elapsed_time(e2))
            t_s.append(e2.elapsed_time(e3))
    ts = float(np.median(t_s)) * 1e-3
    flops = 0
    for i1 in range(0, c, a.block):
        i2 = min(i1 + a.block, c)
        flops += 2 * r * (i2 - i1) * (c - i2) + r * (i2 - i1) * (i2 - i1 - 1)  # trailing + in-block
    out = {"layer": f"{r}x{c}", "bits": a.bits, "block": a.block,
           "hessian_ms": float(np.median(t_h)), "factor_ms": float(np.median(t_u)), "solver_ms": ts * 1e3,
           "solver_f64_tflops": flops / ts / 1e12, "proxy_loss": float(res.loss.item())}
    # CPU: the oracle restatement of the reference solver on a row sample (rows are independent)
    import oracle as O
    hs, us = h.cpu().numpy(), u.cpu().numpy()
    dn = delta0[: a.cpu_rows].cpu().numpy()
    t0 = time.perf_counter()
    O.obs_compress_layer(dn, hs, a.bits, O.SPARSITY_2_4, 128, a.block, u=us)
    tc = time.perf_counter() - t0
    out.update({"cpu_rows": a.cpu_rows, "cpu_sample_s": tc, "cpu_full_layer_s_est": tc * r / a.cpu_rows,
                "cpu_threads": os.cpu_count()})
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
