#!/usr/bin/env python3
"""GPU ΔCompress cost of one Llama-2-7B decoder layer (7 linears, 4-bit 2:4, gs 128, block 32),
extrapolated to the 32-layer model. Calibration: 2048 samples per layer input, synthetic.

Per distinct linear shape: Hessian (DSYRK), inverse-Hessian factor (cuSOLVER), and the OBS
solver (dz_obs_compress), CUDA events, median of 3. q/k/v share their input (one Hessian and
factor), as do gate/up. Prints one JSON line."""

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2312_05215_b200.formats import CompressConfig  # noqa: E402
from paper_2312_05215_b200.solver import hessian_device, inverse_cholesky_factor, obs_solve_device  # noqa: E402


def timed(fn, reps=3):
    ts, out = [], None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), out


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    cfg = CompressConfig(bits=4)
    n_samples = 2048
    # (in, out, number of linears with this shape, linears sharing one Hessian)
    shapes = [(4096, 4096, 4, 3), (4096, 11008, 2, 2), (11008, 4096, 1, 1)]
    res, layer_ms = {}, 0.0
    for cin, cout, n_lin, share in shapes:
        x = torch.randn(cin, n_samples, generator=g, device=dev, dtype=torch.float64)
        t_h, h = timed(lambda: hessian_device(x, cfg.damping))
        t_u, u = timed(lambda: inverse_cholesky_factor(h))
        d0 = torch.randn(cout, cin, generator=g, device=dev, dtype=torch.float64) * 0.01
        t_s, _ = timed(lambda: obs_solve_device(d0.clone(), u, cfg))
        n_factor = 1 + (n_lin - share)  # q/k/v share one factor, o has its own
        total = n_factor * (t_h + t_u) + n_lin * t_s
        res[f"{cout}x{cin}"] = {"hessian_ms": t_h, "factor_ms": t_u, "solver_ms": t_s, "linears": n_lin,
                               "factors": n_factor, "total_ms": total}
        layer_ms += total
        del x, h, u, d0
        torch.cuda.empty_cache()
    print(json.dumps({"model": "llama2-7b decoder layer, 4-bit 2:4, gs 128, block 32, 2048 calibration samples",
                      "per_shape": res, "layer_ms": layer_ms, "model_32_layers_s": layer_ms * 32 / 1e3}))


if __name__ == "__main__":
    main()
