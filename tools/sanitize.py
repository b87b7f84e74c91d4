#!/usr/bin/env python3
"""Small invocations of every product kernel for compute-sanitizer (memcheck / racecheck /
synccheck): K1 unpack (f64/f32/bf16), the native re-layout, K2 decode (base splits 1/3, dense
delta kind, no-base table, fused merge), K3 prefill through a mixed plan (sparse and dense
variants), the on-device plan, and the ΔCompress solver. Shapes are small so a sanitizer run
finishes in minutes; every result is checked against the oracle as well.

    compute-sanitizer --tool racecheck python tools/sanitize.py
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_2312_05215_b200 as P  # noqa: E402
from paper_2312_05215_b200 import engine as E  # noqa: E402


def rel(y, r):
    return float((np.linalg.norm(y - r, axis=1) / np.maximum(np.linalg.norm(r, axis=1), 1e-30)).max())


def main():
    torch.cuda.set_device(0)
    rng = np.random.default_rng(7)
    rows, cols, D = 320, 640, 3
    ods = [O.random_packed_delta(rng, rows, cols, b) for b in (4, 2, 3)]
    for ld in ods[:2]:
        for dt in (torch.float64, torch.float32, torch.bfloat16):
            P.dequantize_layer_device(ld, dt)
    nat = [E.NativeDelta.from_layer_delta(o) for o in ods]
    nat[0].to_dense_f32()
    W = rng.normal(0, 1 / np.sqrt(cols), (rows, cols))
    Wb = torch.from_numpy(W.astype(np.float32)).cuda().to(torch.bfloat16)
    Wh = Wb.float().double().cpu().numpy()
    base = E.NativeBase(Wb)
    table = E.DeltaTable(nat, rows, cols)
    T = 40
    ids = rng.integers(0, D, T).astype(np.int32)
    X = torch.randn(T, cols, device="cuda").to(torch.bfloat16)
    R = O.sbmm_matrix(Wh, dict(enumerate(ods)), ids, X.float().double().cpu().numpy())
    for kw in ({}, {"base_splits": 3}, {"fused_merge": True}, {"delta_splits": 2}):
        Y = E.sbmm_forward(X, E.Plan(ids, table.kinds, D), base, table, y_dtype=torch.float32, **kw)
        assert rel(Y.double().cpu().numpy(), R) <= 1e-2, kw
    dp = E.DevicePlan(T, table.kinds, D).update(torch.from_numpy(ids).cuda())
    E.sbmm_forward(X, dp, base, table, y_dtype=torch.float32)
    dp.check()
    # dense delta kind + no-base table
    dn = E.NativeDelta.from_dense_bf16(P.dequantize_layer_device(ods[0], torch.bfloat16))
    tdn = E.DeltaTable([dn, nat[1]], rows, cols)
    E.sbmm_forward(X, E.Plan(ids % 2, tdn.kinds, 2), base, tdn, y_dtype=torch.float32)
    E.sbmm_forward(X, E.Plan(ids % 2, tdn.kinds, 2, with_base=False), None, tdn, y_dtype=torch.float32)
    # mixed plan: K3 (sparse tcgen05 and the dense-dequantised variants) + K2
    ids2 = np.concatenate([np.zeros(200, np.int32), rng.integers(1, D, 24).astype(np.int32)])
    X2 = torch.randn(ids2.size, cols, device="cuda").to(torch.bfloat16)
    R2 = O.sbmm_matrix(Wh, dict(enumerate(ods)), ids2, X2.float().double().cpu().numpy())
    plan2 = E.Plan(ids2, table.kinds, D, pf_min=128)
    for v in (0, 1, 2):
        Y2 = E.sbmm_forward(X2, plan2, base, table, y_dtype=torch.float32, prefill_variant=v)
        assert rel(Y2.double().cpu().numpy(), R2) <= 1e-2, v
    # GPU ΔCompress
    xs = rng.normal(0, 1, (64, 128))
    h = O.compute_hessian(xs, 0.01)
    P.obs_compress_layer(rng.normal(0, 0.01, (32, 64)), h, P.CompressConfig(bits=4, group_size=32, block_size=16),
                         u=O.inverse_cholesky_factor(h))
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
