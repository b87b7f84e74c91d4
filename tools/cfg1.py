#!/usr/bin/env python3
"""BASELINE configs[0] — the reference's own CPU-runnable case: one 4096x4096 linear, base + 4
ΔCompress deltas (4-bit 2:4), 16 tokens mixed across the deltas (ids i % 4, permuted, seed 11).

Times, on the same synthetic inputs:
  * the reference algorithm on the host (oracle port of inference.sbmm, numpy f64, one call);
  * this package's drop-in `sbmm` (numpy in / numpy out, the reference signature: uploads the
    deltas and runs the fused kernel each call — the reference dequantises per call too);
  * the device-resident path (deltas resident, one fused launch, CUDA events; L2 flushed), issued
    eagerly (device_us: includes the Python argument building, the GPU idles meanwhile) and as a
    CUDA graph replay (graph_us, how the serving stack issues it).
and checks the per-token rel-err against the oracle (<= 1e-2)."""

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402  (the checker / CPU arm only)
import paper_2312_05215_b200 as P  # noqa: E402
from paper_2312_05215_b200.engine import DeltaTable, NativeBase, NativeDelta, Plan, sbmm_forward  # noqa: E402


def main():
    rng = np.random.default_rng(11)
    n, D, T = 4096, 4, 16
    W = rng.normal(0, 1 / np.sqrt(n), (n, n)).astype(np.float32)
    W = torch.from_numpy(W).to(torch.bfloat16).float().numpy().astype(np.float64)  # bf16-representable
    ods = [O.random_packed_delta(rng, n, n, 4) for _ in range(D)]
    ids = rng.permutation(np.arange(T) % D).astype(np.int32)
    X = torch.from_numpy(rng.normal(0, 1, (T, n)).astype(np.float32)).to(torch.bfloat16).double().numpy()

    t0 = time.perf_counter()
    ref = O.sbmm_matrix(W, dict(enumerate(ods)), ids, X)
    t_cpu = time.perf_counter() - t0

    lds = {d: P.LayerDelta(name="l", rows=n, cols=n, packed_values=o.packed_values, index_stream=o.index_stream,
                           scales=o.scales, bits=4, sparsity="two_of_four", group_size=128) for d, o in enumerate(ods)}
    batch = P.BatchInput([(i, int(ids[i]), X[i]) for i in range(T)])
    from paper_2312_05215_b200.resident import CACHE
    CACHE.enabled = False  # the round-1 behaviour: upload + re-layout every call
    P.sbmm(W, lds, batch)  # warm-up (library load, kernel attributes)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = P.sbmm(W, lds, batch)
    t_api_cold = time.perf_counter() - t0
    CACHE.enabled = True  # residency: the same objects' uploads are reused (resident.py)
    P.sbmm(W, lds, batch)
    ts_api = []
    for _ in range(20):
        t0 = time.perf_counter()
        out = P.sbmm(W, lds, batch)
        ts_api.append(time.perf_counter() - t0)
    t_api = float(np.median(ts_api))
    Y = np.stack([out[i] for i in range(T)])
    err_api = float((np.linalg.norm(Y - ref, axis=1) / np.linalg.norm(ref, axis=1)).max())

    dev = torch.device("cuda", 0)
    table = DeltaTable([NativeDelta.from_layer_delta(o) for o in ods], n, n)
    base = NativeBase(torch.from_numpy(W.astype(np.float32)).to(dev).to(torch.bfloat16))
    plan = Plan(ids, table.kinds, D, device=dev)
    Xd = torch.from_numpy(X.astype(np.float32)).to(dev).to(torch.bfloat16)
    Yd = torch.empty(T, n, dtype=torch.bfloat16, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ts = []
    for i in range(23):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sbmm_forward(Xd, plan, base, table, Y=Yd)
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e-3)
    t_dev = float(np.median(ts))  # eager: includes the Python argument building before the launch
    # the same launch captured in a CUDA graph (how the serving stack issues it), L2 flushed
    def graph_time(**kw):
        s_ = torch.cuda.Stream()
        s_.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s_):
            sbmm_forward(Xd, plan, base, table, Y=Yd, **kw)
        torch.cuda.current_stream().wait_stream(s_)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            sbmm_forward(Xd, plan, base, table, Y=Yd, **kw)
        tg = []
        for i in range(23):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            if i >= 3:
                tg.append(a.elapsed_time(b) * 1e-3)
        return float(np.median(tg))

    t_graph = graph_time()
    variants = {f"base_splits={k}": graph_time(base_splits=k) * 1e6 for k in (1, 2, 4)}
    variants["fused_merge"] = graph_time(fused_merge=True) * 1e6
    err_dev = float((np.linalg.norm(Yd.double().cpu().numpy() - ref, axis=1) / np.linalg.norm(ref, axis=1)).max())
    from paper_2312_05215_b200.synth import linear_algorithmic_bytes
    nbytes = linear_algorithmic_bytes(n, n, 4, D, T)
    print(json.dumps({
        "config": "cfg1: 4096x4096, 4 x 4-bit 2:4 deltas, T=16 (ids i%4)",
        "cpu_reference_s": t_cpu, "cpu_tokens_per_s": T / t_cpu,
        "api_sbmm_s": t_api, "api_tokens_per_s": T / t_api, "api_rel_err": err_api,
        "api_sbmm_no_residency_s": t_api_cold,
        "device_us": t_dev * 1e6, "device_tokens_per_s": T / t_dev, "device_GBps": nbytes / t_dev / 1e9,
        "device_rel_err": err_dev, "algorithmic_bytes": nbytes,
        "graph_us": t_graph * 1e6, "graph_GBps": nbytes / t_graph / 1e9, "graph_us_variants": variants,
    }), flush=True)
    assert err_api <= 1e-2 and err_dev <= 1e-2


if __name__ == "__main__":
    main()
