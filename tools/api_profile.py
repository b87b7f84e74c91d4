#!/usr/bin/env python3
"""Where the time of one drop-in `sbmm` call goes (cfg1 shapes: 4096x4096, 4 deltas, T=16):
cProfile of repeated calls with residency on, top functions by own time."""

import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402  (synthetic deltas only)
import paper_2312_05215_b200 as P  # noqa: E402


def main():
    rng = np.random.default_rng(11)
    n, D, T = 4096, 4, 16
    W = torch.from_numpy(rng.normal(0, 1 / 64, (n, n)).astype(np.float32)).to(torch.bfloat16).double().numpy()
    ods = [O.random_packed_delta(rng, n, n, 4) for _ in range(D)]
    ids = rng.permutation(np.arange(T) % D).astype(np.int32)
    X = rng.normal(0, 1, (T, n))
    lds = {d: P.LayerDelta(name="l", rows=n, cols=n, packed_values=o.packed_values, index_stream=o.index_stream,
                           scales=o.scales, bits=4, sparsity="two_of_four", group_size=128) for d, o in enumerate(ods)}
    batch = P.BatchInput([(i, int(ids[i]), X[i]) for i in range(T)])
    for _ in range(5):
        P.sbmm(W, lds, batch)
    torch.cuda.synchronize()
    ts = []
    for _ in range(200):
        t0 = time.perf_counter()
        P.sbmm(W, lds, batch)
        ts.append(time.perf_counter() - t0)
    print(f"sbmm median {np.median(ts) * 1e6:.1f} us, p10 {np.percentile(ts, 10) * 1e6:.1f} us")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        P.sbmm(W, lds, batch)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
