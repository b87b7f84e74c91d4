#!/usr/bin/env python3
"""Layer-stack bench for the BASELINE configs other than the headline (parity/coverage evidence;
the headline line is bench.py):

  cfg3  13B layers, 64 deltas 2-bit 2:4, 8 prefill requests x 256 tokens (8 distinct deltas)
        + 128 decode tokens (i % 64):
        python tools/stackbench.py --model 13b --layers 16 --deltas 64 --bits 2 --prefill 8x256 --decode 128
  cfg4  70B layers, 16 deltas 4-bit, decode 64 — one tensor-parallel rank's shard (rank 0 of
        --world N) timed alone on this GPU (the NCCL all-reduce is not in this number):
        python tools/stackbench.py --model 70b --layers 8 --deltas 16 --decode 64 --world 8
  cfg5  7B shapes, Zipf(1.5) request mix over D deltas, batch B (simulator.py:107-110):
        python tools/stackbench.py --model 7b --layers 4 --deltas 128 --sweep --zipf 1.5

Prints one JSON line: tokens/s of the step, algorithmic HBM bytes and GB/s (base +
distinct routed deltas + activations), algorithmic TFLOP/s (base 2·T·out·in + kept delta MACs),
and the fractions of the measured peaks (MEASURED_PEAKS.json). The step runs in a CUDA graph;
weights and deltas (> L2) are streamed once per step.
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2312_05215_b200.engine import Plan  # noqa: E402
from paper_2312_05215_b200.stack import FUSED, LlamaStack  # noqa: E402


def zipf_ids(n: int, D: int, alpha: float, seed: int) -> np.ndarray:
    """Zipf-distributed delta ids over D deltas (rank-frequency p_k ~ k^-alpha)."""
    rng = np.random.default_rng(seed)
    p = 1.0 / np.arange(1, D + 1) ** alpha
    p /= p.sum()
    return rng.choice(D, size=n, p=p).astype(np.int32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="7b")
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--deltas", type=int, default=32)
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--decode", type=int, default=64)
    ap.add_argument("--prefill", default="", help="RxL: R prefill requests of L tokens, one new delta each")
    ap.add_argument("--zipf", type=float, default=0.0)
    ap.add_argument("--world", type=int, default=1)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--pf-min", type=int, default=None)
    ap.add_argument("--seed", type=int, default=13)
    ap.add_argument("--sweep", action="store_true", help="cfg5: D in 1..128 x batch in 1..256, Zipf ids")
    ap.add_argument("--base-splits", type=int, default=0, help="K-splits of the decode base GEMM (0 = by shape)")
    ap.add_argument("--max-batch", type=int, default=256, help="sweep: largest batch")
    ap.add_argument("--points", default="", help="sweep subset: D:B,D:B,...")
    ap.add_argument("--overlap-sms", type=int, default=None, help="mixed plans: SMs for K3 (0 = no overlap)")
    ap.add_argument("--chain", action="store_true", help="decode step as one chained launch (dz_sbmm_chain)")
    ap.add_argument("--fused-merge", action="store_true", help="in-kernel merge (k_sbmm<true>)")
    ap.add_argument("--prefill-variant", type=int, default=0, help="K3 delta product (0 sparse, 1/2 dense MT=1/2)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)

    R, L = (map(int, args.prefill.split("x")) if args.prefill else (0, 0))  # noqa: N806
    if args.zipf > 0:
        dec = zipf_ids(args.decode, args.deltas, args.zipf, args.seed)
    else:
        dec = (np.random.default_rng(args.seed).permutation(np.arange(args.decode) % args.deltas)).astype(np.int32)
    pre = np.repeat(np.arange(R, dtype=np.int32) % args.deltas, L)  # request r on delta r
    ids = np.concatenate([pre, dec]).astype(np.int32)
    T = int(ids.size)

    st = LlamaStack(args.model, args.layers, args.deltas, args.bits, dev, rank=args.rank, world=args.world)
    st.world = 1  # one rank's shard timed alone: no collective in this process
    st.base_splits = args.base_splits
    st.overlap_sms = args.overlap_sms
    st.fused_merge = args.fused_merge
    st.prefill_variant = args.prefill_variant
    if args.sweep:
        Ds = [d for d in (1, 2, 4, 8, 16, 32, 64, 128) if d <= args.deltas]
        Bs = tuple(b for b in (1, 2, 4, 8, 16, 32, 64, 128, 256) if b <= args.max_batch)
        pts = [tuple(map(int, p.split(":"))) for p in args.points.split(",")] if args.points else \
            [(D, B) for D in Ds for B in Bs]
        for D, B in pts:
            if True:
                sid = zipf_ids(B, D, args.zipf or 1.5, args.seed + 1000 * D + B)
                print(json.dumps(run(args, st, sid, dev, extra={"sweep_D": D, "batch": B,
                                                                "base_splits": args.base_splits})), flush=True)
        return
    print(json.dumps(run(args, st, ids, dev)), flush=True)


def run(args, st, ids, dev, extra=None):
    T = int(ids.size)
    plan = Plan(ids, st.kinds, args.deltas, device=dev, pf_min=args.pf_min)
    bufs = st.buffers(T)
    bufs["x"].copy_(torch.randn(T, bufs["x"].shape[1], device=dev).to(torch.bfloat16))
    step = (lambda: st.step_chained(plan, bufs)) if args.chain else (lambda: st.step(plan, bufs))
    step()
    torch.cuda.synchronize()
    s_ = torch.cuda.Stream()
    s_.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_):
        step()
    torch.cuda.current_stream().wait_stream(s_)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(args.warmup):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    del g

    # algorithmic bytes / flops of one step on this rank
    distinct = int(np.unique(ids).size)
    lb = st.launch_bytes(T, distinct)
    step_bytes = args.layers * sum(lb.values())
    l0 = st.stack[0]
    flops = 0.0
    for f in FUSED:
        o, i = l0[f].out, l0[f].inp
        flops += 2.0 * T * o * i + 2.0 * T * o * i / 2  # base + kept delta MACs (2:4)
    flops *= args.layers
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "bf16_tflops": 2250.0}
    gbs = step_bytes / (ms * 1e-3) / 1e9
    tfl = flops / (ms * 1e-3) / 1e12
    out = {
        "model": args.model, "layers": args.layers, "deltas": args.deltas, "bits": args.bits, "T": T,
        "prefill": args.prefill or None, "decode": args.decode, "zipf": args.zipf or None,
        "distinct_deltas": distinct, "tp": f"rank {args.rank} of {args.world}" if args.world > 1 else None,
        "t_pf": plan.t_pf, "n_pf_jobs": plan.n_pf_jobs, "ms_per_step": ms, "tokens_per_s": T / (ms * 1e-3),
        "step_bytes": step_bytes, "GBps": gbs, "hbm_frac": gbs / peaks["hbm_gbs"],
        "TFLOPs": tfl, "tensor_frac": tfl / peaks["bf16_tflops"], "per_layer_ms": ms / args.layers,
    }
    out.update(extra or {})
    return out


if __name__ == "__main__":
    main()
