"""Per-item timeline of one fused launch across ALL CTAs (DZ_TRACE build).

  DZ_B200_LIB=paper_2312_05215_b200/_dz_b200_trace.so python tools/item_trace.py [out in [T D]]
  (FLUSH=1: the traced launch reads cold, L2 flushed before it)
Prints item-duration stats by kind, the CTA busy fraction and the tail.
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_05215_b200 import _lib as L  # noqa: E402
from paper_2312_05215_b200.engine import DeltaTable, NativeBase, Plan, Workspace, sbmm_forward  # noqa: E402
from paper_2312_05215_b200.synth import random_base, random_native_delta  # noqa: E402

out, inp = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (4096, 4096)
T, D = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (64, 32)
dev = torch.device("cuda")
gen = torch.Generator(device=dev)
gen.manual_seed(1)
base = NativeBase(random_base(out, inp, gen, dev))
nats = [random_native_delta(out, inp, 4, gen, dev) for _ in range(D)]
table = DeltaTable(nats, out, inp)
X = torch.randn(T, inp, device=dev).to(torch.bfloat16)
ids = np.random.default_rng(12).permutation([i % D for i in range(T)]).astype(np.int32)
plan = Plan(ids, table.kinds, D)
ws = Workspace()
for _ in range(3):
    sbmm_forward(X, plan, base, table, workspace=ws)
torch.cuda.synchronize()
if os.environ.get("FLUSH") == "1":
    torch.empty(256 << 20, dtype=torch.uint8, device=dev).zero_()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
sbmm_forward(X, plan, base, table, workspace=ws)
e1.record()
torch.cuda.synchronize()
n_base = 1  # T <= DZ_BASE_JOB_TOKENS: one base job
nsplit = 2 if out <= 4096 else 1  # the default split rule (dz_sbmm.cu base_splits, DZ_SPLIT_RULE 2)
n_items = ((out + 127) // 128) * n_base * nsplit + ((out + 255) // 256) * (plan.n_jobs - n_base)
lib = L.lib()
lib.dz_item_trace_read.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros((n_items, 3), dtype=np.uint64)
lib.dz_item_trace_read(buf.ctypes.data, n_items)
st, en = buf[:, 0].astype(np.int64), buf[:, 1].astype(np.int64)
cta = (buf[:, 2] >> np.uint64(32)).astype(np.int64)
kind = (buf[:, 2] & np.uint64(0xFFFFFFFF)).astype(np.int64)
t0 = st.min()
st, en = (st - t0) / 1e3, (en - t0) / 1e3
dur = en - st
print(f"kernel (events) {e0.elapsed_time(e1) * 1e3:.1f} us; items {n_items}; span {en.max():.1f} us")
for k in sorted(set(kind.tolist())):
    d = dur[kind == k]
    print(f"kind {k}: n={d.size} dur mean {d.mean():.2f} p50 {np.median(d):.2f} p90 {np.percentile(d, 90):.2f} max {d.max():.2f} us")
busy = np.zeros(cta.max() + 1)
first = np.full(cta.max() + 1, 1e9)
last = np.zeros(cta.max() + 1)
for c, a, b in zip(cta, st, en):
    busy[c] += b - a
    first[c] = min(first[c], a)
    last[c] = max(last[c], b)
print(f"CTAs {busy.size}: busy mean {busy.mean():.1f} us; last-end p10 {np.percentile(last, 10):.1f} p50 {np.median(last):.1f} max {last.max():.1f}; first-start max {first.max():.1f}")
starts = np.sort(st)
print("item starts at quantiles:", [round(float(np.percentile(starts, q)), 1) for q in (0, 25, 50, 75, 90, 100)])
