"""Timeline of CTA 0 of the fused kernel (needs the DZ_TRACE build: _build.py --trace).

Events: 1 producer waits for a free stage, 2 producer got it and issues TMA, 3 consumer warp 0
got a full stage, 4 consumer warp 0 released it, 5 item epilogue done.
  DZ_B200_LIB=paper_2312_05215_b200/_dz_b200_trace.so python tools/trace.py [kbench args]
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

out, inp, T, D = 4096, 4096, int(os.environ.get("T", "64")), int(os.environ.get("D", "32"))
case = os.environ.get("CASE", "base_plus_1delta")
dev = torch.device("cuda")
gen = torch.Generator(device=dev)
gen.manual_seed(1)
base = NativeBase(random_base(out, inp, gen, dev))
nats = [random_native_delta(out, inp, 4, gen, dev) for _ in range(D)]
table = DeltaTable(nats, out, inp)
X = torch.randn(T, inp, device=dev).to(torch.bfloat16)
ids = np.zeros(T, np.int32) if case == "base_plus_1delta" else np.random.default_rng(12).permutation(
    [i % D for i in range(T)]).astype(np.int32)
plan = Plan(ids, table.kinds, D, with_base=case != "deltas_only")
ws = Workspace()
lib = L.lib()
lib.dz_trace_read.restype = C.c_int
lib.dz_trace_read.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros((8192, 4), dtype=np.uint64)
DBG = int(os.environ.get("DEBUG", "0"))
for _ in range(3):
    sbmm_forward(X, plan, base if case != "deltas_only" else None, table, workspace=ws, debug=DBG)
torch.cuda.synchronize()
lib.dz_trace_read(buf.ctypes.data, 8192)
sbmm_forward(X, plan, base if case != "deltas_only" else None, table, workspace=ws, debug=DBG)
torch.cuda.synchronize()
n = lib.dz_trace_read(buf.ctypes.data, 8192)
ev = buf[:n]
ev = ev[np.argsort(ev[:, 0], kind="stable")]
t0 = ev[0, 0]
print(f"events {n}")
for row in ev[:1500]:
    print(f"{(int(row[0]) - int(t0)):9d} cyc  w{int(row[1]) >> 8} ev{int(row[1]) & 255} item={int(row[2])} x={int(row[3])}")
