import sys, os, time, json
sys.path.insert(0, '/root/repo')
os.chdir('/root/repo')
import numpy as np, torch
import bench as B
from paper_2312_05215_b200.engine import Plan, DevicePlan
from paper_2312_05215_b200.stack import LlamaStack
dev = torch.device('cuda', 0); torch.cuda.set_device(dev)
st = LlamaStack('7b', 32, 32, 4, dev)
ids = B.token_ids(); kinds = st.kinds
plan = Plan(ids, kinds, 32, device=dev)
bufs = st.buffers(64)
st.step(plan, bufs); torch.cuda.synchronize()
def cap(fn):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): fn()
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g): fn()
    return g
g1 = cap(lambda: st.step(plan, bufs))
dplan = DevicePlan(64, kinds, 32, device=dev)
slots = torch.from_numpy(ids).cuda()
g2 = cap(lambda: (dplan.update(slots), st.step(dplan, bufs)))
xh = torch.randn(64, 4096).to(torch.bfloat16).pin_memory(); yh = torch.empty(64, 4096, dtype=torch.bfloat16).pin_memory()
def full():
    bufs['x'].copy_(xh, non_blocking=True); dplan.update(slots); st.step(dplan, bufs); yh.copy_(bufs['down'], non_blocking=True)
g3 = cap(full)
def t(g, n=10):
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): g.replay()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
for rep in range(2):
    print('step-only', round(t(g1), 3), 'devplan+step', round(t(g2), 3), 'copies+devplan+step', round(t(g3), 3), 'step-only', round(t(g1), 3), flush=True)
