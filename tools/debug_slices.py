import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle as O
from paper_2312_05215_b200 import engine as E
rng = np.random.default_rng(3)
ws = E.Workspace()
def cnt(w):
    torch.cuda.synchronize()
    b = w.get(1, 1, torch.device("cuda"))[:33024].view(torch.int32).cpu().numpy()
    nz = np.nonzero(b)[0]
    return nz[:10], b[nz[:10]]
cases = []
for rows, cols, D, T in ((4096, 512, 3, 24), (96, 384, 2, 9), (1000, 256, 4, 70), (33, 128, 2, 5)):
    ods = [O.random_packed_delta(rng, rows, cols, 4) for _ in range(D)]
    table = E.DeltaTable([E.NativeDelta.from_layer_delta(o) for o in ods], rows, cols)
    base = E.NativeBase((torch.randn(rows, cols, device="cuda") / np.sqrt(cols)).to(torch.bfloat16))
    ids = rng.integers(0, D, T).astype(np.int32)
    X = torch.randn(T, cols, device="cuda").to(torch.bfloat16)
    cases.append((X, E.Plan(ids, table.kinds, D), base, table, ods, ids))
def err(y, c):
    X, p, b, t, ods, ids = c
    R = O.sbmm_matrix(b.W.float().double().cpu().numpy(), dict(enumerate(ods)), ids, X.float().double().cpu().numpy())
    return (np.linalg.norm(y.double().cpu().numpy() - R, axis=1) / np.linalg.norm(R, axis=1)).max()
for i, sp in ((2, 1), (2, 2), (2, 3), (0, 1), (3, 1)):
    c = cases[i]
    y = E.sbmm_forward(c[0], c[1], c[2], c[3], y_dtype=torch.float32, workspace=ws, base_splits=sp)
    print(i, sp, "err", err(y, c), "ws words", cnt(ws), flush=True)
ws2 = E.Workspace()
for i, sp in ((0, 1), (3, 1)):
    c = cases[i]
    y = E.sbmm_forward(c[0], c[1], c[2], c[3], y_dtype=torch.float32, workspace=ws2, base_splits=sp)
    print("fresh ws", i, sp, "err", err(y, c), "ws words", cnt(ws2), flush=True)
