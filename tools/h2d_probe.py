import torch, time
dev = torch.device("cuda", 0)
for n in (1 << 16, 1 << 19, 1 << 22, 1 << 25):
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    t_h2d = e0.elapsed_time(e1) / 20
    e0.record()
    for _ in range(20):
        h.copy_(d, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    t_d2h = e0.elapsed_time(e1) / 20
    # in a graph
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        d.copy_(h, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    t_g = e0.elapsed_time(e1) / 20
    print(f"{n/1e6:.2f} MB: H2D {t_h2d*1e3:.1f} us ({n/t_h2d/1e6:.1f} GB/s), D2H {t_d2h*1e3:.1f} us, graph H2D {t_g*1e3:.1f} us")
