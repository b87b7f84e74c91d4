"""GPU: the on-device plan (dz_plan_device) reproduces the host plan (dz_plan, the reference's
stable group_by_delta, inference.py:106-123) exactly, drives the fused kernel to bit-identical
results, flags unknown slots, and works inside a captured CUDA graph with changing slots."""

import ctypes as C

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2312_05215_b200 import engine
    return engine


@pytest.mark.parametrize("T,D,seed", [(1, 1, 0), (64, 32, 1), (200, 7, 2), (777, 40, 3), (4096, 300, 4)])
def test_device_plan_matches_host_plan(E, T, D, seed):
    from paper_2312_05215_b200 import _lib as L
    rng = np.random.default_rng(seed)
    ids = rng.integers(0, D, T).astype(np.int32)
    kinds = np.where(rng.random(D) < 0.2, L.DZ_KIND_DENSE, L.DZ_KIND_SPARSE4).astype(np.int32)
    hp = E.Plan(ids, kinds, D, upload=False, pf_min=0)
    dp = E.DevicePlan(T, kinds, D).update(torch.from_numpy(ids).cuda())
    dp.check()
    n = int(dp.n_jobs_dev.item())
    assert n == hp.n_jobs
    assert np.array_equal(dp.order.cpu().numpy()[:T], hp.order_host)
    jobs = np.frombuffer(dp.jobs.cpu().numpy().tobytes(), dtype=np.int32).reshape(-1, 4)[:n]
    assert np.array_equal(jobs, hp.jobs_host)


def test_device_plan_unknown_slot(E):
    from paper_2312_05215_b200.errors import UnknownDeltaError
    dp = E.DevicePlan(4, np.ones(3, np.int32), 3).update(torch.tensor([0, 1, 5, 2], dtype=torch.int32).cuda())
    with pytest.raises(UnknownDeltaError):
        dp.check()


def test_device_plan_drives_kernel_in_graph(E):
    rng = np.random.default_rng(9)
    rows, cols, D, T = 256, 512, 6, 48
    ods = [O.random_packed_delta(rng, rows, cols, 4) for _ in range(D)]
    table = E.DeltaTable([E.NativeDelta.from_layer_delta(o) for o in ods], rows, cols)
    base = E.NativeBase((torch.randn(rows, cols, device="cuda") / np.sqrt(cols)).to(torch.bfloat16))
    X = torch.randn(T, cols, device="cuda").to(torch.bfloat16)
    slots = torch.zeros(T, dtype=torch.int32, device="cuda")
    dp = E.DevicePlan(T, table.kinds, D)
    Y = torch.empty(T, rows, dtype=torch.bfloat16, device="cuda")
    ws = E.Workspace()

    def step():
        dp.update(slots)
        E.sbmm_forward(X, dp, base, table, Y=Y, workspace=ws)

    slots.copy_(torch.from_numpy(rng.integers(0, D, T).astype(np.int32)))
    step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        step()
    for trial in range(3):  # new slots every replay, no host planning
        ids = rng.integers(0, D, T).astype(np.int32)
        slots.copy_(torch.from_numpy(ids))
        g.replay()
        torch.cuda.synchronize()
        ref = E.sbmm_forward(X, E.Plan(ids, table.kinds, D), base, table)
        assert torch.equal(Y, ref), trial


def _groups(rng, sizes, D):
    ids = np.concatenate([np.full(n, d, np.int32) for d, n in enumerate(sizes)] +
                         [rng.integers(0, D, 37).astype(np.int32)])
    return ids[rng.permutation(ids.size)]


@pytest.mark.parametrize("sizes,pf_min,seed", [([300, 250, 20, 5], 192, 0), ([600, 33, 260, 0, 241], 64, 1),
                                               ([10, 5, 3], 192, 2), ([500], 1, 3), ([1000, 700, 480], 240, 4)])
def test_device_mixed_plan_matches_host_mixed_plan(E, sizes, pf_min, seed):
    """dz_plan_mixed_device == dz_plan_mixed (staging perm, decode order, prefill and decode jobs,
    t_pf), dense slots excluded from prefill like the host planner."""
    from paper_2312_05215_b200 import _lib as L
    rng = np.random.default_rng(seed)
    D = len(sizes) + 3
    ids = _groups(rng, sizes, D)
    kinds = np.full(D, L.DZ_KIND_SPARSE4, np.int32)
    kinds[-1] = L.DZ_KIND_DENSE
    T = ids.size
    hp = E.Plan(ids, kinds, D, upload=False, pf_min=pf_min)
    dp = E.DevicePlan(T, kinds, D, mixed=True, pf_min=pf_min).update(torch.from_numpy(ids).cuda())
    dp.check()
    n_pf, n_dec, t_pf = (int(v) for v in dp.counts.cpu().numpy())
    assert (n_pf, t_pf) == (hp.n_pf_jobs, hp.t_pf)
    assert n_pf + n_dec == hp.n_jobs
    jobs = np.frombuffer(dp.jobs.cpu().numpy().tobytes(), dtype=np.int32).reshape(-1, 4)
    assert np.array_equal(jobs[:n_pf], hp.jobs_host[:n_pf])
    assert np.array_equal(jobs[T:T + n_dec], hp.jobs_host[n_pf:])
    if hp.perm_host is not None:
        assert np.array_equal(dp.perm.cpu().numpy()[:T], hp.perm_host)
    assert np.array_equal(dp.order.cpu().numpy()[:T - t_pf], hp.order_host[:T - t_pf])


def test_device_mixed_plan_drives_k3_and_k2_in_graph(E):
    """A captured graph of [device mixed plan -> gather -> K3 -> K2 -> finalize] replays with
    changing slots (prefill groups appear and vanish) and equals the host mixed plan bit for bit."""
    rng = np.random.default_rng(7)
    rows, cols, D = 384, 512, 5
    ods = [O.random_packed_delta(rng, rows, cols, 4) for _ in range(D)]
    table = E.DeltaTable([E.NativeDelta.from_layer_delta(o) for o in ods], rows, cols)
    base = E.NativeBase((torch.randn(rows, cols, device="cuda") / np.sqrt(cols)).to(torch.bfloat16))
    T = 400
    X = torch.randn(T, cols, device="cuda").to(torch.bfloat16)
    slots = torch.zeros(T, dtype=torch.int32, device="cuda")
    dp = E.DevicePlan(T, table.kinds, D, mixed=True, pf_min=128)
    Y = torch.empty(T, rows, dtype=torch.float32, device="cuda")
    ws = E.Workspace()
    cases = [_groups(rng, [250, 60], D)[:T], rng.integers(0, D, T).astype(np.int32), _groups(rng, [300], D)[:T]]
    cases = [np.resize(c, T).astype(np.int32) for c in cases]
    slots.copy_(torch.from_numpy(cases[0]))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        dp.update(slots)
        E.sbmm_forward(X, dp, base, table, Y=Y, workspace=ws)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        dp.update(slots)
        E.sbmm_forward(X, dp, base, table, Y=Y, workspace=ws)
    for ids in cases:
        slots.copy_(torch.from_numpy(ids))
        g.replay()
        torch.cuda.synchronize()
        dp.check()
        ref = E.sbmm_forward(X, E.Plan(ids, table.kinds, D, pf_min=128), base, table, y_dtype=torch.float32)
        assert torch.equal(Y, ref)
