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
