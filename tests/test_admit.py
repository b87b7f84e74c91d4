"""Admission (scheduler.select_batch, scheduler.py:73-123): the oracle restatement pinned to 300
traces the reference scheduler produced (tests/golden/make_admit.py), and the on-device kernel
(dz_admit_device) against those traces, against the oracle on large fuzzed queues, and chained
into the device plan without a host round trip."""

import json
import os

import numpy as np
import pytest
import torch

import oracle as O
from conftest import GOLDEN


@pytest.fixture(scope="module")
def traces():
    with open(os.path.join(GOLDEN, "admit_traces.json")) as f:
        return json.load(f)


def _unpack(c):
    return [tuple(r) for r in c["queue"]], [tuple(r) for r in c["running"]]


def test_oracle_matches_reference_traces(traces):
    for c in traces:
        q, r = _unpack(c)
        batch, skips, sel = O.select_batch(q, r, c["K"], c["N"])
        assert batch == c["batch"]
        assert skips == {int(k): v for k, v in c["skips"].items()}
        assert sorted(sel) == c["selected"]


@pytest.fixture(scope="module")
def A():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2312_05215_b200 import admission
    return admission


@pytest.mark.gpu
def test_device_admission_matches_reference_traces(A, traces):
    for c in traces:
        q, r = _unpack(c)
        batch, skips, sel = A.select_batch_host(q, r, c["K"], c["N"])
        assert batch == c["batch"], c
        assert skips == {int(k): v for k, v in c["skips"].items()}
        assert sorted(sel) == c["selected"]


@pytest.mark.gpu
@pytest.mark.parametrize("Q,R,models,K,N", [(8192, 0, 4096, 300, 64), (5000, 40, 500, 2000, 7), (3000, 100, 50, 64, 50),
                                            (1000, 64, 8, 64, 4), (777, 3, 1, 1000, 1)])
def test_device_admission_fuzz_vs_oracle(A, Q, R, models, K, N):
    rng = np.random.default_rng(Q + R)
    ids = rng.permutation(Q + R) + 1
    arr = rng.integers(0, Q // 2 + 2, Q + R).astype(float)  # many ties: ordering falls back to the id
    mdl = np.minimum(rng.zipf(1.3, Q + R) - 1, models - 1)
    running = [(int(ids[k]), arr[k], int(mdl[k])) for k in range(R)]
    queue = sorted(((int(ids[k]), arr[k], int(mdl[k])) for k in range(R, Q + R)), key=lambda t: (t[1], t[0]))
    ref = O.select_batch(queue, running, K, N)
    got = A.select_batch_host(queue, running, K, N)
    assert got[0] == ref[0] and got[1] == ref[1] and got[2] == ref[2]


@pytest.mark.gpu
def test_admission_feeds_the_device_plan(A):
    """admission -> slots -> dz_plan_device on the device (no host round trip between them); the
    resulting plan equals the host plan of the same batch."""
    from paper_2312_05215_b200 import _lib as L
    from paper_2312_05215_b200.engine import DevicePlan, Plan
    rng = np.random.default_rng(4)
    Q, R, models, K, N = 200, 6, 12, 48, 5
    dev = torch.device("cuda", 0)
    q_model = torch.from_numpy(rng.integers(0, models, Q).astype(np.int32)).to(dev)
    q_id = torch.arange(100, 100 + Q, dtype=torch.int32, device=dev)
    r_model = torch.from_numpy(rng.integers(0, models, R).astype(np.int32)).to(dev)
    r_id = torch.arange(R, dtype=torch.int32, device=dev)
    adm = A.DeviceAdmission(Q, models, dev).select(q_model, q_id, torch.arange(R, R + Q, dtype=torch.int32, device=dev),
                                                   r_model, r_id, torch.arange(R, dtype=torch.int32, device=dev), K, N)
    slot_of_model = torch.arange(models, dtype=torch.int32, device=dev)  # table slot = delta id here
    slots, valid = A.batch_slots(adm, q_model, r_model, slot_of_model)
    kinds = np.full(models, L.DZ_KIND_SPARSE4, np.int32)
    # compact the valid rows on the device (order preserved), then plan them on the device
    rows = torch.nonzero(valid).flatten()
    n = int(adm.counts[0].item()) + R  # (test only: the capacity-free plan needs T)
    dp = DevicePlan(n, kinds, models, device=dev).update(slots[rows[:n]].contiguous())
    dp.check()
    host_slots = slots[rows[:n]].cpu().numpy()
    hp = Plan(host_slots, kinds, models, upload=False, pf_min=0)
    nj = int(dp.n_jobs_dev.item())
    assert nj == hp.n_jobs
    assert np.array_equal(dp.order.cpu().numpy()[:n], hp.order_host)
    assert np.array_equal(dp.jobs.cpu().numpy().view(np.int32).reshape(-1, 4)[:nj], hp.jobs_host)
