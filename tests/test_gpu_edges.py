"""GPU: edge cases of the decode path the reference's tests reach or imply — an empty batch, a
zero-token launch, a large batch over many deltas, several base jobs (T > 128 tokens), and a
delta table with slots no token uses. Results are checked against the oracle (rel-err <= 1e-2)
and, where the contract is bit-exact, against solo launches of the same rows."""

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu
REL = 1e-2


@pytest.fixture(scope="module")
def E():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2312_05215_b200 import engine
    return engine


def _setup(E, rows, cols, D, bits, seed):
    rng = np.random.default_rng(seed)
    ods = [O.random_packed_delta(rng, rows, cols, bits) for _ in range(D)]
    table = E.DeltaTable([E.NativeDelta.from_layer_delta(o) for o in ods], rows, cols)
    W = (torch.randn(rows, cols, device="cuda") / np.sqrt(cols)).to(torch.bfloat16)
    return rng, ods, table, E.NativeBase(W), W


def _rel(Y, R):
    return float((np.linalg.norm(Y - R, axis=1) / np.linalg.norm(R, axis=1)).max())


def test_empty_batch_api():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2312_05215_b200 as P
    W = np.zeros((32, 128))
    assert P.sbmm(W, {}, P.BatchInput([])) == {}


def test_zero_token_launch(E):
    _, _, table, base, _ = _setup(E, 256, 512, 2, 4, 1)
    X = torch.empty(0, 512, dtype=torch.bfloat16, device="cuda")
    Y = E.sbmm_forward(X, E.Plan(np.zeros(0, np.int32), table.kinds, 2), base, table, y_dtype=torch.float32)
    assert Y.shape == (0, 256)


def test_large_batch_many_deltas(E):
    """T = 1024 tokens over 64 deltas (Zipf-like skew): thousands of jobs, several base jobs."""
    rng, ods, table, base, W = _setup(E, 384, 1024, 64, 4, 2)
    ids = np.minimum(rng.zipf(1.3, 1024) - 1, 63).astype(np.int32)
    X = torch.randn(1024, 1024, device="cuda").to(torch.bfloat16)
    Y = E.sbmm_forward(X, E.Plan(ids, table.kinds, 64), base, table, y_dtype=torch.float32)
    sel = rng.choice(1024, 96, replace=False)
    R = O.sbmm_matrix(W.float().double().cpu().numpy(), dict(enumerate(ods)), ids[sel],
                      X[torch.from_numpy(sel).cuda()].float().double().cpu().numpy())
    assert _rel(Y[torch.from_numpy(sel).cuda()].double().cpu().numpy(), R) <= REL


@pytest.mark.parametrize("T", [129, 300])
def test_several_base_jobs_one_delta_bit_exact(E, T):
    """All tokens on one delta of a 5-slot table (4 unused), T > 128: several base jobs and a group
    wider than a job; every row equals its solo launch bit for bit (the group stays on the decode
    kernel: pf_min=0) and the reference within tolerance."""
    rng, ods, table, base, W = _setup(E, 260, 640, 5, 2, 3 + T)
    ids = np.full(T, 3, np.int32)
    X = torch.randn(T, 640, device="cuda").to(torch.bfloat16)
    Y = E.sbmm_forward(X, E.Plan(ids, table.kinds, 5, pf_min=0), base, table, y_dtype=torch.float32)
    for i in (0, 127, 128, T - 1):
        solo = E.sbmm_forward(X[i:i + 1].contiguous(), E.Plan(ids[i:i + 1], table.kinds, 5, pf_min=0), base, table,
                              y_dtype=torch.float32)
        assert torch.equal(solo[0], Y[i]), i
    R = O.sbmm_matrix(W.float().double().cpu().numpy(), dict(enumerate(ods)), ids, X.float().double().cpu().numpy())
    assert _rel(Y.double().cpu().numpy(), R) <= REL
