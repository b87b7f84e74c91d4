"""GPU: decode-path (K2) merge and base K-split properties. Every output element is the fixed-order
sum of the base K-split partials and the token's delta partial (k_finalize by default, or the
fused combiner warp), so results are deterministic, independent of the batch for a given split
count, and within fp32 rounding of each other across split counts. The base stage shape depends
on the launch's token count (narrow 32-row X tile and 3 W chunks per stage at T <= 32), never on
which tokens share the batch, so a token's row is bit-identical across batch sizes."""

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


@pytest.mark.parametrize("rows,cols", [(512, 1024), (200, 1152)])
def test_base_splits_agree_and_batch_invariant(E, rows, cols):
    rng = np.random.default_rng(rows + cols)
    D, T = 5, 40
    ods = [O.random_packed_delta(rng, rows, cols, 4) for _ in range(D)]
    table = E.DeltaTable([E.NativeDelta.from_layer_delta(o) for o in ods], rows, cols)
    W = (torch.randn(rows, cols, device="cuda") / np.sqrt(cols)).to(torch.bfloat16)
    base = E.NativeBase(W)
    ids = rng.integers(0, D, T).astype(np.int32)
    X = torch.randn(T, cols, device="cuda").to(torch.bfloat16)
    plan = E.Plan(ids, table.kinds, D)
    ys = {}
    for sp in (1, 2, 3, 4):
        y = E.sbmm_forward(X, plan, base, table, y_dtype=torch.float32, base_splits=sp)
        assert torch.equal(y, E.sbmm_forward(X, plan, base, table, y_dtype=torch.float32, base_splits=sp))
        # batch invariance at a fixed split count: a 3-token sub-batch reproduces its rows bit-exactly
        sel = np.array([0, 7, T - 1])
        ysub = E.sbmm_forward(X[torch.from_numpy(sel).cuda()].contiguous(), E.Plan(ids[sel], table.kinds, D), base,
                              table, y_dtype=torch.float32, base_splits=sp)
        assert torch.equal(ysub, y[torch.from_numpy(sel).cuda()])
        ys[sp] = y
    for sp in (2, 3, 4):
        rel = (torch.linalg.norm(ys[sp] - ys[1], dim=1) / torch.linalg.norm(ys[1], dim=1)).max().item()
        assert rel < 1e-5, rel
    R = O.sbmm_matrix(W.float().double().cpu().numpy(), dict(enumerate(ods)), ids, X.float().double().cpu().numpy())
    err = np.linalg.norm(ys[4].double().cpu().numpy() - R, axis=1) / np.linalg.norm(R, axis=1)
    assert err.max() <= 1e-2


@pytest.mark.parametrize("rows,cols", [(256, 11008), (130, 2944)])
def test_narrow_base_stage_batch_invariant(E, rows, cols):
    """T <= 32 launches use the narrow base stage (UMMA N 32, 3 K-chunks per stage), larger ones the
    wide one (N 128, 2 chunks): same K-split boundaries and chunk order, so every row agrees bit
    for bit across T = 1, 32, 33, 64 at each split count, and with the reference algorithm."""
    rng = np.random.default_rng(rows * 7 + cols)
    D, T = 3, 64
    ods = [O.random_packed_delta(rng, rows, cols, 4) for _ in range(D)]
    table = E.DeltaTable([E.NativeDelta.from_layer_delta(o) for o in ods], rows, cols)
    W = (torch.randn(rows, cols, device="cuda") / np.sqrt(cols)).to(torch.bfloat16)
    base = E.NativeBase(W)
    ids = rng.integers(0, D, T).astype(np.int32)
    X = torch.randn(T, cols, device="cuda").to(torch.bfloat16)
    for sp in (1, 2, 3):
        y = E.sbmm_forward(X, E.Plan(ids, table.kinds, D), base, table, y_dtype=torch.float32, base_splits=sp)
        for n in (1, 32, 33):
            sel = np.arange(T - n, T)
            ysub = E.sbmm_forward(X[T - n:].contiguous(), E.Plan(ids[sel], table.kinds, D), base, table,
                                  y_dtype=torch.float32, base_splits=sp)
            assert torch.equal(ysub, y[T - n:]), (sp, n)
    R = O.sbmm_matrix(W.float().double().cpu().numpy(), dict(enumerate(ods)), ids, X.float().double().cpu().numpy())
    err = np.linalg.norm(y.double().cpu().numpy() - R, axis=1) / np.linalg.norm(R, axis=1)
    assert err.max() <= 1e-2


@pytest.mark.parametrize("bits", [4, 2])
def test_delta_splits_agree_and_batch_invariant(E, bits):
    rng = np.random.default_rng(77 + bits)
    rows, cols, D, T = 384, 2048, 6, 33
    ods = [O.random_packed_delta(rng, rows, cols, bits) for _ in range(D)]
    table = E.DeltaTable([E.NativeDelta.from_layer_delta(o) for o in ods], rows, cols)
    base = E.NativeBase((torch.randn(rows, cols, device="cuda") / np.sqrt(cols)).to(torch.bfloat16))
    ids = rng.integers(0, D, T).astype(np.int32)
    X = torch.randn(T, cols, device="cuda").to(torch.bfloat16)
    plan = E.Plan(ids, table.kinds, D)
    y1 = E.sbmm_forward(X, plan, base, table, y_dtype=torch.float32, delta_splits=1)
    y2 = E.sbmm_forward(X, plan, base, table, y_dtype=torch.float32, delta_splits=2, base_splits=2)
    assert torch.equal(y2, E.sbmm_forward(X, plan, base, table, y_dtype=torch.float32, delta_splits=2, base_splits=2))
    sel = np.array([1, 5, 30])
    ysub = E.sbmm_forward(X[torch.from_numpy(sel).cuda()].contiguous(), E.Plan(ids[sel], table.kinds, D), base, table,
                          y_dtype=torch.float32, delta_splits=2, base_splits=2)
    assert torch.equal(ysub, y2[torch.from_numpy(sel).cuda()])
    rel = (torch.linalg.norm(y2 - y1, dim=1) / torch.linalg.norm(y1, dim=1)).max().item()
    assert rel < 1e-5, rel


def test_slice_counters_rearm_across_shapes(E):
    """The per-slice arrival counters live in a fixed workspace region that every launch leaves at
    zero: launches of different widths, split counts and a mixed plan sharing ONE workspace keep
    producing bit-identical results, and the counter region reads back as zeros."""
    rng = np.random.default_rng(3)
    ws = E.Workspace()
    cases = []
    for rows, cols, D, T in ((4096, 512, 3, 24), (96, 384, 2, 9), (1000, 256, 4, 70), (33, 128, 2, 5)):
        ods = [O.random_packed_delta(rng, rows, cols, 4) for _ in range(D)]
        table = E.DeltaTable([E.NativeDelta.from_layer_delta(o) for o in ods], rows, cols)
        base = E.NativeBase((torch.randn(rows, cols, device="cuda") / np.sqrt(cols)).to(torch.bfloat16))
        ids = rng.integers(0, D, T).astype(np.int32)
        X = torch.randn(T, cols, device="cuda").to(torch.bfloat16)
        cases.append((X, E.Plan(ids, table.kinds, D), base, table, ods, ids))
    first = [E.sbmm_forward(X, p, b, t, y_dtype=torch.float32, workspace=ws) for X, p, b, t, _, _ in cases]
    for rep in range(3):
        for (X, p, b, t, _, _), y0 in zip(cases, first):
            for sp in (0, 3):
                y = E.sbmm_forward(X, p, b, t, y_dtype=torch.float32, workspace=ws, base_splits=sp)
                if sp == 0:
                    assert torch.equal(y, y0)
    torch.cuda.synchronize()
    buf = ws.get(1, 1, cases[0][0].device)
    assert int(buf[256: 256 + 4 * 8192].count_nonzero()) == 0
    for (X, p, b, t, ods, ids), y0 in zip(cases, first):
        W = b.W.float().double().cpu().numpy()
        R = O.sbmm_matrix(W, dict(enumerate(ods)), ids, X.float().double().cpu().numpy())
        err = (np.linalg.norm(y0.double().cpu().numpy() - R, axis=1) / np.linalg.norm(R, axis=1)).max()
        assert err <= 1e-2


@pytest.mark.parametrize("rows,cols,D,T,bits", [(4096, 512, 3, 24, 4), (1000, 256, 4, 70, 4), (33, 128, 2, 5, 2),
                                                 (640, 384, 5, 200, 4)])
def test_fused_merge_matches_finalize_launch(E, rows, cols, D, T, bits):
    """fused_merge=1 (the combiner warp writes Y inside k_sbmm, no k_finalize launch) sums the same
    planes in the same order as the default k_finalize path: bit-identical, for every base split
    count, with tanh, bf16 output, a mixed prefill plan and the on-device plan."""
    rng = np.random.default_rng(rows + T)
    ods = [O.random_packed_delta(rng, rows, cols, bits) for _ in range(D)]
    table = E.DeltaTable([E.NativeDelta.from_layer_delta(o) for o in ods], rows, cols)
    base = E.NativeBase((torch.randn(rows, cols, device="cuda") / np.sqrt(cols)).to(torch.bfloat16))
    ids = rng.integers(0, D, T).astype(np.int32)
    X = torch.randn(T, cols, device="cuda").to(torch.bfloat16)
    plans = [E.Plan(ids, table.kinds, D), E.DevicePlan(T, table.kinds, D).update(torch.from_numpy(ids).cuda())]
    if T >= 128:
        plans.append(E.Plan(ids, table.kinds, D, pf_min=32))
        assert plans[-1].t_pf > 0
    ws = E.Workspace()
    for plan in plans:
        for sp, act, yd in ((1, 0, torch.float32), (3, 1, torch.bfloat16), (2, 0, torch.bfloat16)):
            y0 = E.sbmm_forward(X, plan, base, table, y_dtype=yd, act=act, base_splits=sp, workspace=ws)
            for _ in range(2):
                y1 = E.sbmm_forward(X, plan, base, table, y_dtype=yd, act=act, base_splits=sp, workspace=ws,
                                    fused_merge=True)
                assert torch.equal(y0, y1), (type(plan).__name__, sp, act)
    buf = ws.get(1, 1, X.device)
    torch.cuda.synchronize()
    assert int(buf[256: 256 + 4 * 8192].count_nonzero()) == 0  # slice counters re-armed


@pytest.mark.parametrize("bits", [4, 2, 3])
def test_sparse_job_width_does_not_change_results(E, bits):
    """8- and 16-token 2:4 jobs (the narrow and the wide kernel instantiation, host and device plans)
    give bit-identical results: the n-tiles of a job are independent MMA columns with the same K
    order, so the plan's automatic width choice (it depends on the batch) keeps batch invariance."""
    rng = np.random.default_rng(40 + bits)
    rows, cols, D = 520, 640, 4
    ods = [O.random_packed_delta(rng, rows, cols, bits) for _ in range(D)]
    table = E.DeltaTable([E.NativeDelta.from_layer_delta(o) for o in ods], rows, cols)
    base = E.NativeBase((torch.randn(rows, cols, device="cuda") / np.sqrt(cols)).to(torch.bfloat16))
    ids = np.concatenate([np.zeros(37, np.int32), rng.integers(1, D, 21).astype(np.int32)])
    ids = ids[rng.permutation(ids.size)]
    X = torch.randn(ids.size, cols, device="cuda").to(torch.bfloat16)
    ys = [E.sbmm_forward(X, E.Plan(ids, table.kinds, D, sparse_job_tokens=w), base, table, y_dtype=torch.float32)
          for w in (8, 16)]
    dp = E.DevicePlan(ids.size, table.kinds, D, sparse_job_tokens=16).update(torch.from_numpy(ids).cuda())
    ys.append(E.sbmm_forward(X, dp, base, table, y_dtype=torch.float32))
    assert E.Plan(ids, table.kinds, D).sparse_job_tokens == 16  # a 37-token group: wide jobs
    assert torch.equal(ys[0], ys[1]) and torch.equal(ys[0], ys[2])
    # a solo row equals its row in the batch
    i = int(np.nonzero(ids == 0)[0][5])
    solo = E.sbmm_forward(X[i:i + 1].contiguous(), E.Plan(ids[i:i + 1], table.kinds, D), base, table,
                          y_dtype=torch.float32)
    assert torch.equal(solo[0], ys[1][i])
    R = O.sbmm_matrix(base.W.float().double().cpu().numpy(), dict(enumerate(ods)), ids, X.float().double().cpu().numpy())
    err = (np.linalg.norm(ys[1].double().cpu().numpy() - R, axis=1) / np.linalg.norm(R, axis=1)).max()
    assert err <= 1e-2
