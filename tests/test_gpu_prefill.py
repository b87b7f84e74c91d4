"""GPU parity of the prefill path (K3: tcgen05 base + dequantised-delta MMAs into one TMEM tile)
and of mixed prefill + decode batches (K3 + K2 in one dz_sbmm call), against the CPU oracle
(the reference's sbmm, inference.py:126-154) and a torch fp32 reference built from the
bit-exact K1 unpack. Tolerance: rel-err <= 1e-2 per token (north star)."""

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

REL_TOL = 1e-2


@pytest.fixture(scope="module")
def E():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2312_05215_b200 import engine
    return engine


def bf16_round(a):
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().double().numpy()


def rel_err_rows(Y, R):
    return np.linalg.norm(Y - R, axis=-1) / np.maximum(np.linalg.norm(R, axis=-1), 1e-30)


def _setup(E, rng, rows, cols, bits_list):
    W = bf16_round(rng.normal(0, 1 / np.sqrt(cols), (rows, cols)))
    ods = [O.random_packed_delta(rng, rows, cols, b) for b in bits_list]
    nat = [E.NativeDelta.from_layer_delta(o) for o in ods]
    table = E.DeltaTable(nat, rows, cols)
    base = E.NativeBase(torch.from_numpy(W.astype(np.float32)).cuda().to(torch.bfloat16))
    return W, ods, table, base


def _ids(rng, counts):
    ids = np.concatenate([np.full(c, d, np.int32) for d, c in enumerate(counts)])
    return rng.permutation(ids).astype(np.int32)


@pytest.mark.parametrize("rows,cols,bits", [(256, 512, 4), (300, 448, 4), (136, 520, 2), (128, 1024, 3),
                                            (384, 256, 2)])
def test_prefill_vs_oracle(E, rows, cols, bits):
    rng = np.random.default_rng(rows * 7 + cols + bits)
    counts = [300, 150, 40, 2, 1]  # two prefill groups (300 -> 2 jobs), the rest decode
    W, ods, table, base = _setup(E, rng, rows, cols, [bits] * len(counts))
    ids = _ids(rng, counts)
    X = bf16_round(rng.normal(0, 1, (ids.size, cols)))
    Xd = torch.from_numpy(X.astype(np.float32)).cuda().to(torch.bfloat16)
    plan = E.Plan(ids, table.kinds, len(counts), pf_min=64)
    assert plan.n_pf_jobs == 3 and plan.t_pf == 450  # 300 -> 240 + 60-token remainder job; 150 -> one job
    Y = E.sbmm_forward(Xd, plan, base, table, y_dtype=torch.float32)
    R = O.sbmm_matrix(W, dict(enumerate(ods)), ids, X)
    err = rel_err_rows(Y.cpu().double().numpy(), R)
    assert err.max() <= REL_TOL, err.max()
    # the decode-only plan of the same batch agrees within tolerance (different instruction paths)
    Yd = E.sbmm_forward(Xd, E.Plan(ids, table.kinds, len(counts), pf_min=0), base, table, y_dtype=torch.float32)
    assert rel_err_rows(Y.cpu().double().numpy(), Yd.cpu().double().numpy()).max() <= 5e-3


def test_prefill_only_no_base_and_tanh(E):
    rng = np.random.default_rng(5)
    rows, cols = 192, 384
    W, ods, table, base = _setup(E, rng, rows, cols, [4, 2])
    ids = _ids(rng, [200, 70])
    X = bf16_round(rng.normal(0, 1, (ids.size, cols)))
    Xd = torch.from_numpy(X.astype(np.float32)).cuda().to(torch.bfloat16)
    plan = E.Plan(ids, table.kinds, 2, with_base=False, pf_min=32)
    assert plan.t_pf == ids.size and plan.n_pf_jobs == 2
    Y = E.sbmm_forward(Xd, plan, None, table, y_dtype=torch.float32).cpu().double().numpy()
    R = O.sbmm_matrix(np.zeros_like(W), dict(enumerate(ods)), ids, X)
    assert rel_err_rows(Y, R).max() <= REL_TOL
    plan = E.Plan(ids, table.kinds, 2, pf_min=32)
    Y = E.sbmm_forward(Xd, plan, base, table, y_dtype=torch.float32, act=1).cpu().double().numpy()
    R = np.tanh(O.sbmm_matrix(W, dict(enumerate(ods)), ids, X))
    assert rel_err_rows(Y, R).max() <= REL_TOL


def test_prefill_bf16_output_and_dense_groups_stay_on_decode(E):
    """Dense-kind deltas (8-bit here) never become prefill jobs; bf16 output path."""
    rng = np.random.default_rng(11)
    rows, cols = 160, 384
    W, ods, table, base = _setup(E, rng, rows, cols, [4, 8])
    ids = _ids(rng, [150, 150])
    X = bf16_round(rng.normal(0, 1, (ids.size, cols)))
    Xd = torch.from_numpy(X.astype(np.float32)).cuda().to(torch.bfloat16)
    plan = E.Plan(ids, table.kinds, 2, pf_min=64)
    assert plan.n_pf_jobs == 1 and plan.t_pf == 150
    Y = E.sbmm_forward(Xd, plan, base, table).float().cpu().double().numpy()
    R = O.sbmm_matrix(W, dict(enumerate(ods)), ids, X)
    assert rel_err_rows(Y, R).max() <= REL_TOL


def test_prefill_deterministic_and_grid_invariant(E):
    rng = np.random.default_rng(3)
    rows, cols = 512, 1024
    W, ods, table, base = _setup(E, rng, rows, cols, [4] * 4)
    ids = _ids(rng, [256, 256, 100, 8])
    Xd = torch.randn(ids.size, cols, device="cuda").to(torch.bfloat16)
    plan = E.Plan(ids, table.kinds, 4, pf_min=64)
    Y0 = E.sbmm_forward(Xd, plan, base, table).clone()
    for grid in (0, 1, 5, 200):
        for _ in range(3):
            assert torch.equal(E.sbmm_forward(Xd, plan, base, table, grid=grid), Y0)


def test_prefill_batch_invariant_within_regime(E):
    """A prefill token's result does not depend on the other groups in the call (bit-exact), as
    long as its group stays on the prefill path (test_inference.py:233-245 property)."""
    rng = np.random.default_rng(8)
    rows, cols = 256, 512
    W, ods, table, base = _setup(E, rng, rows, cols, [4, 4, 2])
    ids = _ids(rng, [130, 90, 5])
    Xd = torch.randn(ids.size, cols, device="cuda").to(torch.bfloat16)
    Y = E.sbmm_forward(Xd, E.Plan(ids, table.kinds, 3, pf_min=64), base, table)
    sel = np.nonzero(ids == 0)[0]
    Ys = E.sbmm_forward(Xd[torch.from_numpy(sel).cuda()].contiguous(), E.Plan(ids[sel], table.kinds, 3, pf_min=64),
                        base, table)
    assert torch.equal(Y[torch.from_numpy(sel).cuda()], Ys)


@pytest.mark.slow
@pytest.mark.parametrize("out_f,in_f,bits", [(5120, 5120, 2), (13824, 5120, 2), (5120, 13824, 2), (4096, 4096, 4)])
def test_prefill_full_size(E, out_f, in_f, bits):
    """BASELINE cfg3 shapes (13B, 2-bit): 2 prefill groups of 256 tokens + 16 decode tokens vs an
    fp32 torch reference from the bit-exact K1 unpack."""
    from paper_2312_05215_b200.compress import dequantize_layer_device
    rng = np.random.default_rng(out_f + in_f)
    D = 4
    ods = [O.random_packed_delta(rng, out_f, in_f, bits) for _ in range(D)]
    table = E.DeltaTable([E.NativeDelta.from_layer_delta(o) for o in ods], out_f, in_f)
    Wt = (torch.randn(out_f, in_f, device="cuda") / np.sqrt(in_f)).to(torch.bfloat16)
    base = E.NativeBase(Wt)
    ids = _ids(rng, [256, 256, 8, 8])
    X = torch.randn(ids.size, in_f, device="cuda").to(torch.bfloat16)
    plan = E.Plan(ids, table.kinds, D, pf_min=64)
    assert plan.n_pf_jobs == 2 and plan.t_pf == 512  # each 256-token group: one job
    Y = E.sbmm_forward(X, plan, base, table, y_dtype=torch.float32)
    R = X.float() @ Wt.float().T
    for d in range(D):
        sel = torch.from_numpy(np.nonzero(ids == d)[0]).cuda()
        R[sel] += X[sel].float() @ dequantize_layer_device(ods[d], torch.float32).T
    err = (torch.linalg.norm(Y - R, dim=1) / torch.linalg.norm(R, dim=1)).max().item()
    assert err <= REL_TOL, err


def test_prefill_strided_input_view(E):
    """X as a column slice of a wider activation (the stack's o / down inputs): the staged copy
    must use its own compact row stride."""
    rng = np.random.default_rng(17)
    rows, cols = 256, 512
    W, ods, table, base = _setup(E, rng, rows, cols, [4, 4, 4])
    ids = _ids(rng, [160, 3, 2])
    X = bf16_round(rng.normal(0, 1, (ids.size, cols)))
    wide = torch.zeros(ids.size, 3 * cols, dtype=torch.bfloat16, device="cuda")
    wide[:, cols:2 * cols] = torch.from_numpy(X.astype(np.float32)).cuda().to(torch.bfloat16)
    Xv = wide[:, cols:2 * cols]
    assert Xv.stride(0) == 3 * cols
    plan = E.Plan(ids, table.kinds, 3, pf_min=64)
    assert plan.t_pf == 160
    Y = E.sbmm_forward(Xv, plan, base, table, y_dtype=torch.float32).cpu().double().numpy()
    R = O.sbmm_matrix(W, dict(enumerate(ods)), ids, X)
    assert rel_err_rows(Y, R).max() <= REL_TOL


@pytest.mark.parametrize("rows,cols,bits", [(640, 512, 4), (300, 448, 2)])
def test_prefill_item_height_does_not_change_results(E, rows, cols, bits, monkeypatch):
    """K3 items of 128 rows (MT=1) and 256 rows (MT=2, two M tiles sharing each X tile) issue the
    same MMA sequence per output element: bit-identical results, both within tolerance."""
    rng = np.random.default_rng(rows + bits)
    W, ods, table, base = _setup(E, rng, rows, cols, [bits] * 3)
    ids = _ids(rng, [256, 140, 9])
    X = bf16_round(rng.normal(0, 1, (ids.size, cols)))
    Xd = torch.from_numpy(X.astype(np.float32)).cuda().to(torch.bfloat16)
    plan = E.Plan(ids, table.kinds, 3, pf_min=64)
    ys = []
    for mt in (1, 2):  # both heights on the dense-dequantised delta product
        ys.append(E.sbmm_forward(Xd, plan, base, table, y_dtype=torch.float32, prefill_variant=mt))
    assert torch.equal(ys[0], ys[1])
    R = O.sbmm_matrix(W, dict(enumerate(ods)), ids, X)
    assert rel_err_rows(ys[1].cpu().double().numpy(), R).max() <= REL_TOL


@pytest.mark.parametrize("rows,cols,bits", [(640, 512, 4), (300, 448, 2), (136, 520, 3)])
def test_prefill_sparse_tcgen05_vs_dense(E, rows, cols, bits, monkeypatch):
    """The default 2:4-sparse tcgen05 delta product (compressed kept values in shared memory, index
    nibbles as TMEM metadata) against the dense-dequantised variant and the oracle."""
    rng = np.random.default_rng(rows + 3 * bits)
    W, ods, table, base = _setup(E, rng, rows, cols, [bits] * 3)
    ids = _ids(rng, [256, 200, 9])
    X = bf16_round(rng.normal(0, 1, (ids.size, cols)))
    Xd = torch.from_numpy(X.astype(np.float32)).cuda().to(torch.bfloat16)
    plan = E.Plan(ids, table.kinds, 3, pf_min=64)
    ys = {}
    for sp, variant in (("1", 0), ("0", 1)):
        ys[sp] = E.sbmm_forward(Xd, plan, base, table, y_dtype=torch.float32,
                                prefill_variant=variant).cpu().double().numpy()
    R = O.sbmm_matrix(W, dict(enumerate(ods)), ids, X)
    assert rel_err_rows(ys["1"], R).max() <= REL_TOL
    assert rel_err_rows(ys["1"], ys["0"]).max() <= 1e-4  # same bf16 ΔW values, fp32 sums in another order
