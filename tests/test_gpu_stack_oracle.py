"""GPU: the Llama stack driver (stack.py) and its tensor-parallel shards checked
against the REFERENCE algorithm, not against another run of the same kernels.

For every ORIGINAL linear the stack keeps its bf16 base weight and its deltas' reference-layout
bytes (`keep_refs=True`). The reference output of a launch is rebuilt per original linear from
those: `y_t = W x_t + dequantize_layer(ΔW_{id(t)}) x_t` (inference.py:126-154), with the delta
dequantised by K1 in float64 (bit-identical to the reference's dequantize_layer, pinned by
test_gpu_parity.py) and the products in float64, then sliced and concatenated the way the
reference's tp_partition / the QKV and gate/up fusion would cut the layer (inference.py:162-243).
So a bug in concat_rows, shard_sub, tp_bounds, the mixed plan or the kernels shows up here.
A CPU oracle spot check (oracle.sbmm_matrix) anchors the float64 rebuild itself.

  (a) one 7B decoder layer at the exact bench config (D=32 4-bit 2:4, T=64, ids perm(i%32)):
      the captured-graph step of bench.py, every one of the four launches;
  (b) one 13B layer of cfg3 through the mixed plan: 8 prefill requests x 256 tokens (K3) +
      128 decode tokens (K2), 64 deltas at 2-bit;
  (c) cfg4 70B shards (16 deltas, T=64): TP8 ranks 0 and 7 (k/v shards of 128 rows) and TP2 rank 1,
      row-parallel partials against the matching column slices.
"""

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

REL = 1e-2


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2312_05215_b200 import stack
    return stack


def k1_f64(ref) -> torch.Tensor:
    """K1 (dz_unpack, DZ_F64): the reference's dequantize_layer of reference-layout device bytes."""
    from paper_2312_05215_b200 import _lib as L
    from paper_2312_05215_b200.device import ErrFlag, stream_ptr
    st, _ = ref
    out = torch.empty(st.rows, st.cols, dtype=torch.float64, device="cuda")
    err = ErrFlag(out.device)
    L.check(L.lib().dz_unpack(st, L.DZ_F64, out.data_ptr(), st.cols, err.ptr, stream_ptr()), "k1")
    err.raise_if_set("k1")
    return out


def host_delta(ref) -> "O.OracleDelta":
    """The reference LayerDelta held in the device bytes, copied to the host for the CPU oracle."""
    st, (packed, index, scales) = ref
    return O.OracleDelta(rows=st.rows, cols=st.cols,
                         packed_values=packed[: st.n_words].cpu().numpy().view("<u4").copy(),
                         index_stream=index[: st.index_bytes].cpu().numpy().tobytes(),
                         scales=scales[: st.n_scales].cpu().numpy().astype("<f4"), bits=st.bits,
                         sparsity=O.SPARSITY_2_4, group_size=st.group_size)


def ref_member(st, l, m, X64, ids, rows, cols):
    """float64 reference of one original linear's slice [rows, cols] for inputs X64 [T, cols]."""
    r0, r1 = rows
    c0, c1 = cols
    W = st.base_full[(l, m)][r0:r1, c0:c1].double()
    Y = X64 @ W.T
    for d in np.unique(ids):
        tok = torch.from_numpy(np.nonzero(ids == d)[0]).to(X64.device)
        dq = k1_f64(st.refs[(l, m, int(d))])[r0:r1, c0:c1]
        Y[tok] += X64[tok] @ dq.T
        del dq
    return Y


def ref_launch(S, st, l, fname, X, ids):
    """Reference output of one fused launch on this rank: column-parallel members are cut to the
    rank's output rows and concatenated (QKV, gate/up), row-parallel ones use the rank's input
    columns (the partial sum before the all-reduce)."""
    X64 = X.double()
    rows = {"q": st.h_b, "k": st.kv_b, "v": st.kv_b, "gate": st.i_b, "up": st.i_b}
    cols = {"o": st.h_b, "down": st.i_b}
    parts = []
    for m in S.FUSED[fname]:
        out, inp = st.shapes[m]
        parts.append(ref_member(st, l, m, X64, ids, rows.get(m, (0, out)), cols.get(m, (0, inp))))
    return torch.cat(parts, dim=1)


def rel_rows(Y, R):
    Y, R = Y.double(), R.double()
    return float((torch.linalg.norm(Y - R, dim=1) / torch.linalg.norm(R, dim=1).clamp_min(1e-30)).max())


def test_stack_7b_layer_bench_config(S):
    """(a) The bench's decode step (CUDA graph, tail-prefetch chain) on one 7B layer with D=32,
    T=64: all four launches against the reference rebuilt per original linear."""
    import bench
    from paper_2312_05215_b200.engine import Plan
    dev = torch.device("cuda", 0)
    st = S.LlamaStack("7b", 1, bench.D_DELTAS, bench.BITS, dev, keep_refs=True)
    ids = bench.token_ids()
    plan = Plan(ids, st.kinds, bench.D_DELTAS, device=dev)
    assert plan.t_pf == 0
    bufs = st.buffers(bench.T_TOKENS)
    torch.manual_seed(0)
    bufs["x"].copy_(torch.randn_like(bufs["x"], dtype=torch.float32).to(torch.bfloat16))
    st.prepare_chain(plan, bufs)
    g = torch.cuda.CUDAGraph()
    st.step(plan, bufs)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        st.step(plan, bufs)
    g.replay()
    torch.cuda.synchronize()
    src = {"qkv": bufs["x"], "o": bufs["v"], "gate_up": bufs["x"], "down": bufs["up"]}
    for f in ("qkv", "o", "gate_up", "down"):
        R = ref_launch(S, st, 0, f, src[f], ids)
        err = rel_rows(bufs[f], R)
        assert err <= REL, (f, err)
    # CPU oracle anchor: the o projection of the tokens of deltas 0 and 1
    sel = np.nonzero(ids <= 1)[0]
    W = st.base_full[(0, "o")].double().cpu().numpy()
    Xs = bufs["v"][torch.from_numpy(sel).to(dev)].double().cpu().numpy()
    Ro = O.sbmm_matrix(W, {d: host_delta(st.refs[(0, "o", d)]) for d in (0, 1)}, ids[sel], Xs)
    assert rel_rows(bufs["o"][torch.from_numpy(sel).to(dev)].cpu(), torch.from_numpy(Ro)) <= REL


def test_stack_13b_layer_cfg3_mixed_plan(S):
    """(b) cfg3 on one 13B layer: 8 x 256 prefill tokens on 8 deltas (K3, tcgen05 + 2:4 sparse
    tcgen05.mma.sp) + 128 decode tokens on 64 deltas (K2), 2-bit; every launch vs the reference."""
    from paper_2312_05215_b200.engine import Plan
    from paper_2312_05215_b200.engine import sbmm_forward
    dev = torch.device("cuda", 0)
    D = 64
    st = S.LlamaStack("13b", 1, D, 2, dev, keep_refs=True)
    pre = np.repeat(np.arange(8, dtype=np.int32), 256)
    dec = np.random.default_rng(14).permutation(np.arange(128) % D).astype(np.int32)
    ids = np.concatenate([pre, dec])
    ids = ids[np.random.default_rng(15).permutation(ids.size)]  # prefill rows interleaved with decode rows
    plan = Plan(ids, st.kinds, D, device=dev)
    assert plan.t_pf >= 8 * 240 and plan.n_pf_jobs >= 8
    torch.manual_seed(1)
    for f in ("qkv", "o", "gate_up", "down"):
        lin = st.stack[0][f]
        X = torch.randn(ids.size, lin.inp, device=dev).to(torch.bfloat16)
        Y = sbmm_forward(X, plan, lin.base, lin.table, y_dtype=torch.float32)
        R = ref_launch(S, st, 0, f, X, ids)
        err = rel_rows(Y, R)
        assert err <= REL, (f, err)


@pytest.mark.parametrize("rank,world", [(0, 8), (7, 8), (1, 2)])
def test_stack_70b_tp_shards(S, rank, world):
    """(c) cfg4 shards: this rank's column-parallel rows (q 1024, k/v 128 at TP8) and row-parallel
    input columns (o 1024, down 3584 at TP8), all four launches vs the reference slices."""
    from paper_2312_05215_b200.engine import Plan
    from paper_2312_05215_b200.engine import sbmm_forward
    dev = torch.device("cuda", 0)
    D, T = 16, 64
    st = S.LlamaStack("70b", 1, D, 4, dev, rank=rank, world=world, keep_refs=True)
    if world == 8:
        assert st.kv_b[1] - st.kv_b[0] == 128 and st.stack[0]["qkv"].out == 1024 + 2 * 128
    ids = np.random.default_rng(16).permutation(np.arange(T) % D).astype(np.int32)
    plan = Plan(ids, st.kinds, D, device=dev)
    torch.manual_seed(2)
    for f in ("qkv", "o", "gate_up", "down"):
        lin = st.stack[0][f]
        X = torch.randn(T, lin.inp, device=dev).to(torch.bfloat16)
        Y = sbmm_forward(X, plan, lin.base, lin.table, y_dtype=torch.float32)
        R = ref_launch(S, st, 0, f, X, ids)
        err = rel_rows(Y, R)
        assert err <= REL, (f, rank, world, err)
