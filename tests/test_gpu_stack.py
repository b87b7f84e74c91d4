"""GPU: the Llama stack driver (stack.py) and its tensor-parallel sharding. Every rank's shards
are built on this one GPU and the all-reduce of the row-parallel layers is done by summing the
rank partials, so the test checks that TP over 2/4 ranks reproduces the unsharded stack
(the reference's tp_forward contract, inference.py:180-225) within the bf16 tolerance."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

REL_TOL = 1e-2


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2312_05215_b200 import stack
    return stack


def _run_tp(S, stacks, plan, x):
    """One layer, TP over `stacks` (one per rank): column-parallel outputs stay per rank, the
    row-parallel partials are summed (the NCCL all-reduce)."""
    world = len(stacks)
    bufs = [st.buffers(x.shape[0]) for st in stacks]
    for b in bufs:
        b["x"].copy_(x)
    from paper_2312_05215_b200.engine import sbmm_forward
    for f, src in S.STEP_ORDER:
        outs = []
        for st, b in zip(stacks, bufs):
            lin = st.stack[0][f]
            X = {"h": b["x"], "v": b["v"], "up": b["up"]}[src]
            outs.append(sbmm_forward(X, plan, lin.base, lin.table, y_dtype=torch.float32))
        if f in S.ROW_PARALLEL and world > 1:
            tot = sum(o for o in outs)
            for b in bufs:
                b[f].copy_(tot.to(torch.bfloat16))
        else:
            for b, o in zip(bufs, outs):
                b[f].copy_(o.to(torch.bfloat16))
    return bufs[0]["down"].float()


@pytest.mark.parametrize("world", [2, 4])
def test_tp_shards_reproduce_unsharded_layer(S, world):
    from paper_2312_05215_b200.engine import Plan
    dev = torch.device("cuda", 0)
    D, T = 4, 24
    full = S.LlamaStack("tiny", 1, D, 4, dev)
    ranks = [S.LlamaStack("tiny", 1, D, 4, dev, rank=r, world=world) for r in range(world)]
    # shards partition the model: per-rank widths add up
    assert sum(st.stack[0]["gate_up"].out for st in ranks) == full.stack[0]["gate_up"].out
    assert sum(st.stack[0]["down"].inp for st in ranks) == full.stack[0]["down"].inp
    ids = np.random.default_rng(1).integers(0, D, T).astype(np.int32)
    plan = Plan(ids, full.kinds, D, device=dev)
    x = torch.randn(T, 1024, device=dev).to(torch.bfloat16)
    y1 = _run_tp(S, [full], plan, x)
    yn = _run_tp(S, ranks, plan, x)
    err = (torch.linalg.norm(yn - y1, dim=1) / torch.linalg.norm(y1, dim=1)).max().item()
    assert err <= REL_TOL, err


def test_stack_step_graph_and_bytes(S):
    """The decode step (4 launches per layer) under CUDA-graph capture equals the eager step
    bit-for-bit, and the algorithmic byte count follows SURVEY §8(d)."""
    from paper_2312_05215_b200.engine import Plan
    from paper_2312_05215_b200.synth import linear_algorithmic_bytes
    dev = torch.device("cuda", 0)
    D, T = 4, 16
    st = S.LlamaStack("tiny", 2, D, 4, dev)
    plan = Plan(np.arange(T) % D, st.kinds, D, device=dev)
    bufs = st.buffers(T)
    bufs["x"].copy_(torch.randn(T, 1024, device=dev).to(torch.bfloat16))
    y_eager = st.step(plan, bufs).clone()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        st.step(plan, bufs)
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        st.step(plan, bufs)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(bufs["down"], y_eager)
    # NVTX-annotated step (set_nvtx): same launches, same bits
    from paper_2312_05215_b200 import set_nvtx
    set_nvtx(True)
    try:
        assert torch.equal(st.step(plan, bufs), y_eager)
    finally:
        set_nvtx(False)
    lb = st.launch_bytes(T, D)
    assert lb["o"] == linear_algorithmic_bytes(1024, 1024, 4, D, T)
    assert lb["down"] == linear_algorithmic_bytes(1024, 1408, 4, D, T)


@pytest.mark.parametrize("T,D,layers", [(16, 4, 2), (130, 3, 2), (64, 32, 1)])
def test_chained_step_equals_launch_per_linear(S, T, D, layers):
    """dz_sbmm_chain (every linear of the step in ONE persistent launch, Y merged in-kernel, each
    linear's X waiting for the previous linear's rows) equals the step of one launch per linear
    bit for bit — eager, and replayed in a CUDA graph — for decode plans with one or two base
    jobs (T=130) and 8- or 16-token delta jobs."""
    from paper_2312_05215_b200.engine import Plan
    dev = torch.device("cuda", 0)
    st = S.LlamaStack("tiny", layers, D, 4, dev)
    ids = np.random.default_rng(T).integers(0, D, T).astype(np.int32)
    for width in (8, 16):
        plan = Plan(ids, st.kinds, D, device=dev, sparse_job_tokens=width)
        bufs = st.buffers(T)
        bufs["x"].copy_(torch.randn(T, 1024, device=dev).to(torch.bfloat16))
        x0 = bufs["x"].clone()
        y_ref = st.step(plan, bufs).clone()
        bufs["x"].copy_(x0)
        y_chain = st.step_chained(plan, bufs).clone()
        assert torch.equal(y_chain, y_ref), width
        for f in ("qkv", "o", "gate_up"):  # every intermediate buffer too (last layer's)
            assert torch.isfinite(bufs[f].float()).all()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            st.step_chained(plan, bufs)
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            st.step_chained(plan, bufs)
        for _ in range(3):
            bufs["x"].copy_(x0)
            g.replay()
        torch.cuda.synchronize()
        assert torch.equal(bufs["down"], y_ref), width
