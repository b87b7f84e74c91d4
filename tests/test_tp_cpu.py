"""Host logic of the multi-GPU path on CPU: the tensor-parallel partition of the Llama stack
(stack.tp_bounds / split_units) and a world-size-2 gloo run of the column/row-parallel layer
pair whose all-reduce reproduces the unsharded layer (§5.3, inference.py:180-225).
The arithmetic here is the CPU oracle (the checker); the product path needs a GPU."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2312_05215_b200.stack import split_units, tp_bounds
from paper_2312_05215_b200.synth import llama_linears


@pytest.mark.parametrize("n,world,unit", [(11008, 1, 128), (11008, 2, 128), (11008, 4, 128), (11008, 8, 128),
                                          (4096, 8, 128), (1024, 8, 128), (28672, 8, 128), (13824, 8, 128),
                                          (1408, 4, 128), (1000, 3, 16)])
def test_split_units_partition(n, world, unit):
    b = split_units(n, world, unit)
    assert b[0][0] == 0 and b[-1][1] == n and len(b) == world
    for (s0, e0), (s1, _) in zip(b, b[1:]):
        assert e0 == s1
    sizes = [e - s for s, e in b]
    for s, e in b[:-1]:
        assert (e - s) % unit == 0 and s % unit == 0
    assert max(sizes) - min(sizes) <= unit
    assert min(sizes) > 0


def test_split_units_too_many_parts():
    with pytest.raises(ValueError):
        split_units(256, 4, 128)


@pytest.mark.parametrize("model", ["7b", "13b", "70b"])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_tp_bounds_native_aligned(model, world):
    """Every shard of every linear is a sub-grid of native 16x128 blocks (no dequantisation)."""
    shapes = {n: (o, i) for n, o, i in llama_linears(model)}
    parts = [tp_bounds(model, r, world) for r in range(world)]
    for dim, k in (("hid", 0), ("kv", 1), ("inter", 2)):
        full = {"hid": shapes["q"][1], "kv": shapes["k"][0], "inter": shapes["gate"][0]}[dim]
        assert parts[0][k][0] == 0 and parts[-1][k][1] == full
        for p in parts:
            s, e = p[k]
            assert s % 128 == 0 and (e % 128 == 0 or e == full) and e > s


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)  # identical model on every rank
    shapes = {n: (o, i) for n, o, i in llama_linears("tiny")}
    hid, inter = shapes["gate"][1], shapes["gate"][0]
    Wg = rng.normal(0, 1 / np.sqrt(hid), (inter, hid))
    Wd = rng.normal(0, 1 / np.sqrt(inter), (hid, inter))
    dg = O.dequantize_layer(O.random_packed_delta(rng, inter, hid, 4))
    dd = O.dequantize_layer(O.random_packed_delta(rng, hid, inter, 4))
    x = rng.normal(0, 1, (3, hid))
    _, _, (i0, i1) = tp_bounds("tiny", rank, world)
    # column-parallel gate (this rank's intermediate rows), then row-parallel down on that slice
    h = x @ (Wg[i0:i1] + dg[i0:i1]).T
    part = h @ (Wd[:, i0:i1] + dd[:, i0:i1]).T
    t = torch.from_numpy(part)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    full = (x @ (Wg + dg).T) @ (Wd + dd).T
    q.put((rank, float(np.abs(t.numpy() - full).max() / np.abs(full).max()), i0, i1))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_column_row_pair_allreduce(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(err < 1e-12 for _, err, _, _ in res)
    assert res[0][2] == 0 and res[-1][3] == 1408 and res[0][3] == res[1][2]
