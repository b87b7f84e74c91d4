"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports every symbol the
header declares, the host-only plan (group_by_delta) is right, and the host API raises the
reference's exceptions before touching the GPU."""

import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle as O
from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "dz_b200.h")


def _header_define(name):
    m = re.search(rf"#define {name} (\d+)", open(HEADER).read())
    return int(m.group(1))


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dz_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2312_05215_b200 import _lib
    return _lib.lib()


def test_library_exports_every_header_symbol(lib):
    from paper_2312_05215_b200 import _lib
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} missing from ctypes signatures"
    assert set(_lib.SIGNATURES) == set(syms)
    assert lib.dz_version().decode().startswith("dz_b200")


def test_status_strings_and_mapping(lib):
    from paper_2312_05215_b200 import _lib, errors
    for code, exc in [(1, errors.ShapeError), (2, errors.EncodingError), (3, errors.FormatError),
                      (4, errors.PartitionError), (5, errors.UnknownDeltaError), (8, errors.CudaError)]:
        with pytest.raises(exc):
            _lib.check(code)
    assert "FormatError" in lib.dz_strerror(3).decode()


def test_exception_hierarchy_matches_reference():
    from paper_2312_05215_b200 import errors as E
    assert issubclass(E.ShapeError, ValueError) and issubclass(E.ShapeError, E.DeltaZipError)
    assert issubclass(E.UnknownDeltaError, KeyError)
    assert issubclass(E.FormatError, ValueError)
    assert E.FormatError("x", offset=3).offset == 3


def _plan(lib, slots, kinds, with_base=1):
    from paper_2312_05215_b200 import _lib
    s = np.asarray(slots, dtype=np.int32)
    k = np.asarray(kinds, dtype=np.int32)
    T = s.size
    maxj = lib.dz_plan_max_jobs(T)
    order = np.zeros(max(T, 1), np.int32)
    jobs = (_lib.DzJob * max(maxj, 1))()
    nj = C.c_int32(0)
    st = lib.dz_plan(s.ctypes.data, T, k.ctypes.data, k.size, with_base, order.ctypes.data, jobs, maxj, C.byref(nj), 8)
    return st, order[:T], [(jobs[i].slot, jobs[i].tok_begin, jobs[i].tok_count, jobs[i].kind) for i in range(nj.value)]


def test_plan_is_stable_group_by_delta(lib, kat):
    st, order, jobs = _plan(lib, [2, 0, 2, 1], [1, 1, 1])
    assert st == 0
    perm = [0] * 4
    for pos, orig in enumerate(order):
        perm[orig] = pos
    assert perm == kat["group_by_delta_perm"]
    assert jobs[0] == (-1, 0, 4, 0)  # base job over all tokens
    assert [(j[0], j[1], j[2]) for j in jobs[1:]] == [(0, 0, 1), (1, 1, 1), (2, 2, 2)]
    rng = np.random.default_rng(17)
    for _ in range(50):
        ids = rng.integers(0, 5, size=int(rng.integers(0, 40))).tolist()
        st, order, jobs = _plan(lib, ids, [1, 2, 3, 1, 1])
        assert st == 0
        operm, _ = O.group_by_delta(ids)
        for orig, pos in enumerate(operm):
            assert order[pos] == orig
        covered = sorted(t for j in jobs if j[0] >= 0 for t in order[j[1]:j[1] + j[2]])
        assert covered == list(range(len(ids)))
        for j in jobs:
            if j[0] >= 0:
                assert j[2] <= (32 if j[3] == 3 else 8)
                assert all(ids[t] == j[0] for t in order[j[1]:j[1] + j[2]])


def test_plan_unknown_slot(lib):
    st, _, _ = _plan(lib, [0, 7], [1, 1])
    assert st == 5


def test_api_raises_before_compute():
    import paper_2312_05215_b200 as P
    with pytest.raises(P.UnknownDeltaError):
        P.sbmm(np.eye(4), {}, P.BatchInput([(0, 9, np.ones(4))]))
    with pytest.raises(P.ShapeError):
        P.BatchInput([(0, 0, np.ones(3)), (1, 0, np.ones(4))])
    with pytest.raises(P.PartitionError):
        P.tp_partition(np.zeros((2, 3)), "column", 2)
    with pytest.raises(P.PartitionError):
        P.TpLayout(0)
    assert P.sbmm(np.eye(4), {}, P.BatchInput([])) == {}
    shards = P.tp_partition(np.arange(8.0).reshape(4, 2), "row", 2)
    assert len(shards) == 2 and shards[0].shape == (2, 2)


def test_host_producer_codec_matches_oracle(kat):
    import paper_2312_05215_b200 as P
    assert P.pack_codes([-7, 0, 7, 1, 2, 3, -1, -2], 4).tolist() == kat["pack_spec_word"]
    assert P.pack_codes([0] * 8, 4).tolist() == kat["pack_zero_word"]
    rng = np.random.default_rng(5)
    for bits in (2, 3, 4, 8, 16):
        q = (1 << (bits - 1)) - 1
        c = rng.integers(-q, q + 1, size=101)
        assert np.array_equal(P.pack_codes(c, bits), O.pack_codes(c, bits))
    keep = np.zeros((3, 8), dtype=bool)
    for r in range(3):
        keep[r, [0, 2]] = True
        keep[r, [5, 7]] = True
    assert P.encode_mask_indices(keep) == O.encode_mask_indices(keep)
    with pytest.raises(P.EncodingError):
        P.pack_codes([8], 4)


def test_product_has_no_cpu_fallback(monkeypatch):
    """Without a CUDA device the product path must fail loudly, not compute on the CPU."""
    import torch
    import paper_2312_05215_b200 as P
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(P.CudaError):
        P.dequantize_layer(O.random_packed_delta(np.random.default_rng(0), 4, 8, 4))
    with pytest.raises(P.CudaError):
        P.sbmm(np.eye(8), {0: O.random_packed_delta(np.random.default_rng(0), 8, 8, 4)},
               P.BatchInput([(0, 0, np.ones(8))]))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2312_05215_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_plan_mixed_prefill_decode_host_logic():
    """dz_plan_mixed (host C): prefill groups staged first in 256-token jobs (remainders below
    pf_min go to decode), decode tokens after them in original order, decode jobs exactly as
    dz_plan over the staged rows, and every token covered once by one delta job."""
    from paper_2312_05215_b200.engine import Plan
    rng = np.random.default_rng(5)
    for _ in range(40):
        D = int(rng.integers(1, 7))
        counts = rng.integers(0, 700, size=D) * (rng.random(D) < 0.5)
        ids = rng.permutation(np.concatenate([np.full(int(c), d) for d, c in enumerate(counts)] + [
            rng.integers(0, D, 30)])).astype(np.int32)
        kinds = np.where(rng.random(D) < 0.15, 3, 1).astype(np.int32)
        p = Plan(ids, kinds, D, upload=False, pf_min=64)
        T = ids.size
        cnt = np.bincount(ids, minlength=D)
        J, RM = _header_define("DZ_PREFILL_JOB_TOKENS"), _header_define("DZ_PREFILL_REM_MIN")

        def n_prefill(c):  # dz_plan_mixed's rule (pf_min = 64): the group, a small remainder left to K2
            if c < 64:
                return 0
            return c - c % J if c >= J and c % J < RM else c
        npf = np.array([0 if kinds[s] == 3 else n_prefill(cnt[s]) for s in range(D)])
        assert p.t_pf == npf.sum()
        perm = p.perm_host if p.t_pf else np.arange(T)
        assert sorted(perm.tolist()) == list(range(T))
        dec = perm[p.t_pf:]
        assert np.all(np.diff(dec) > 0)  # decode tokens keep their original order
        jobs = p.jobs_host
        covered = []
        for k, (slot, b, c, kind) in enumerate(jobs):
            if k < p.n_pf_jobs:
                nj = -(-npf[slot] // J)
                assert 0 < c <= -(-(-(-npf[slot] // nj)) // 16) * 16 <= J and kind == kinds[slot] and kind != 3
                rows = perm[b:b + c]
                assert np.all(ids[rows] == slot)
                covered += rows.tolist()
            elif slot >= 0:
                rows = perm[p.order_host[b:b + c]]
                assert np.all(ids[rows] == slot) and c <= (32 if kind == 3 else _header_define("DZ_SPARSE_JOB_TOKENS"))
                covered += rows.tolist()
            else:
                assert b >= p.t_pf and c <= 128
        assert sorted(covered) == list(range(T))


def test_plain_c_host_links_the_abi(tmp_path):
    """The C ABI is usable from a plain C host (no Python, no torch): compile tests/c_host/host_demo.c
    against include/dz_b200.h, link _dz_b200.so, run the host-side entry points."""
    import shutil
    import subprocess
    from paper_2312_05215_b200 import _lib
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no C compiler")
    lib = _lib.LIB_PATH
    exe = tmp_path / "host_demo"
    src = os.path.join(ROOT, "tests", "c_host", "host_demo.c")
    r = subprocess.run([gcc, "-O1", "-std=c11", f"-I{os.path.join(ROOT, 'include')}", src, "-o", str(exe), lib,
                        f"-Wl,-rpath,{os.path.dirname(lib)}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    for case in ("dzdl_b4.dzdl", "dzdl_b4_deflate.dzdl"):
        r = subprocess.run([str(exe), os.path.join(ROOT, "tests", "golden", case)], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "all ok" in r.stdout and "layer 1: 64x128" in r.stdout


def test_obs_workspace_and_config_checks(lib):
    """dz_obs_workspace_bytes (host-only) validates the ΔCompress config like the reference's
    CompressConfig and sizes the solver's scratch; invalid configs give 0."""
    from paper_2312_05215_b200 import _lib as L
    ok = L.DzObsCfg(4, 1, 128, 32)
    n = lib.dz_obs_workspace_bytes(4096, 4096, C.byref(ok))
    # err window (rows x group) + kept codes (rows*cols/2 int32) + nibbles + loss partials
    assert n >= 4096 * 128 * 8 + 4096 * 4096 // 2 * 4 + 4096 * 4096 // 4 + 128 * 4096 * 8
    for bad in [L.DzObsCfg(5, 1, 128, 32), L.DzObsCfg(4, 1, 128, 6), L.DzObsCfg(4, 1, 0, 32),
                L.DzObsCfg(4, 1, 128, 512)]:
        assert lib.dz_obs_workspace_bytes(64, 64, C.byref(bad)) == 0
    assert lib.dz_obs_workspace_bytes(64, 66, C.byref(ok)) == 0  # 2:4 needs cols % 4 == 0


def test_obs_api_raises_before_compute():
    """obs_compress_layer checks shapes (ShapeError) before it needs a GPU."""
    import paper_2312_05215_b200 as P
    with pytest.raises(P.ShapeError):
        P.obs_compress_layer(np.zeros((4, 8)), np.eye(6), P.CompressConfig())


def test_group_by_delta_large_groups_matches_reference_rule():
    """group_by_delta is the stable sort of the reference (inference.py:106-123) at any group size:
    a group past the prefill threshold (>= 192 rows) must not turn `order` into a staged-row
    index list."""
    import paper_2312_05215_b200 as P
    import oracle as O
    rng = np.random.default_rng(5)
    for ids in ([0] * 195 + [1] * 5, list(rng.permutation([0] * 300 + [3] * 7 + [1] * 250)),
                list(rng.integers(0, 4, 1000)), [7] * 256):
        batch = P.BatchInput([(i, int(d), np.zeros(2)) for i, d in enumerate(ids)])
        perm, groups = P.group_by_delta(batch)
        rperm, rgroups = O.group_by_delta([int(d) for d in ids])
        assert perm == list(rperm) and [tuple(g) for g in groups] == [tuple(g) for g in rgroups]
