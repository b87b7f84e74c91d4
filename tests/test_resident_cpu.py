"""Residency cache of the drop-in API (resident.py): hits on the same objects, misses on any
replaced array / field / configuration or an edited sampled element, entries dropped with the
object. Host-only logic (the build callback stands in for the device upload)."""

import gc

import numpy as np

from paper_2312_05215_b200 import resident as R
from paper_2312_05215_b200.compress import LayerDelta


def _ld(rng, rows=16, cols=256):
    return LayerDelta(name="l", rows=rows, cols=cols, packed_values=rng.integers(0, 2**32, rows * cols // 16, dtype=np.uint64).astype("<u4"),
                      index_stream=bytes(rng.integers(0, 256, rows * cols // 8, dtype=np.uint8)),
                      scales=rng.random(rows * (cols // 128)).astype("<f4"), bits=4, sparsity="two_of_four", group_size=128)


def test_hits_and_invalidation_rules():
    rng = np.random.default_rng(0)
    c = R.ResidentCache()
    builds = []
    w = rng.normal(size=(300, 200))
    get = lambda o: c.get(o, R._array_sig, lambda: builds.append(1) or len(builds))  # noqa: E731
    assert get(w) == 1 and get(w) == 1 and len(builds) == 1
    w[0, 0] += 1.0  # first row is always fingerprinted
    assert get(w) == 2
    w[150, 100] += 1.0  # an unsampled interior element: documented limitation -> invalidate()
    c.invalidate(w)
    assert get(w) == 3
    v = w.copy()
    assert get(v) == 4  # another object
    ld = _ld(rng)
    getd = lambda o: c.get(o, R.delta_sig, lambda: builds.append(1) or len(builds))  # noqa: E731
    assert getd(ld) == getd(ld) == 5
    ld.scales = ld.scales.copy()  # field replaced
    assert getd(ld) == 6
    ld.bits = 2  # configuration changed
    assert getd(ld) == 7
    ld.packed_values[0] ^= 1  # sampled element (index 0) edited in place
    assert getd(ld) == 8
    n = len(c)
    del w, v, ld
    gc.collect()
    assert len(c) == n - 3  # entries follow their objects' lifetime


def test_disabled_cache_always_builds():
    c = R.ResidentCache()
    c.enabled = False
    a = np.zeros((4, 4))
    calls = []
    for _ in range(3):
        c.get(a, R._array_sig, lambda: calls.append(1))
    assert len(calls) == 3 and len(c) == 0


def test_nvtx_ranges_toggle():
    """NVTX annotation is opt-in (set_nvtx) and balanced push/pop works without a GPU."""
    import paper_2312_05215_b200 as P
    from paper_2312_05215_b200 import device
    assert device._NVTX[0] is False
    P.set_nvtx(True)
    try:
        device.nvtx_push("dz test")
        device.nvtx_pop()
    finally:
        P.set_nvtx(False)
    assert device._NVTX[0] is False
