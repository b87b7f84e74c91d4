"""CPU oracle for the DeltaZip SBMM hot path — TEST INFRASTRUCTURE ONLY.

This package is the *checker*. It restates, in numpy float64, the reference
algorithm of `/root/reference/pkg/src/deltazip` for the serving hot path:
the ΔCompress codec (`compress.py:243-314`), `dequantize_layer`
(`compress.py:467-497`), `group_by_delta` / `sbmm` / `decoupled_linear`
(`inference.py:94-154`) and the tensor-parallel pair `tp_partition` /
`tp_forward` (`inference.py:162-225`).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline`
leg and `--impl reference`) may import it. The product package
`paper_2312_05215_b200` never imports, links or executes anything here.

Parity is pinned: `tests/test_oracle.py` checks this restatement against the
golden vectors in `tests/golden/` that `tests/golden/make_golden.py` produced
by importing the reference itself, plus the reference's own KATs
(`tests/test_compress.py:126-166`, `tests/test_inference.py:75-80`).
"""

from .deltazip_ref import *  # noqa: F401,F403
