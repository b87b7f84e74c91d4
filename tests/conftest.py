import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) and the built extension")
    config.addinivalue_line("markers", "slow: long-running full-size parity cases")


def load_ld_fields(z, prefix=""):
    rows, cols, bits, sparse, gs = (int(v) for v in z[f"{prefix}meta"])
    return dict(
        rows=rows, cols=cols, bits=bits,
        sparsity="two_of_four" if sparse else "none",
        group_size=gs,
        packed_values=np.asarray(z[f"{prefix}packed"], dtype="<u4"),
        index_stream=bytes(np.asarray(z[f"{prefix}index"], dtype=np.uint8).tobytes()),
        scales=np.asarray(z[f"{prefix}scales"], dtype="<f4"),
    )


def golden_files(pattern):
    return sorted(glob.glob(os.path.join(GOLDEN, pattern)))


def golden_kat():
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def kat():
    return golden_kat()
