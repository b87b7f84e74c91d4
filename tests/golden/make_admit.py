"""Admission traces from the REFERENCE scheduler (scheduler.select_batch, scheduler.py:73-123):
random queues and running sets (fixed seed), the reference's batch, line skips with parents and
selected deltas. Pins oracle.select_batch and the device kernel (tests/test_*admit*).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_admit.py
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from deltazip.scheduler import Request, SchedulerConfig, SchedulerState, select_batch  # noqa: E402


def main():
    rng = np.random.default_rng(2312)
    cases = []
    for c in range(300):
        n_models = int(rng.integers(1, 12))
        Q = int(rng.integers(0, 60))
        R = int(rng.integers(0, 10))
        K = int(rng.integers(1, 40))
        N = int(rng.integers(1, 6))
        st = SchedulerState()
        ids = rng.permutation(1000)[: Q + R] + 1
        arrivals = np.round(rng.random(Q + R) * 20, 1)  # ties on arrival resolved by id
        running, queue = [], []
        for k in range(R):
            r = Request(id=int(ids[k]), arrival=float(arrivals[k]), model_id=int(rng.integers(0, n_models)),
                        prompt_tokens=4, decode_tokens=8)
            st.running[r.id] = r
            running.append([r.id, r.arrival, r.model_id])
        for k in range(R, R + Q):
            r = Request(id=int(ids[k]), arrival=float(arrivals[k]), model_id=int(rng.integers(0, n_models)),
                        prompt_tokens=4, decode_tokens=8)
            st.enqueue(r)
        queue = [[r.id, r.arrival, r.model_id] for r in st.queue]
        batch, to_load = select_batch(st, SchedulerConfig(max_requests=K, max_deltas=N))
        cases.append({"K": K, "N": N, "queue": queue, "running": running,
                      "batch": [r.id for r in batch],
                      "skips": {str(r.id): r.parent_id for r in batch if r.skipped_line},
                      "selected": sorted({r.model_id for r in batch}), "to_load": sorted(to_load)})
    with open(os.path.join(HERE, "admit_traces.json"), "w") as f:
        json.dump(cases, f)
    print(len(cases), "traces;", sum(len(c["skips"]) for c in cases), "line skips")


if __name__ == "__main__":
    main()
