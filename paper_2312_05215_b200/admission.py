"""On-device admission: scheduler.select_batch's decision (scheduler.py:73-123)
on the GPU, feeding the device plan without a host round trip.

`DeviceAdmission.select(...)` enqueues one CTA (dz_admit_device) over device tensors describing
the arrival-ordered queue and the running requests; the outputs stay on the device. A serving
loop turns the admitted requests into token slots on the device (`batch_slots`) and plans them
with `engine.DevicePlan.update`. `select_batch_host` runs the same kernel on host lists and
returns the reference's result shape (batch ids, line skips with parents, deltas to load) for
tests and for callers that keep their queue on the host.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .device import require_cuda, stream_ptr


class DeviceAdmission:
    """Output buffers of one admission call (reused across calls of the same capacity)."""

    def __init__(self, max_queue: int, n_models: int, device=None):
        dev = device or require_cuda()
        self.device, self.max_queue, self.n_models = dev, int(max_queue), int(n_models)
        q = max(1, self.max_queue)
        self.admitted = torch.zeros(q, dtype=torch.uint8, device=dev)
        self.skipped = torch.zeros(q, dtype=torch.uint8, device=dev)
        self.parent = torch.full((q,), -1, dtype=torch.int32, device=dev)
        self.selected = torch.zeros(self.n_models, dtype=torch.uint8, device=dev)
        self.counts = torch.zeros(2, dtype=torch.int32, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)

    def select(self, q_model, q_id, q_rank, r_model, r_id, r_rank, K: int, N: int) -> "DeviceAdmission":
        """All inputs int32 CUDA tensors; the queue in (arrival, id) order. Stream-ordered."""
        Q, R = int(q_model.numel()), int(r_model.numel())
        if Q > self.max_queue:
            raise ValueError(f"queue of {Q} > capacity {self.max_queue}")
        for t in (q_model, q_id, q_rank, r_model, r_id, r_rank):
            if t.dtype != torch.int32 or not t.is_cuda:
                raise ValueError("admission inputs must be int32 CUDA tensors")
        ptr = lambda t: t.data_ptr() if t.numel() else None  # noqa: E731
        L.check(L.lib().dz_admit_device(ptr(q_model), ptr(q_id), ptr(q_rank), Q, ptr(r_model), ptr(r_id),
                                        ptr(r_rank), R, self.n_models, int(K), int(N), self.admitted.data_ptr(),
                                        self.skipped.data_ptr(), self.parent.data_ptr(), self.selected.data_ptr(),
                                        self.counts.data_ptr(), self.err.data_ptr(), stream_ptr()), "admission")
        self.Q = Q
        return self

    def check(self) -> None:
        L.check(int(self.err.item()), "admission: delta id out of range")


def batch_slots(adm: DeviceAdmission, q_model: torch.Tensor, r_model: torch.Tensor, slot_of_model: torch.Tensor):
    """Device delta-table slots of the batch rows: the running requests, then the admitted queue
    requests in queue order (no host sync; the row count is the capacity R + Q, padded rows get
    slot -1 and a validity mask)."""
    adm_mask = adm.admitted[: adm.Q].bool()
    rows_model = torch.cat([r_model, torch.where(adm_mask, q_model, torch.full_like(q_model, -1))])
    valid = torch.cat([torch.ones_like(r_model, dtype=torch.bool), adm_mask])
    slots = torch.where(valid, slot_of_model[rows_model.clamp_min(0).long()], torch.full_like(rows_model, -1))
    return slots, valid


def select_batch_host(queue, running, K: int, N: int, device=None):
    """select_batch on host records: queue / running = lists of (request id, arrival, model id),
    the queue in (arrival, id) order as SchedulerState keeps it. Returns (batch ids in the
    reference's batch order, {id: parent id} of the line skips, set of selected deltas)."""
    dev = device or require_cuda()
    allr = sorted([(a, i) for i, a, _ in queue] + [(a, i) for i, a, _ in running])
    rank = {i: k for k, (_, i) in enumerate(allr)}
    models = [m for _, _, m in queue] + [m for _, _, m in running]
    n_models = max(models) + 1 if models else 1
    t = lambda v: torch.tensor(np.asarray(v, dtype=np.int32), device=dev)  # noqa: E731
    adm = DeviceAdmission(max(1, len(queue)), n_models, dev)
    adm.select(t([m for _, _, m in queue]), t([i for i, _, _ in queue]), t([rank[i] for i, _, _ in queue]),
               t([m for _, _, m in running]), t([i for i, _, _ in running]), t([rank[i] for i, _, _ in running]), K, N)
    adm.check()
    a = adm.admitted[: len(queue)].cpu().numpy()
    s = adm.skipped[: len(queue)].cpu().numpy()
    p = adm.parent[: len(queue)].cpu().numpy()
    sel = set(np.nonzero(adm.selected.cpu().numpy())[0].tolist())
    run_sorted = [i for (_, i) in sorted((a_, i) for i, a_, _ in running)]
    batch = run_sorted + [queue[k][0] for k in range(len(queue)) if a[k]]
    skips = {queue[k][0]: int(p[k]) for k in range(len(queue)) if s[k]}
    return batch, skips, sel
