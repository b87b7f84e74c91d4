"""Peer memory for the fused tensor-parallel reduction (dz_tp.cu): one reduce buffer pair + ready
flags per rank in peer-shareable device memory, IPC handles exchanged over torch.distributed,
every peer's buffers opened in this process (NVLink / NVSwitch loads and stores).

Replaces the row-parallel all-reduce (the reference's shard-order sum, inference.py:216-223) by
a two-shot finalize kernel over peer memory (reduce-scatter of the fp32 partial sums, then an
all-gather of the reduced chunks in Y's dtype): no NCCL call on the path.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L
from .errors import CudaError

FLAG_BYTES = 512  # ready flags [2 phases][64] (int32) at the head of every rank's buffer


class PeerGroup:
    """This rank's view of the world's reduce buffers: per rank two fp32 reduce buffers R and two
    gather buffers G (capacity `max_elems` elements each, double-buffered by epoch parity)."""

    def __init__(self, rank: int, world: int, max_elems: int, device, group=None):
        import torch.distributed as dist
        if not (1 <= world <= 64) or not (0 <= rank < world):
            raise ValueError("bad rank / world")
        lib = L.lib()
        self.rank, self.world, self.max_elems, self.device = rank, world, int(max_elems), device
        nbytes = FLAG_BYTES + 4 * self.max_elems * 4  # R[2] + G[2]
        ptr = C.c_void_p()
        with torch.cuda.device(device):
            L.check(lib.dz_peer_alloc(nbytes, C.byref(ptr)), "peer alloc")
            self.local = ptr.value
            h = (C.c_uint8 * 64)()
            L.check(lib.dz_ipc_handle(C.c_void_p(self.local), h), "ipc handle")
            handles = [None] * world
            dist.all_gather_object(handles, bytes(h), group=group)
            self.opened = []
            ptrs = []
            ok = True
            for r in range(world):
                if r == rank:
                    ptrs.append(self.local)
                    continue
                hb = (C.c_uint8 * 64).from_buffer_copy(handles[r])
                p = C.c_void_p()
                if lib.dz_ipc_open(hb, C.byref(p)) != L.DZ_OK:
                    ok = False
                    break
                self.opened.append(p.value)
                ptrs.append(p.value)
            # every rank learns whether all ranks could map all peers before anyone proceeds
            flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=device)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
            if int(flag.item()) == 0:
                self.close()
                raise CudaError("CUDA IPC: a rank could not map its peers' buffers")
        self.peer_R = torch.tensor([p + FLAG_BYTES for p in ptrs], dtype=torch.int64, device=device)
        self.peer_flags = torch.tensor(ptrs, dtype=torch.int64, device=device)
        self.sync = torch.zeros(4, dtype=torch.int32, device=device)  # epoch, barrier count, generation
        self.ctx = L.DzTpCtx(self.peer_R.data_ptr(), self.peer_flags.data_ptr(), self.sync.data_ptr(),
                             self.max_elems, rank, world)
        dist.barrier(group=group)  # every rank opened every handle before any kernel signals

    def close(self) -> None:
        lib = L.lib()
        for p in self.opened:
            lib.dz_ipc_close(C.c_void_p(p))
        self.opened = []
        if self.local:
            lib.dz_peer_free(C.c_void_p(self.local))
            self.local = None
