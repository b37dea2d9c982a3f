"""Point-split exact FPS over one process per GPU.

Every rank holds the whole cloud (N float4, 16 MB at N = 2^20) and owns the
original indices [g*ceil(N/G), (g+1)*ceil(N/G)).  Each FPS iteration every
rank reduces its shard inside one thread-block cluster and writes its
shard record (six tagged 64-bit words) into every rank's mailbox -- device
memory of the receiving GPU, mapped into the sender through CUDA IPC, written
with system-scope stores over NVLink -- then reduces the G records with the
chunk-merge rule of _kernels.fps_update_chunk / first_untaken
(/root/reference/pkg/src/pointsample/_kernels.py:77-100).  There is no NCCL
call on the data path; ``torch.distributed`` only exchanges the IPC handles
once and provides the timing barrier.

The same kernel runs all G ranks on one GPU (``engine.fps_split``), which is
how the protocol is tested on a single device.
"""

from __future__ import annotations

import ctypes
import math

import torch
import torch.distributed as dist

from . import _lib


def _p(t):
    return 0 if t is None else t.data_ptr()


class PointSplitFPS:
    """Per-rank state of a point-split FPS over the default process group.

    ``B`` clouds of ``N`` points; call ``run(xyz4, n)`` collectively on all
    ranks.  Results (idx, curve) are identical on every rank."""

    def __init__(self, B: int, N: int, group=None, device=None):
        self.B, self.N = int(B), int(N)
        self.group = group
        self.G = dist.get_world_size(group)
        self.g = dist.get_rank(group)
        if self.G > 32:
            raise ValueError("the point split exchanges one warp lane per rank: at most 32 ranks")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        # every peer GPU must be reachable with peer stores (NVLink / P2P);
        # ranks sharing a GPU (tests) need nothing
        devs = [None] * self.G
        dist.all_gather_object(devs, self.device.index, group=group)
        for r, d in enumerate(devs):
            if r != self.g and d != self.device.index and not torch.cuda.can_device_access_peer(self.device, d):
                raise RuntimeError(f"rank {self.g}: GPU {self.device.index} cannot access peer GPU {d} "
                                   "(the point split needs P2P / NVLink between all ranks)")
        nbytes = int(_lib.raw("ps_fps_mailbox_bytes", self.B, self.G))
        # a dedicated cudaMalloc allocation: an IPC handle opens at the base of
        # the allocation it names, which a caching-allocator tensor is not
        box = ctypes.c_void_p()
        _lib.call("ps_device_alloc", nbytes, 0xFF, ctypes.byref(box))
        self.box_ptr = box.value
        handle = ctypes.create_string_buffer(64)
        _lib.call("ps_ipc_handle", self.box_ptr, handle)
        handles = [None] * self.G
        dist.all_gather_object(handles, bytes(handle.raw), group=group)
        self._opened = []
        ptrs = []
        for r, h in enumerate(handles):
            if r == self.g:
                ptrs.append(self.box_ptr)
                continue
            out = ctypes.c_void_p()
            _lib.call("ps_ipc_open", ctypes.create_string_buffer(h, 64), ctypes.byref(out))
            self._opened.append(out.value)
            ptrs.append(out.value)
        self.ptrs = torch.tensor(ptrs, dtype=torch.int64, device=self.device)
        self.seq = 0
        dist.barrier(group=group)

    def close(self):
        """Collective: wait for this rank's launches (they write the peers'
        mailboxes), unmap the peers' mailboxes, then -- after every rank did
        the same -- free this rank's."""
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        for p in self._opened:
            _lib.call("ps_ipc_close", p)
        self._opened = []
        dist.barrier(group=self.group)
        if self.box_ptr:
            _lib.call("ps_device_free", self.box_ptr)
            self.box_ptr = 0

    def run(self, xyz4: torch.Tensor, n: int, seed_index: int = 0, k_stop: int | None = None):
        """Collective exact FPS of every cloud; returns (idx, curve, md, taken)
        with md / taken valid on this rank's shard."""
        B, N, _ = xyz4.shape
        if (B, N) != (self.B, self.N):
            raise ValueError(f"expected clouds of shape ({self.B}, {self.N}), got ({B}, {N})")
        stop = n if k_stop is None else int(k_stop)
        if self.seq + stop + 1 >= 0xFFFFFFFF:
            raise RuntimeError("mailbox sequence space exhausted; build a new PointSplitFPS")
        md = torch.empty(B, N, dtype=torch.float64, device=self.device)
        taken = torch.empty(B, N, dtype=torch.uint8, device=self.device)
        out = torch.full((B, n), -1, dtype=torch.int64, device=self.device)
        curve = torch.full((B, n), math.inf, dtype=torch.float64, device=self.device)
        _lib.call("ps_fps_split", _p(xyz4), B, N, _p(md), _p(taken), _p(out), _p(curve), n, stop, int(seed_index),
                  self.G, self.g, 1, _p(self.ptrs), self.seq, 1, torch.cuda.current_stream().cuda_stream)
        self.seq += stop + 1
        return out, curve, md, taken


def shard_range(N: int, G: int, g: int) -> tuple[int, int]:
    """Original-index range [lo, hi) owned by rank g (the kernel's partition)."""
    Ns = (N + G - 1) // G
    lo = min(N, g * Ns)
    return lo, min(N, lo + Ns)
