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


class PointSplitFastPoint:
    """FastPoint (MDPS) of one huge cloud over one process per GPU -- config
    C5's MDPS.  Every rank holds the cloud; rank g owns the
    points of shard_range(N, G, g) and the exclusion rows of those points.

      prefix      point-split FPS of k0 samples (mailboxes, as PointSplitFPS)
      thresholds  every rank (the replicated prefix curve -> identical radii)
      exclusion   rank g builds its rows (ps_excl_build_shard) with spill
                  sub-arena g; the row index entries, counts and row offsets
                  go to rank 0 (point-to-point; d2 stays where it was built)
      sampler     rank 0 over all rows; indices, reached, entered, exhausted
                  and RNG state broadcast
      early term  rank g seeds md of its points from its own rows
                  (ps_early_termination_shard), then the point-split FPS tail
                  (ps_fps_split_loop)
      grouping    rank g answers the sampled centroids it owns from its
                  rows; the disjoint answers are summed (all-reduce)

    Collectives go through torch.distributed (NCCL on GPUs; gloo stages
    through host memory, which is what the one-GPU tests use)."""

    def __init__(self, N: int, n: int, *, exponent: float, p: float = 0.1, nseg: int = 6, extra_radii=(),
                 seed_index: int = 0, group=None, device=None, cap_entries=None):
        from . import engine

        self.split = PointSplitFPS(1, N, group=group, device=device)
        self.group, self.G, self.g, self.device = group, self.split.G, self.split.g, self.split.device
        self.fp = engine.FastPoint(1, N, n, p=p, nseg=nseg, estimator="power", exponent=exponent,
                                   extra_radii=extra_radii, seed_index=seed_index, cap_entries=cap_entries,
                                   device=self.device)
        self.N, self.n = int(N), int(n)
        self.lo, self.hi = shard_range(self.N, self.G, self.g)
        self.ranges = [shard_range(self.N, self.G, r) for r in range(self.G)]
        ws = int(_lib.raw("ps_excl_workspace_bytes", 1, self.N, 1, 2))
        self.ws = torch.empty(ws, dtype=torch.int8, device=self.device).view(torch.uint8)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.gloo = dist.get_backend(group) == "gloo"

    # -- collectives (device tensors; gloo stages through host memory) --------
    def _bcast(self, t):
        if self.gloo:
            h = t.cpu()
            dist.broadcast(h, src=0, group=self.group)
            t.copy_(h)
        else:
            dist.broadcast(t, src=0, group=self.group)

    def _allreduce(self, t, op):
        if self.gloo:
            h = t.cpu()
            dist.all_reduce(h, op=op, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=op, group=self.group)

    def _spill(self, r):
        c = self.fp.csr
        spill = c.cap_entries - self.N * c.stride
        per = (spill // self.G) & ~3
        return r * per, ((r + 1) * per if r < self.G - 1 else spill)

    def run(self, xyz4, rng_seed: int = 0, k: int = 32, radius=None):
        """Collective MDPS of the cloud xyz4 [1, N, 4] -> (indices int64[n],
        rf groups (idx [n, k], dist, cnt) when ``radius`` is baked in)."""
        fp, N, n = self.fp, self.N, self.n
        st = torch.cuda.current_stream(self.device).cuda_stream
        fp.xyz4.copy_(xyz4)
        fp.set_rng([rng_seed])
        # 1. prefix: point-split FPS, every rank writes out/curve
        s = self.split
        if s.seq + n + fp.k0 + 2 >= 0xFFFFFFFF:
            raise RuntimeError("mailbox sequence space exhausted; build a new PointSplitFastPoint")
        _lib.call("ps_fps_split", _p(fp.xyz4), 1, N, _p(fp.md), _p(fp.taken), _p(fp.out), _p(fp.curve), n, fp.k0,
                  fp.seed_index, self.G, self.g, 1, _p(s.ptrs), s.seq, 1, st)
        s.seq += fp.k0 + 1
        # 2. thresholds (replicated)
        fp._thresholds()
        # 3. row-sharded exclusion build (every rank grows the capacity and
        # rebuilds while any rank's spill arena overflows), rows to rank 0
        from .engine import DeviceCsr

        for _ in range(8):
            c = fp.csr
            sl, sh = self._spill(self.g)
            _lib.call("ps_excl_build_shard", _p(fp.xyz4), 1, N, _p(c.levels), fp.L, c.levels.shape[1], self.lo,
                      self.hi, sl, sh, _p(c.indptr), _p(c.nbr), _p(c.d2), _p(c.counts), c.cap_entries, _p(self.ws),
                      _p(self.status), st)
            self._allreduce(self.status, dist.ReduceOp.MAX)
            if int(self.status.item()) == 0:
                break
            full = min(N * (N + 1) + 16 * N, (1 << 31) - 1)
            if c.cap_entries >= full:
                raise RuntimeError("exclusion lists overflow at the largest capacity")
            grow = min(2 * c.cap_entries, full)
            levels = c.levels.clone()
            fp.csr = DeviceCsr.allocate(1, N, fp.L, grow, grow // 2 + 1, self.device, 2)
            fp.csr.levels.copy_(levels)
        c = fp.csr
        c.status.copy_(self.status)
        stride = c.stride

        def pieces(r):
            lo, hi = self.ranges[r]
            a, b = self._spill(r)
            cnt = c.counts[0, :, lo:hi]
            return [c.nbr[0, lo * stride:hi * stride], c.nbr[0, N * stride + a:N * stride + b],
                    c.indptr[0, lo:hi], cnt.contiguous() if r == self.g else cnt]

        if self.g == 0:
            # counts arrive as contiguous [L, hi-lo] blocks: receive, then scatter
            def recv_pieces(r):
                p = pieces(r)
                self._cnt_tmp = torch.empty(p[3].shape, dtype=p[3].dtype, device=self.device)
                return p[:3] + [self._cnt_tmp]

            if self.G > 1:
                for r in range(1, self.G):
                    self._to_rank0_one(r, recv_pieces(r))
                    lo, hi = self.ranges[r]
                    c.counts[0, :, lo:hi].copy_(self._cnt_tmp)
        else:
            self._to_rank0_one(self.g, pieces(self.g))
        # 4. sampler on rank 0 over all rows; results broadcast
        if self.g == 0:
            fp._sampler()
        for t in (fp.out, fp.reached, fp.exhausted, fp.entered, fp.state):
            self._bcast(t)
        # 5. early termination: own rows seed own md, split FPS tail
        lvl1 = c.counts[:, int(fp.seg_level_rows[0]), :]
        _lib.call("ps_early_termination_shard", _p(c.indptr), _p(c.nbr), _p(c.d2), c.cap_entries, _p(lvl1),
                  fp.L * N, _p(fp.taken), _p(fp.md), _p(fp.out), n, _p(fp.reached), n, 1, N, self.lo, self.hi, st)
        _lib.call("ps_fps_split_loop", _p(fp.xyz4), 1, N, _p(fp.md), _p(fp.taken), _p(fp.out), _p(fp.curve), n, 1,
                  _p(fp.reached), n, self.G, self.g, 1, _p(s.ptrs), s.seq, 1, st)
        s.seq += n + 1
        if radius is None:
            return fp.out[0]
        # 6. centroid-sharded grouping from the owners' rows
        mine = torch.where((fp.out >= self.lo) & (fp.out < self.hi), fp.out, torch.full_like(fp.out, -1))
        gi, gd, gc = fp.group_rf(radius, k, centroids=mine)
        own = gc >= 0
        acc_i = torch.where(own[..., None], gi + 1, 0)
        acc_d = torch.where(own[..., None], gd, 0.0)
        acc_c = torch.where(own, gc + 1, 0)
        for t in (acc_i, acc_d, acc_c):
            self._allreduce(t, dist.ReduceOp.SUM)
        return fp.out[0], (acc_i[0] - 1, acc_d[0], acc_c[0] - 1)

    def _to_rank0_one(self, r, ts):
        """Move rank r's pieces ts (on rank r: the sources; on rank 0: the
        destinations) to rank 0."""
        if self.g == r and r != 0:
            for t in ts:
                dist.send(t.cpu() if self.gloo else t.contiguous(), dst=0, group=self.group)
        elif self.g == 0 and r != 0:
            for t in ts:
                buf = torch.empty(t.shape, dtype=t.dtype) if self.gloo else torch.empty(t.shape, dtype=t.dtype,
                                                                                          device=self.device)
                dist.recv(buf, src=r, group=self.group)
                t.copy_(buf)

    def close(self):
        self.split.close()
