"""Sharded lane: one graph, vertices 1-D partitioned over ranks.

Every rank holds the prepared graph; rank r improves the policy of vertices
``[r*chunk, (r+1)*chunk)`` only (the O(M) part of an iteration). After each
improvement pass the ranks exchange the policy slices (all-gather of
``succ_e``, ``succ_v``, ``succ_w`` in chunk-sized pieces, NCCL over NVLink
between GPUs) and max-reduce the per-region change flags; cycle detection,
the vote and value determination then run replicated on every rank, so the
ranks stay bit-identical without exchanging values. Each rank's native
session stops at the exchange point (``ocm_session_shard_step``) and resumes
after it.

The exchange is pluggable: :class:`TorchComm` uses ``torch.distributed``
(one process per GPU, NCCL; gloo on CPU), :class:`LocalComm` exchanges
between several shards held by one process (all on one device) -- the
single-GPU check that the partitioned iteration reproduces the unsharded one.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Union

import numpy as np

from . import (Generator, Graph, Solution, SolveOptions, _check, _lib, _ShardBuffers, _ShardPeer,
               _Sol, _solution)

__all__ = ["ShardSession", "TorchComm", "LocalComm", "solve_sharded", "connect_local",
           "connect_torch", "solve_fused"]


class _DeviceArray:
    """Zero-copy ``__cuda_array_interface__`` view of a session buffer."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None, "stream": None}


class ShardSession:
    """Rank ``rank`` of ``world`` of a sharded solve of one graph."""

    def __init__(self, source: Union[Graph, Generator], opt: Optional[SolveOptions] = None,
                 rank: int = 0, world: int = 1):
        self.opt = opt or SolveOptions()
        h = C.c_void_p()
        if isinstance(source, Graph):
            _check(_lib.ocm_session_create_shard(source._h, None, C.byref(self.opt._c()),
                                                 int(rank), int(world), C.byref(h)))
        else:
            _check(_lib.ocm_session_create_shard(None, C.byref(source._c()),
                                                 C.byref(self.opt._c()), int(rank), int(world),
                                                 C.byref(h)))
        self._h = h
        b = _ShardBuffers()
        _check(_lib.ocm_session_shard_buffers(h, C.byref(b)))
        self.buffers = b
        self.rank, self.world, self.chunk, self.n = b.rank, b.world, b.chunk, b.n
        self._tensors = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and _lib is not None:
            _lib.ocm_session_free(h)
            self._h = C.c_void_p(None)

    def tensors(self):
        """torch views of the exchanged buffers: (succ_e, succ_v, succ_w) of
        world*chunk entries each, and the two region-flag arrays."""
        if self._tensors is None:
            import torch
            b = self.buffers
            full = int(b.world) * int(b.chunk)
            wt = "<i4" if b.succ_w_bytes == 4 else "<f8"
            dev = torch.device("cuda", self.opt.device)
            views = [_DeviceArray(b.succ_e, full, "<u4"), _DeviceArray(b.succ_v, full, "<u4"),
                     _DeviceArray(b.succ_w, full, wt), _DeviceArray(b.changed0, b.regions, "<i4"),
                     _DeviceArray(b.changed1, b.regions, "<i4")]
            # uint32 has no torch equivalent everywhere: exchange the bits as int32
            ts = []
            for v in views:
                t = torch.as_tensor(v, device=dev)
                if t.dtype == torch.uint32:
                    t = t.view(torch.int32)
                ts.append(t)
            self._tensors = (ts[:3], ts[3:], views)
        return self._tensors[0], self._tensors[1]

    def step(self) -> bool:
        done = C.c_int32()
        _check(_lib.ocm_session_shard_step(self._h, C.byref(done)))
        return bool(done.value)

    def finish(self) -> Solution:
        sol = _Sol()
        cyc = np.empty(max(self.n, 1), np.uint32)
        _check(_lib.ocm_session_shard_finish(self._h, C.byref(sol), cyc.ctypes.data_as(
            C.POINTER(C.c_uint32)), cyc.shape[0]))
        return _solution(sol, cyc)

    def values(self):
        from . import Session
        return Session.values(self)  # same native call on the session handle

    # ---- fused lane (one launch per solve per rank, exchange inside the kernel)
    def peer_info(self) -> bytes:
        """This rank's exchange-buffer descriptor (device pointers + IPC handles)."""
        info = _ShardPeer()
        _check(_lib.ocm_session_shard_peer_info(self._h, C.byref(info)))
        return bytes(info)

    def connect(self, infos: Sequence[bytes], use_ipc: bool) -> None:
        """Map every rank's buffers (rank-ordered descriptors)."""
        arr = (_ShardPeer * len(infos))()
        for q, raw in enumerate(infos):
            C.memmove(C.byref(arr[q]), raw, C.sizeof(_ShardPeer))
        _check(_lib.ocm_session_shard_connect(self._h, arr, len(infos), 1 if use_ipc else 0))

    def fused_launch(self) -> None:
        _check(_lib.ocm_session_shard_fused_launch(self._h))

    def fused_finish(self) -> Solution:
        sol = _Sol()
        cyc = np.empty(max(self.n, 1), np.uint32)
        _check(_lib.ocm_session_shard_fused_finish(self._h, C.byref(sol), cyc.ctypes.data_as(
            C.POINTER(C.c_uint32)), cyc.shape[0]))
        return _solution(sol, cyc)


class TorchComm:
    """Exchange over torch.distributed: one local shard per process."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.inplace = dist.get_backend(group) == "nccl"

    def exchange_arrays(self, policy: Sequence, flags: Sequence, chunk: int) -> None:
        """All-gather the rank's chunk of every policy array (in place) and
        max-reduce the flag arrays. Non-NCCL backends (gloo: CPU tests, or
        several ranks sharing one GPU) exchange through host copies."""
        for t in policy:
            mine = t.narrow(0, self.rank * chunk, chunk)
            if self.inplace:
                # NCCL allows the send buffer to be the receiver's own slice
                self.dist.all_gather_into_tensor(t, mine, group=self.group)
            else:
                host = t.cpu()
                self.dist.all_gather_into_tensor(
                    host, host.narrow(0, self.rank * chunk, chunk).clone(), group=self.group)
                t.copy_(host)
        for f in flags:
            if self.inplace:
                self.dist.all_reduce(f, op=self.dist.ReduceOp.MAX, group=self.group)
            else:
                host = f.cpu()
                self.dist.all_reduce(host, op=self.dist.ReduceOp.MAX, group=self.group)
                f.copy_(host)

    def exchange(self, shards: Sequence[ShardSession]) -> None:
        import torch
        (sh,) = shards
        policy, flags = sh.tensors()
        self.exchange_arrays(policy, flags, sh.chunk)
        torch.cuda.synchronize()  # the next shard step (session stream) reads them


class LocalComm:
    """Exchange between shards held by one process (one device)."""

    def exchange(self, shards: Sequence[ShardSession]) -> None:
        import torch
        tens = [sh.tensors() for sh in shards]
        chunk = shards[0].chunk
        for r, sh in enumerate(shards):  # owner's slice -> everyone
            for k in range(3):
                src = tens[r][0][k].narrow(0, r * chunk, chunk)
                for q in range(len(shards)):
                    if q != r:
                        tens[q][0][k].narrow(0, r * chunk, chunk).copy_(src)
        for k in range(2):
            m = tens[0][1][k].clone()
            for q in range(1, len(shards)):
                m = torch.maximum(m, tens[q][1][k])
            for q in range(len(shards)):
                tens[q][1][k].copy_(m)
        torch.cuda.synchronize()


def solve_sharded(shards: Sequence[ShardSession], comm) -> List[Solution]:
    """Drive the local shard(s) through one solve: step to the exchange
    point, exchange, repeat until the (replicated) convergence test stops
    every rank at the same launch."""
    while True:
        done = [sh.step() for sh in shards]
        if all(done):
            break
        if any(done):
            raise RuntimeError("sharded lane: ranks disagree on convergence")
        comm.exchange(shards)
    return [sh.finish() for sh in shards]


def connect_local(shards: Sequence[ShardSession]) -> None:
    """Connect shards held by one process (raw device pointers)."""
    infos = [sh.peer_info() for sh in shards]
    for sh in shards:
        sh.connect(infos, use_ipc=False)


def connect_torch(shard: ShardSession, group=None) -> None:
    """Connect one shard per process: descriptors all-gathered over
    torch.distributed, peers' buffers opened through CUDA IPC."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    infos = [None] * world
    dist.all_gather_object(infos, shard.peer_info(), group=group)
    shard.connect(infos, use_ipc=True)


def solve_fused(shards: Sequence[ShardSession]) -> List[Solution]:
    """One fused solve of the local (connected) shard(s): launch every local
    rank first -- their kernels must run concurrently, they wait for each
    other at the cross-rank barriers -- then collect."""
    for sh in shards:
        sh.fused_launch()
    return [sh.fused_finish() for sh in shards]
