"""Multi-GPU kernelization: one process (rank) per GPU, one exchange per phase.

SURVEY.md 8(e): the incidence operand is replicated (every rank packs it from
the same CSR), each rank runs an interleaved share of the phase's triangle tile
list (``mhsk_tile_list``; interleaved share, :func:`shard_share`), and the per-item
deleter counts -- the only data that crosses GPUs -- are summed in place
between the Gram product and the commit.  Integer sums are order-independent,
so every rank commits bit-identical deletions and the alive state stays
replicated with no further traffic.  The sum is an NCCL all-reduce over
NVLink (:class:`TorchDistAllreduce` on a ``torch.distributed`` NCCL group);
:class:`InProcessAllreduce` is the same contract for several ranks driven
from one process (threads), used by the single-GPU tests.
"""

from __future__ import annotations

import threading

import numpy as np

from . import _native


def shard_share(total: int, rank: int, world: int) -> range:
    """Indices of the tiles rank runs out of a `total`-tile list: rank,
    rank + world, ... (mirrors shard_share in csrc/mhsk_capi.cu).  Interleaving
    keeps the ranks balanced when later rounds shrink M and only a prefix-like
    subset of the tile list stays inside it."""
    return range(min(rank, total), total, world)


def _wrap_device_int32(ptr: int, count: int, device: int):
    import torch

    class _CAI:
        __cuda_array_interface__ = {"shape": (count,), "typestr": "<i4", "data": (ptr, False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_CAI(), device=torch.device("cuda", device))


class TorchDistAllreduce:
    """Sum the library's device buffer over a torch.distributed group (NCCL),
    ordered on the library's stream."""

    def __init__(self, device: int, group=None):
        self.device = device
        self.group = group
        self._streams: dict[int, object] = {}

    def __call__(self, ptr: int, count: int, stream: int) -> None:
        import torch
        import torch.distributed as dist

        s = self._streams.get(stream)
        if s is None:
            s = torch.cuda.ExternalStream(stream, device=torch.device("cuda", self.device))
            self._streams[stream] = s
        buf = _wrap_device_int32(ptr, count, self.device)
        with torch.cuda.stream(s):
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group)


class InProcessAllreduce:
    """All-reduce (sum) among `world` ranks that run as threads of one
    process, each with its own libmhsk context.  Host-side exchange: no
    kernel ever waits on another rank's kernel."""

    def __init__(self, world: int):
        self.world = world
        self._barrier = threading.Barrier(world)
        self._parts: list[np.ndarray | None] = [None] * world
        self._total: np.ndarray | None = None

    def for_rank(self, rank: int, device: int):
        def reduce(ptr: int, count: int, stream: int) -> None:
            import torch

            torch.cuda.ExternalStream(stream, device=torch.device("cuda", device)).synchronize()
            buf = _wrap_device_int32(ptr, count, device)
            self._parts[rank] = buf.cpu().numpy().copy()
            if self._barrier.wait() == 0:
                self._total = np.sum(np.stack(self._parts), axis=0, dtype=np.int64).astype(np.int32)
            self._barrier.wait()
            buf.copy_(torch.from_numpy(self._total))
            torch.cuda.synchronize(device)
            self._barrier.wait()

        return reduce


def kernelize_sharded(csr, *, rank: int, world: int, allreduce, rule: str = "dp",
                      device: int = 0, backend: str = "tc", options: dict | None = None):
    """Run one rank of a `world`-rank kernelization; returns (vertex_alive,
    edge_alive, stats) -- identical on every rank."""
    ctx = _native.Context(device, backend=backend)
    try:
        for k, v in (options or {}).items():
            ctx.set_option(k, v)
        ctx.set_shard(rank, world, allreduce)
        return ctx.kernelize(csr, rule)
    finally:
        ctx.close()


def kernelize_in_process(csr, world: int, *, rule: str = "dp", device: int = 0,
                         backend: str = "tc", options: dict | None = None):
    """`world` ranks as threads on one device (test harness for the sharded
    path); returns the list of per-rank results."""
    ar = InProcessAllreduce(world)
    out: list = [None] * world
    errors: list = []

    def run(r: int):
        try:
            out[r] = kernelize_sharded(csr, rank=r, world=world, allreduce=ar.for_rank(r, device),
                                       rule=rule, device=device, backend=backend, options=options)
        except BaseException as exc:  # surface in the caller
            errors.append(exc)
            ar._barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return out
