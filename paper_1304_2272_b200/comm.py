"""Communicators of the multi-GPU engines (reference transport.py:47-140).

The distributed engine needs a handful of collectives on DEVICE tensors -- sum / max all-reduce,
broadcast, both on the whole world and on the row / column sub-groups of the process grid --
plus a few host-side ones (barrier, object gather, byte all-to-all for the element-cyclic
adapters).  Two realisations share one interface:

* ``TorchComm``: torch.distributed.  NCCL over NVLink / NVSwitch on the B200 box (one process
  per GPU, device tensors in place); gloo in the CPU tests.  Row / column groups are NCCL
  sub-communicators (``dist.new_group``), so panel broadcasts move only m_loc x nb / n_loc x nb
  elements per rank instead of world all-reduces of n x nb.
* ``TransportComm``: any object with the reference's Transport contract (rank, size, send, recv,
  broadcast, allgather, alltoall, barrier, allgather_obj -- transport.py:47-140), e.g. the
  reference's in-process or socket transports driving our ``distgrid.run_dist`` after
  ``plugin.install``.  Device tensors travel as host bytes; sums are formed in member order, so
  results are deterministic; sub-group collectives use the transport's ordered point-to-point
  messages.

``as_comm(x)`` accepts None (single rank), the torch.distributed module, a communicator, or a
transport.
"""

from __future__ import annotations

import os

import numpy as np


def _np_dtype(t):
    import torch

    return {torch.float64: np.float64, torch.float32: np.float32, torch.int64: np.int64,
            torch.int32: np.int32, torch.int8: np.int8, torch.uint8: np.uint8}[t.dtype]


class TorchComm:
    """torch.distributed (world or one sub-group) as the engine's communicator."""

    def __init__(self, dist=None, group=None, members=None):
        if dist is None:
            import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.members = members                     # world ranks of the group (None: world)
        self.rank = dist.get_rank(group) if group is not None else dist.get_rank()
        self.size = dist.get_world_size(group) if group is not None else dist.get_world_size()
        self.backend = str(dist.get_backend(group) if group is not None else dist.get_backend())
        self._subs = {}

    def _src(self, root):
        return self.members[root] if self.members is not None else root

    def _run(self, what, fn, *a, **kw):
        """A collective; a communicator failure (NCCL error or watchdog timeout surfaced by
        torch.distributed) becomes TransportFailure(rank, ...) -- the reference's class for a
        failed exchange (errors.py) and the C-ABI's GG_ENCCL meaning."""
        try:
            return fn(*a, **kw)
        except RuntimeError as e:
            from .errors import TransportFailure

            raise TransportFailure(self.rank, f"{what} on {self.backend} failed: {e}") from e

    def all_reduce(self, t, op="sum"):
        if self.size > 1:
            d = self.dist
            self._run("all_reduce", d.all_reduce, t,
                      op=d.ReduceOp.MAX if op == "max" else d.ReduceOp.SUM, group=self.group)
        return t

    def broadcast(self, t, root):
        if self.size > 1:
            self._run("broadcast", self.dist.broadcast, t, src=self._src(root), group=self.group)
        return t

    def barrier(self):
        if self.size > 1:
            self._run("barrier", self.dist.barrier, group=self.group)

    def allgather_obj(self, obj):
        out = [None] * self.size
        if self.size == 1:
            return [obj]
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def alltoall_bytes(self, slices):
        """slices[d] (bytes) goes to member d; returns what every member sent here."""
        import torch

        if self.size == 1:
            return [bytes(slices[0])]
        dev = torch.device("cuda", torch.cuda.current_device()) if self.backend == "nccl" \
            else torch.device("cpu")
        lens = torch.tensor([len(s) for s in slices], dtype=torch.int64, device=dev)
        rlens = torch.empty_like(lens)
        self.dist.all_to_all_single(rlens, lens, group=self.group)
        rl = rlens.cpu().tolist()
        send = torch.from_numpy(np.frombuffer(b"".join(slices), dtype=np.uint8).copy()).to(dev)
        recv = torch.empty(sum(rl), dtype=torch.uint8, device=dev)
        self.dist.all_to_all_single(recv, send, rl, [len(s) for s in slices], group=self.group)
        host = recv.cpu().numpy().tobytes()
        out, off = [], 0
        for n in rl:
            out.append(host[off:off + n])
            off += n
        return out

    def subgroups(self, groups, mine):
        """Collective: create one sub-communicator per member list in ``groups`` (every rank calls
        with the same lists, in the same order) and return the one at index ``mine``."""
        key = tuple(tuple(g) for g in groups)
        if key not in self._subs:
            made = [self.dist.new_group(list(g)) if len(g) > 1 else None for g in groups]
            self._subs[key] = made
        g = self._subs[key][mine]
        if g is None:
            return _SelfComm()
        return TorchComm(self.dist, group=g, members=list(groups[mine]))


class _SelfComm:
    """A group of one: every collective is the identity."""

    rank, size = 0, 1

    def all_reduce(self, t, op="sum"):
        return t

    def broadcast(self, t, root):
        return t

    def barrier(self):
        pass

    def allgather_obj(self, obj):
        return [obj]

    def alltoall_bytes(self, slices):
        return [bytes(slices[0])]

    def subgroups(self, groups, mine):
        return self


class TransportComm:
    """A reference-contract transport (transport.py:47-140) as the engine's communicator;
    ``members`` (world ranks, in order) selects a sub-group."""

    def __init__(self, t, members=None):
        self.t = t
        self.members = list(members) if members is not None else list(range(t.size))
        self.world = len(self.members) == t.size
        self.rank = self.members.index(t.rank)
        self.size = len(self.members)

    # -- host byte helpers -------------------------------------------------------------------
    def _gather_bytes(self, raw):
        """Every member's bytes, in member order, on every member."""
        t = self.t
        if self.world:
            return list(t.allgather(raw))
        lead = self.members[0]
        if t.rank == lead:
            parts = [raw] + [t.recv(src) for src in self.members[1:]]
            packed = _pack(parts)
            for dst in self.members[1:]:
                t.send(dst, packed)
            return parts
        t.send(lead, raw)
        return _unpack(t.recv(lead))

    def all_reduce(self, x, op="sum"):
        if self.size == 1:
            return x
        import torch

        dt = _np_dtype(x)
        parts = self._gather_bytes(x.detach().cpu().contiguous().numpy().tobytes())
        acc = np.frombuffer(parts[0], dtype=dt).copy()
        for p in parts[1:]:
            a = np.frombuffer(p, dtype=dt)
            acc = np.maximum(acc, a) if op == "max" else acc + a
        x.copy_(torch.from_numpy(acc.reshape(tuple(x.shape))).to(x.device))
        return x

    def broadcast(self, x, root):
        if self.size == 1:
            return x
        import torch

        t = self.t
        src = self.members[root]
        raw = x.detach().cpu().contiguous().numpy().tobytes() if t.rank == src else b""
        if self.world:
            raw = t.broadcast(src, raw)
        elif t.rank == src:
            for dst in self.members:
                if dst != src:
                    t.send(dst, raw)
        else:
            raw = t.recv(src)
        if t.rank != src:
            a = np.frombuffer(raw, dtype=_np_dtype(x)).reshape(tuple(x.shape))
            x.copy_(torch.from_numpy(a.copy()).to(x.device))
        return x

    def barrier(self):
        if self.world:
            self.t.barrier()
        else:
            self._gather_bytes(b"")

    def allgather_obj(self, obj):
        if self.world:
            return list(self.t.allgather_obj(obj))
        import pickle

        return [pickle.loads(p) for p in self._gather_bytes(pickle.dumps(obj))]

    def alltoall_bytes(self, slices):
        if self.world:
            return list(self.t.alltoall([bytes(s) for s in slices]))
        raise NotImplementedError("byte all-to-all on a transport sub-group")

    def subgroups(self, groups, mine):
        g = groups[mine]
        return TransportComm(self.t, g) if len(g) > 1 else _SelfComm()


def _pack(parts):
    import struct

    out = [struct.pack("<I", len(parts))]
    for p in parts:
        out.append(struct.pack("<Q", len(p)))
        out.append(p)
    return b"".join(out)


def _unpack(data):
    import struct

    (count,) = struct.unpack_from("<I", data, 0)
    off, parts = 4, []
    for _ in range(count):
        (ln,) = struct.unpack_from("<Q", data, off)
        off += 8
        parts.append(bytes(data[off:off + ln]))
        off += ln
    return parts


def init_process_group(backend, rank=None, world_size=None, device=None):
    """torch.distributed.init_process_group with the engine's failure policy: NCCL's async error
    handling on (a failed or hung collective aborts the communicator and surfaces as an
    exception instead of blocking every rank forever) and a bounded timeout
    (GG_COLLECTIVE_TIMEOUT_S, default 1800 s)."""
    import datetime

    import torch.distributed as dist

    os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")
    kw = {"timeout": datetime.timedelta(
        seconds=float(os.environ.get("GG_COLLECTIVE_TIMEOUT_S", "1800")))}
    if rank is not None:
        kw.update(rank=rank, world_size=world_size)
    if device is not None and backend == "nccl":
        kw["device_id"] = device
    dist.init_process_group(backend, **kw)
    return dist


def as_comm(x):
    """None -> None (single rank); a communicator -> itself; the torch.distributed module (or an
    object carrying ``comm``) -> TorchComm; a reference Transport -> TransportComm."""
    if x is None:
        return None
    if isinstance(x, (TorchComm, TransportComm, _SelfComm)):
        return x
    if getattr(x, "comm", None) is not None:            # transport.NcclTransport
        return x.comm
    if hasattr(x, "all_reduce") and hasattr(x, "ReduceOp"):
        if not (x.is_available() and x.is_initialized()):
            return None
        return TorchComm(x)
    if hasattr(x, "allgather") and hasattr(x, "send") and hasattr(x, "size"):
        return TransportComm(x)
    raise TypeError(f"cannot use {type(x).__name__} as a communicator")


class GridComm:
    """World + row + column communicators of an r x c process grid (collective to build)."""

    def __init__(self, comm, grid):
        self.world = comm
        pr, pc = grid.coord(comm.rank)
        rows = [[grid.rank_of(i, j) for j in range(grid.c)] for i in range(grid.r)]
        cols = [[grid.rank_of(i, j) for i in range(grid.r)] for j in range(grid.c)]
        self.row = comm.subgroups(rows, pr)       # member index = process column
        self.col = comm.subgroups(cols, pc)       # member index = process row
