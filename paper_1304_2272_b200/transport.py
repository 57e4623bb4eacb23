"""The ``transport="nccl"`` realisation of the reference's SPMD launcher (transport.py:267-327).

``run_spmd(size, fn, *args, transport="nccl")`` starts ``size`` worker processes (spawned; one
per GPU, device = rank mod device count), joins them in one torch.distributed group (NCCL on the
B200 box; ``GG_SPMD_BACKEND=gloo`` for CPU tests or several ranks sharing one GPU), runs
``fn(t, *args)`` on every rank and returns the per-rank results in rank order, re-raising the
first failure -- the reference's contract.  ``t`` is an ``NcclTransport``: the reference's
Transport interface (rank, size, send/recv of bytes, barrier, broadcast, allgather, alltoall,
broadcast_obj, allgather_obj, counters; transport.py:47-140) for host messages, plus ``t.comm``,
the device communicator the B200 engine uses (comm.TorchComm: NCCL all-reduce / broadcast on
device tensors, row / column sub-communicators).  ``fn`` must be picklable (a module-level
function such as distgrid.run_dist).

The reference's "inproc" and "socket" realisations are not re-implemented here (SURVEY §2 marks
them out of scope); ``plugin.install`` routes only transport="nccl" to this module.
"""

from __future__ import annotations

import os
import pickle
import socket
import traceback

import numpy as np

from .comm import TorchComm, init_process_group
from .errors import TransportFailure


class NcclTransport:
    """The reference Transport contract over torch.distributed (host bytes on a gloo group, the
    engine's device collectives on the default group through ``comm``)."""

    def __init__(self, rank, size):
        import torch.distributed as dist

        self.dist = dist
        self.rank, self.size = rank, size
        self.backend = str(dist.get_backend())
        # host messages always travel on gloo (NCCL moves device tensors only)
        self._cpu = dist.new_group(backend="gloo") if self.backend != "gloo" else None
        self.comm = TorchComm(dist)
        self.bytes_sent = 0
        self.bytes_received = 0

    # -- point to point ------------------------------------------------------------------------
    def send(self, dst, data, _channel=0):
        import torch

        if not 0 <= dst < self.size:
            raise TransportFailure(self.rank, f"bad destination {dst}")
        data = bytes(data)
        self.bytes_sent += len(data)
        self.dist.send(torch.tensor([len(data)], dtype=torch.int64), dst, group=self._cpu)
        if data:
            self.dist.send(torch.from_numpy(np.frombuffer(data, dtype=np.uint8).copy()), dst,
                           group=self._cpu)

    def recv(self, src, _channel=0):
        import torch

        n = torch.empty(1, dtype=torch.int64)
        self.dist.recv(n, src, group=self._cpu)
        k = int(n.item())
        buf = torch.empty(k, dtype=torch.uint8)
        if k:
            self.dist.recv(buf, src, group=self._cpu)
        self.bytes_received += k
        return buf.numpy().tobytes()

    # -- collectives ---------------------------------------------------------------------------
    def barrier(self):
        self.dist.barrier(group=self._cpu)

    def broadcast_obj(self, root, obj=None):
        box = [obj]
        self.dist.broadcast_object_list(box, src=root, group=self._cpu)
        return box[0]

    def allgather_obj(self, obj):
        out = [None] * self.size
        self.dist.all_gather_object(out, obj, group=self._cpu)
        return out

    def broadcast(self, root, data=b""):
        return self.broadcast_obj(root, bytes(data) if self.rank == root else None)

    def allgather(self, data):
        return self.allgather_obj(bytes(data))

    def alltoall(self, slices):
        """slices[d] to rank d (pairwise exchange in a fixed order: deterministic)."""
        out = [None] * self.size
        out[self.rank] = bytes(slices[self.rank])
        for step in range(1, self.size):
            dst = (self.rank + step) % self.size
            src = (self.rank - step) % self.size
            if self.rank < dst:
                self.send(dst, slices[dst])
                out[src] = self.recv(src)
            else:
                out[src] = self.recv(src)
                self.send(dst, slices[dst])
        return out

    def counters(self):
        return self.bytes_sent + self.bytes_received

    def close(self):
        pass


def _free_port():
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, size, port, backend, fn, args, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(size), LOCAL_RANK=str(rank))
    try:
        device = None
        if torch.cuda.is_available():
            dev = rank % torch.cuda.device_count()
            torch.cuda.set_device(dev)
            device = torch.device("cuda", dev)
        init_process_group(backend, rank=rank, world_size=size, device=device)
        t = NcclTransport(rank, size)
        try:
            res = fn(t, *args)
            q.put((rank, "ok", pickle.dumps(res)))
        finally:
            dist.destroy_process_group()
    except BaseException as e:      # noqa: BLE001 - shipped to the launcher
        try:
            payload = pickle.dumps(e)
        except Exception:          # unpicklable exception: ship its text
            payload = pickle.dumps(TransportFailure(rank, traceback.format_exc()))
        q.put((rank, "err", payload))


def run_spmd(size, fn, *args, transport="nccl"):
    """Run fn(t, *args) on ``size`` ranks (one process each); per-rank results in rank order."""
    if transport != "nccl":
        raise ValueError(f"unknown transport {transport!r} (this package realises 'nccl'; the "
                         "reference provides 'inproc' and 'socket')")
    import torch.multiprocessing as mp

    backend = os.environ.get("GG_SPMD_BACKEND", "nccl")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port, backend, fn, args, q))
             for r in range(size)]
    for p in procs:
        p.start()
    timeout = float(os.environ.get("GG_SPMD_TIMEOUT", "3600"))
    outs = {}
    try:
        for _ in range(size):
            rank, status, payload = q.get(timeout=timeout)
            outs[rank] = (status, pickle.loads(payload))
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for r in range(size):
        status, val = outs[r]
        if status == "err":
            raise val
    return [outs[r][1] for r in range(size)]
