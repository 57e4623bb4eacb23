"""Test-only in-process SPMD harness with the reference's Transport contract (transport.py:47-140:
rank, size, send/recv, barrier, broadcast, allgather, alltoall, broadcast_obj, allgather_obj):
ranks are threads exchanging bytes through queues.  It stands in for the reference's own
``run_spmd(transport="inproc")`` so the CPU tests can drive the reference-signature adapters
(distgrid.dist_cholesky / dist_trsolve / run_dist) without importing /root/reference.
"""

import pickle
import queue
import threading

import numpy as np


class InprocT:
    def __init__(self, rank, size, boxes):
        self.rank, self.size, self._boxes = rank, size, boxes
        self.bytes_sent = self.bytes_received = 0

    def send(self, dst, data, _channel=0):
        self.bytes_sent += len(data)
        self._boxes[(self.rank, dst, _channel)].put(bytes(data))

    def recv(self, src, _channel=0):
        d = self._boxes[(src, self.rank, _channel)].get(timeout=120)
        self.bytes_received += len(d)
        return d

    def barrier(self):
        self.allgather(b"")

    def broadcast(self, root, data=b""):
        if self.rank == root:
            for d in range(self.size):
                if d != root:
                    self.send(d, data, 1)
            return bytes(data)
        return self.recv(root, 1)

    def allgather(self, data):
        for d in range(self.size):
            if d != self.rank:
                self.send(d, data, 1)
        return [bytes(data) if s == self.rank else self.recv(s, 1) for s in range(self.size)]

    def alltoall(self, slices):
        for d in range(self.size):
            if d != self.rank:
                self.send(d, slices[d], 1)
        return [bytes(slices[s]) if s == self.rank else self.recv(s, 1)
                for s in range(self.size)]

    def broadcast_obj(self, root, obj=None):
        return pickle.loads(self.broadcast(root, pickle.dumps(obj) if self.rank == root else b""))

    def allgather_obj(self, obj):
        return [pickle.loads(b) for b in self.allgather(pickle.dumps(obj))]

    def counters(self):
        return self.bytes_sent + self.bytes_received


def run_spmd(size, fn, *args):
    boxes = {(s, d, ch): queue.SimpleQueue() for s in range(size) for d in range(size)
             for ch in (0, 1)}
    res, errs = [None] * size, [None] * size

    def work(r):
        try:
            res[r] = fn(InprocT(r, size, boxes), *args)
        except BaseException as e:      # noqa: BLE001 - re-raised below
            errs[r] = e

    ths = [threading.Thread(target=work, args=(r,)) for r in range(size)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    for e in errs:
        if e is not None:
            raise e
    return res


class EC:
    """Element-cyclic DistMatrix2D stand-in (the reference's layout, distgrid.py:76-89:
    local = A[prow::r, pcol::c])."""

    def __init__(self, gr, gc, grid, rank, local):
        self.gr, self.gc, self.grid, self.rank, self.local = gr, gc, grid, rank, local

    @classmethod
    def of(cls, A, grid, rank):
        pr, pc = grid.coord(rank)
        return cls(A.shape[0], A.shape[1], grid, rank, np.array(A[pr::grid.r, pc::grid.c]))


def gather_ec(D, t):
    parts = t.allgather_obj(D.local)
    out = np.zeros((D.gr, D.gc))
    for src, part in enumerate(parts):
        pr, pc = D.grid.coord(src)
        out[pr::D.grid.r, pc::D.grid.c] = part
    return out

