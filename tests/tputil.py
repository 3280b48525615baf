"""Single-process, multi-device driver of malleus_k_tp_reduce (one member per visible GPU, peer
access enabled between them) for the TP-reduction parity test and tools/tp_bench.py."""
from __future__ import annotations

import ctypes as C

import torch

from paper_2410_13333_b200 import _lib as L

TPF_WORDS = 64


def enable_peer_access(k: int) -> None:
    from cuda.bindings import runtime as rt  # cuda-python
    for i in range(k):
        rt.cudaSetDevice(i)
        for j in range(k):
            if i != j:
                err, = rt.cudaDeviceEnablePeerAccess(j, 0)
                if err not in (rt.cudaError_t.cudaSuccess, rt.cudaError_t.cudaErrorPeerAccessAlreadyEnabled):
                    raise RuntimeError(f"peer access {i}->{j}: {err}")
    rt.cudaGetLastError()


def _ptrs(ts):
    arr = (C.c_void_p * len(ts))(*[t.data_ptr() if t is not None else None for t in ts])
    return arr


class Group:
    """k members: double-buffered partials, flag blocks, destinations.  devices[j] is member j's GPU
    (default cuda:j, one member per GPU, peer access enabled); members sharing one GPU each run on
    their own stream (their grids must be small enough to be co-resident).  rows: optional uneven
    row split [k + 1] (row_split of malleus_k_tp_reduce)."""

    def __init__(self, k: int, T: int, h: int, part_dtype=torch.float32, sum_bf16: bool = False,
                 devices=None, rows=None):
        self.k, self.T, self.h = k, T, h
        # part_dtype bit 0: bf16 partials, bit 1: bf16 SUM output
        self.pdt = (1 if part_dtype == torch.bfloat16 else 0) | (2 if sum_bf16 else 0)
        self.devices = list(range(k)) if devices is None else list(devices)
        dev = [torch.device("cuda", j) for j in self.devices]
        self.part = [[torch.zeros(T, h, device=d, dtype=part_dtype) for d in dev] for _ in range(2)]
        self.flags = [torch.zeros(TPF_WORDS, dtype=torch.int64, device=d) for d in dev]
        self.out32 = [torch.zeros(T, h, device=d, dtype=torch.bfloat16 if sum_bf16 else torch.float32) for d in dev]
        self.x1 = [torch.zeros(T, h, dtype=torch.bfloat16, device=d) for d in dev]
        self.a = [torch.zeros(T, h, dtype=torch.bfloat16, device=d) for d in dev]
        self.rstd = [torch.zeros(T, device=d) for d in dev]
        self.streams = [torch.cuda.Stream(device=d) for d in dev]
        self.rows = (C.c_int32 * (k + 1))(*rows) if rows is not None else None
        self.epoch = 0
        for d in set(self.devices):
            torch.cuda.synchronize(d)

    def launch(self, mode: int, x=None, g=None, eps: float = 1e-5, skip=()) -> None:
        """One reduction of the partials in buffer (epoch + 1) & 1; all members launched
        asynchronously, each on its own stream (after the device's current stream).  Members in
        `skip` are not launched (an unresponsive member, for the failure-detection tests)."""
        self.epoch += 1
        buf = self.epoch & 1
        parts = _ptrs(self.part[buf])
        flags = _ptrs(self.flags)
        if mode == 0:
            d0, d1, d2 = _ptrs(self.out32), None, None
        elif mode == 1:
            d0, d1, d2 = _ptrs(self.x1), _ptrs(self.a), _ptrs(self.rstd)
        else:
            d0, d1, d2 = _ptrs(self.x1), None, None
        for j in range(self.k):
            if j in skip:
                continue
            dj = self.devices[j]
            with torch.cuda.device(dj):
                self.streams[j].wait_stream(torch.cuda.current_stream(dj))
                st = self.streams[j].cuda_stream
                r = L.lib.malleus_k_tp_reduce(self.k, j, self.T, self.h, mode, self.pdt, eps, self.epoch,
                                              C.cast(parts, C.c_void_p), C.cast(flags, C.c_void_p),
                                              C.cast(d0, C.c_void_p), C.cast(d1, C.c_void_p) if d1 else None,
                                              C.cast(d2, C.c_void_p) if d2 else None,
                                              x[j].data_ptr() if x is not None else None,
                                              g[j].data_ptr() if g is not None else None,
                                              C.cast(self.rows, C.c_void_p) if self.rows is not None else None, st)
                assert r == 0, r

    def sync(self) -> None:
        for d in set(self.devices):
            torch.cuda.synchronize(d)
