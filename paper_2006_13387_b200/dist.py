"""Multi-GPU strips: attach a communicator to the C-ABI context.

One process per GPU (torchrun).  ``init_nccl()`` shares an NCCL unique id
over the already-initialised ``torch.distributed`` group and attaches a
native NCCL communicator: all halo exchanges, dot-product allreduces and the
coarse-residual allreduce then run inside the device-resident PCG loop (and
are captured into its CUDA graphs).  ``init_host_callbacks()`` attaches a
communicator that calls back into ``torch.distributed`` with host staging --
any backend, including gloo with several ranks on ONE GPU (their kernels
never wait on each other); it exists to test the multi-rank logic.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._context import default_context


def strip_rows(nrows, world, rank):
    lo, hi = C.c_int(), C.c_int()
    _lib.check(_lib.load().ms_strip_rows(int(nrows), int(world), int(rank), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def halo_plan(lo, hi, ny, k, rank, world):
    """The C++ halo plan: [(send_lo, send_n, dst, recv_lo, recv_n, src)] x 2 slots."""
    out = (C.c_int * 12)()
    _lib.check(_lib.load().ms_halo_plan(lo, hi, ny, k, rank, world, out))
    v = list(out)
    return [tuple(v[0:6]), tuple(v[6:12])]


def init_nccl(device=None):
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    ctx = default_context(device)
    lib = _lib.load()
    uid = C.create_string_buffer(128)
    if rank == 0:
        _lib.check(lib.ms_nccl_unique_id(uid))
    obj = [bytes(uid.raw)]
    dist.broadcast_object_list(obj, src=0)
    _lib.check(lib.ms_ctx_attach_nccl(ctx.handle, rank, world, obj[0]), ctx.handle)
    return ctx


class _HostComm:
    """torch.distributed collectives on host copies of device buffers."""

    def __init__(self):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        lib = _lib.load()
        self.copy = lib.ms_copy

        def allreduce(user, dev, n):
            try:
                h = np.empty(n, dtype=np.float64)
                _lib.check(self.copy(h.ctypes.data, dev, h.nbytes))
                t = torch.from_numpy(h)
                dist.all_reduce(t)
                _lib.check(self.copy(dev, h.ctypes.data, h.nbytes))
                return 0
            except Exception:  # pragma: no cover
                return 1

        def broadcast(user, dev, nbytes, root):
            try:
                h = np.empty(nbytes, dtype=np.uint8)
                if dist.get_rank() == root:
                    _lib.check(self.copy(h.ctypes.data, dev, nbytes))
                t = torch.from_numpy(h)
                dist.broadcast(t, src=root)
                if dist.get_rank() != root:
                    _lib.check(self.copy(dev, h.ctypes.data, nbytes))
                return 0
            except Exception:  # pragma: no cover
                return 1

        def sendrecv(user, sdev, sbytes, dst, rdev, rbytes, src):
            try:
                reqs = []
                if dst >= 0 and sbytes > 0:
                    hs = np.empty(sbytes, dtype=np.uint8)
                    _lib.check(self.copy(hs.ctypes.data, sdev, sbytes))
                    reqs.append(dist.isend(torch.from_numpy(hs), dst))
                hr = None
                if src >= 0 and rbytes > 0:
                    hr = np.empty(rbytes, dtype=np.uint8)
                    reqs.append(dist.irecv(torch.from_numpy(hr), src))
                for q in reqs:
                    q.wait()
                if hr is not None:
                    _lib.check(self.copy(rdev, hr.ctypes.data, rbytes))
                return 0
            except Exception:  # pragma: no cover
                return 1

        self._keep = (_lib.ALLREDUCE_CB(allreduce), _lib.BROADCAST_CB(broadcast), _lib.SENDRECV_CB(sendrecv))
        self.struct = _lib.CommCallbacks(None, *self._keep)


_HOST_COMMS = []


def init_host_callbacks(device=None):
    import torch.distributed as dist

    ctx = default_context(device)
    hc = _HostComm()
    _HOST_COMMS.append(hc)  # keep the ctypes callbacks alive
    _lib.check(_lib.load().ms_ctx_attach_callbacks(ctx.handle, dist.get_rank(), dist.get_world_size(),
                                                   C.byref(hc.struct)), ctx.handle)
    return ctx
