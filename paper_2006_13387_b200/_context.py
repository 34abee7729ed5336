"""Process-wide CUDA context handles for the C ABI (one stream per context)."""

from __future__ import annotations

import ctypes as C
import threading

from . import _lib

_lock = threading.Lock()
_contexts = {}


class Context:
    def __init__(self, device=0):
        lib = _lib.load()
        h = C.c_void_p()
        _lib.check(lib.ms_ctx_create(int(device), C.byref(h)))
        self.handle = h
        self.device = int(device)


def default_context(device=None):
    if device is None:
        try:
            import torch

            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        except Exception:
            device = 0
    with _lock:
        if device not in _contexts:
            _contexts[device] = Context(device)
        return _contexts[device]
