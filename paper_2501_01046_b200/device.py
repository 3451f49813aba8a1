"""Device context: one ``nd_ctx`` (CUDA device, streams, uploaded family,
scratch) per process and GPU, the B200 analogue of the reference's worker pool
(util.cpp:81-122)."""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _lib
from ._lib import check


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class Context:
    """Owns an nd_ctx on ``device``, or -- with ``devices`` -- one context over
    several GPUs (nd_ctx_create_multi: signatures and dedup sharded over the
    devices, records exchanged over NVLink peer copies; a device may repeat).
    Not reentrant (nd_ctx contract)."""

    def __init__(self, device: int = 0, stream: int | None = None, devices=None):
        self.lib = _lib.load()
        h = C.c_void_p()
        if devices is not None:
            devs = (C.c_int * len(devices))(*devices)
            check(self.lib.nd_ctx_create_multi(devs, len(devices), C.byref(h)))
            device = devices[0]
        else:
            check(self.lib.nd_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self.devices = list(devices) if devices is not None else [device]
        self._family_key = None
        if stream is not None:
            self.set_stream(stream)

    def set_stream(self, stream: int | None) -> None:
        check(self.lib.nd_ctx_set_stream(self.h, C.c_void_p(stream or 0)), self.h)

    @property
    def shards(self) -> int:
        return int(self.lib.nd_ctx_shard_count(self.h))

    def close(self) -> None:
        if self.h:
            self.lib.nd_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int) -> None:
        check(rc, self.h)

    def upload_family(self, family) -> None:
        key = (family.seed, family.hash_count, family.shingle_len, int(family.unit),
               bytes(family.functions))
        if key == self._family_key:
            return
        self.check(self.lib.nd_family_upload(self.h, family.functions, family.hash_count,
                                             family.shingle_len, int(family.unit)))
        self._family_key = key


_default: dict[int, Context] = {}
_default_lock = threading.Lock()


def default_context(device: int = 0) -> Context:
    with _default_lock:
        ctx = _default.get(device)
        if ctx is None:
            ctx = Context(device)
            _default[device] = ctx
        return ctx
