"""Expert store + peer-to-peer migration of swapped experts (K11).

``ExpertStore`` keeps every local slot's expert state (bf16 weights, fp32
master weights, Adam moments) as slot-major torch views over one CUDA-IPC
region; ``migrate(r, c)`` applies a planned slot swap (apply_swap,
swap.py:255-259) to the physical state, moving bytes over NVLink when the two
slots live on different GPUs.  All GPUs call it with the same pair.
"""

from __future__ import annotations

import ctypes
import math

import torch

from . import _lib
from .layer import exchange_handles

_ESZ = {torch.bfloat16: 2, torch.float32: 4, torch.float16: 2, torch.int32: 4, torch.uint8: 1}


class ExpertStore:
    def __init__(self, slots_per_gpu: int, arrays: dict, gpus: int = 1, gpu_index: int = 0,
                 group=None):
        """arrays: name -> (per-slot shape, dtype)."""
        lib = _lib.load()
        self.names = list(arrays)
        self.shapes = {k: tuple(v[0]) for k, v in arrays.items()}
        self.dtypes = {k: v[1] for k, v in arrays.items()}
        slices = [math.prod(self.shapes[k]) * _ESZ[self.dtypes[k]] for k in self.names]
        sl = (ctypes.c_int64 * len(slices))(*slices)
        h = ctypes.c_void_p()
        _lib.check(lib.hm_store_create(gpus, gpu_index, slots_per_gpu, sl, len(slices),
                                       ctypes.byref(h)), "hm_store_create")
        self._h = h
        self.slots_per_gpu, self.gpus, self.gpu_index = slots_per_gpu, gpus, gpu_index
        if gpus > 1:
            import torch.distributed as dist
            n = int(lib.hm_world_ipc_handle_size())
            mine = (ctypes.c_uint8 * n)()
            _lib.check(lib.hm_store_ipc_handle(h, mine), "hm_store_ipc_handle")
            allh = exchange_handles(bytes(mine), gpu_index, gpus, group)
            buf = (ctypes.c_uint8 * len(allh)).from_buffer_copy(allh)
            _lib.check(lib.hm_store_open_peers(h, buf), "hm_store_open_peers")
            dist.barrier(group=group)
        self.views = {}
        for i, k in enumerate(self.names):
            p = ctypes.c_void_p()
            _lib.check(lib.hm_store_array(h, i, ctypes.byref(p)), "hm_store_array")
            self.views[k] = _wrap(p.value, (slots_per_gpu, *self.shapes[k]), self.dtypes[k])

    def __getitem__(self, name: str) -> torch.Tensor:
        return self.views[name]

    def migrate(self, slot_r: int, slot_c: int) -> None:
        _lib.call("hm_migrate", self._h, int(slot_r), int(slot_c), _lib.stream_ptr())

    def check_status(self) -> None:
        out = (ctypes.c_int32 * 4)()
        _lib.call("hm_store_status", self._h, out)
        if out[0]:
            raise RuntimeError(f"ExpertStore: device status {out[0]} (pair barrier timeout)")

    def bytes_per_slot(self) -> int:
        return sum(math.prod(self.shapes[k]) * _ESZ[self.dtypes[k]] for k in self.names)

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and _lib._lib is not None:
            self.views = {}
            _lib._lib.hm_store_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _Raw:
    """Minimal __cuda_array_interface__ exporter for a raw device pointer."""

    _TYPESTR = {torch.bfloat16: "<f2", torch.float32: "<f4", torch.float16: "<f2",
                torch.int32: "<i4", torch.uint8: "|u1"}

    def __init__(self, ptr: int, shape, dtype):
        # bf16 is exported as int16 and reinterpreted (the interface has no bf16)
        ts = "<i2" if dtype == torch.bfloat16 else self._TYPESTR[dtype]
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": tuple(shape),
                                         "typestr": ts, "version": 3, "strides": None}


def _wrap(ptr: int, shape, dtype) -> torch.Tensor:
    t = torch.as_tensor(_Raw(ptr, shape, dtype), device="cuda")
    return t.view(dtype) if dtype == torch.bfloat16 else t
