"""ctypes binding of libhiermoe.so (the C-ABI in include/hiermoe.h).

The product path has no CPU fallback: if the library or a CUDA device is
missing, every call raises.  Status codes map to ValueError (< 0, invalid
argument -- the reference's error family, e.g. traffic.py:62-63) and
RuntimeError (> 0, CUDA error).
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int32, c_int64, c_size_t, c_void_p
from pathlib import Path

import torch

LIB_PATH = Path(__file__).resolve().parent / "libhiermoe.so"
# developer A/B runs only: HM_LIB=<path> loads another build of the same library
if os.environ.get("HM_LIB"):
    LIB_PATH = Path(os.environ["HM_LIB"])

_lib = None

_SIGS = {
    "hm_last_error": (ctypes.c_char_p, []),
    "hm_version": (c_int32, []),
    "hm_launch_count": (ctypes.c_uint64, []),
    "hm_mask_pack": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    "hm_mask_unpack": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_void_p]),
    "hm_ids_to_bits": (c_int32, [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p, c_void_p,
                                 c_void_p]),
    "hm_level_counts": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_int32, c_void_p, c_void_p,
                                  c_void_p, c_int32, c_void_p]),
    "hm_scan_workspace": (c_size_t, [c_int64]),
    "hm_scan_i64": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "hm_propagate_count": (c_int32, [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p]),
    "hm_propagate_emit": (c_int32, [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p,
                                    c_void_p, c_void_p, c_void_p, c_void_p]),
    "hm_swap_partials": (c_int32, [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "hm_swap_tensor": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int32,
                                 c_int32, c_void_p, c_void_p]),
    "hm_swap_cost": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                               c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                               c_int32, c_int32, c_int64, c_double, c_void_p, c_int32,
                               c_void_p, c_void_p, c_void_p]),
    "hm_swap_select": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_void_p]),
    "hm_time_model": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_int64, c_void_p,
                                c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                c_void_p, c_void_p]),
    "hm_np_pow": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "hm_smooth_max_rows": (c_int32, [c_void_p, c_int64, c_int32, c_double, c_void_p, c_void_p]),
    "hm_world_create": (c_int32, [c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, c_int32,
                                  c_int64, c_int64, c_int32, c_int32, POINTER(c_void_p)]),
    "hm_relay_ids": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "hm_world_destroy": (c_int32, [c_void_p]),
    "hm_world_ipc_handle_size": (c_int64, []),
    "hm_world_ipc_handle": (c_int32, [c_void_p, c_void_p]),
    "hm_world_open_peers": (c_int32, [c_void_p, c_void_p]),
    "hm_world_buffer": (c_int32, [c_void_p, c_int32, c_int32, POINTER(c_void_p), POINTER(c_int64)]),
    "hm_world_info": (c_int32, [c_void_p, c_void_p]),
    "hm_world_barrier": (c_int32, [c_void_p, c_void_p]),
    "hm_world_set_option": (c_int32, [c_void_p, c_int32, c_int32]),
    "hm_memcpy": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p]),
    "hm_world_set_timing": (c_int32, [c_void_p, c_int32]),
    "hm_world_timings": (c_int32, [c_void_p, c_void_p, c_int32]),
    "hm_route_topk": (c_int32, [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_int32, c_void_p,
                                c_void_p, c_void_p, c_void_p]),
    "hm_route_set_option": (c_int32, [c_int32]),
    "hm_route_group": (c_int32, [c_void_p, c_int64, c_int32, c_int32, c_int32, c_int32, c_void_p,
                                 ctypes.c_float, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "hm_dispatch": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_void_p]),
    "hm_ffn_set_option": (c_int32, [c_int32, c_int32]),
    "hm_dispatch_plan": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_void_p]),
    "hm_dispatch_push": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_void_p]),
    "hm_expand": (c_int32, [c_void_p, c_void_p]),
    "hm_dispatch_meta": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "hm_experts_overlap": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_int32,
                                     c_void_p, c_void_p, c_void_p]),
    "hm_dispatch_grad": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_void_p,
                                   c_void_p]),
    "hm_combine_grad": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_void_p]),
    "hm_bf16_to_f32": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p]),
    "hm_gate_backward": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int32,
                                   c_int32, c_int32, c_float, c_void_p, c_int32, c_void_p]),
    "hm_gemm_f32": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_int32, c_int32, c_int32,
                              c_void_p, c_int64, c_void_p]),
    "hm_wgrad_f32": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_int32, c_int32,
                               c_void_p, c_int64, c_int32, c_void_p]),
    "hm_wgrad_f32_scratch_bytes": (c_int64, [c_int64, c_int32, c_int32]),
    "hm_gemm_add_bf16": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_int32, c_int32,
                                   c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    "hm_wgrad_f32_split": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_int32, c_int32,
                                     c_void_p, c_int64, c_int32, c_void_p, c_int64, c_void_p]),
    "hm_sum_to_bf16": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    "hm_combine": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_void_p]),
    "hm_combine_add": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_void_p,
                                 c_void_p]),
    "hm_grouped_gemm_kn": (c_int32, [c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_int32,
                                     c_int32, c_void_p, c_int64, c_void_p]),
    "hm_grouped_gemm": (c_int32, [c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_int32,
                                  c_int32, c_int32, c_void_p, c_int64, c_void_p]),
    "hm_store_create": (c_int32, [c_int32, c_int32, c_int32, c_void_p, c_int32, POINTER(c_void_p)]),
    "hm_store_destroy": (c_int32, [c_void_p]),
    "hm_store_ipc_handle": (c_int32, [c_void_p, c_void_p]),
    "hm_store_open_peers": (c_int32, [c_void_p, c_void_p]),
    "hm_store_array": (c_int32, [c_void_p, c_int32, POINTER(c_void_p)]),
    "hm_store_status": (c_int32, [c_void_p, c_void_p]),
    "hm_migrate": (c_int32, [c_void_p, c_int32, c_int32, c_void_p]),
    "hm_expert_ffn_backward": (c_int32, [c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_void_p,
                                         c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p,
                                         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                         c_void_p]),
    "hm_expert_ffn": (c_int32, [c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_void_p,
                                c_int32, c_int32, c_void_p, c_void_p, c_void_p]),
    "hm_expert_ffn_save": (c_int32, [c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_void_p,
                                     c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    "hm_expert_ffn_gather": (c_int32, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int32,
                                       c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p,
                                       c_void_p, c_void_p]),
    "hm_expert_ffn_backward_gather": (c_int32, [c_void_p, c_int64, c_void_p, c_int64, c_void_p,
                                                c_int32, c_void_p, c_void_p, c_void_p, c_int32,
                                                c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                                c_void_p, c_void_p, c_void_p, c_void_p, c_int32,
                                                c_void_p]),
    "hm_expert_ffn_multi": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_int32,
                                      c_void_p, c_int32, c_void_p, c_void_p, c_int32, c_int32,
                                      c_void_p, c_void_p, c_void_p, c_void_p]),
    "hm_expert_ffn_groups": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_int32,
                                       c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_void_p,
                                       c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_int32,
                                       c_void_p]),
    "hm_expert_ffn_backward_multi": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_int64,
                                               c_int32, c_void_p, c_int32, c_void_p, c_void_p,
                                               c_void_p, c_int32, c_int32, c_void_p, c_void_p,
                                               c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                               c_void_p, c_int32, c_int32, c_void_p]),
    "hm_expert_ffn_backward_saved": (c_int32, [c_void_p, c_int64, c_void_p, c_int32, c_void_p,
                                               c_void_p, c_void_p, c_int32, c_int32, c_void_p,
                                               c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                               c_void_p, c_void_p, c_int32, c_void_p]),
}


def exported_symbols() -> list[str]:
    return sorted(_SIGS)


def load(require_cuda: bool = True):
    """Load the library (and, for compute calls, insist on a CUDA device)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               f"(there is no CPU fallback)")
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_cuda and not torch.cuda.is_available():
        raise RuntimeError("paper_2508_09591_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return _lib


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    msg = (_lib.hm_last_error() or b"").decode(errors="replace")
    if status < 0:
        raise ValueError(msg or f"{what}: invalid argument ({status})")
    raise RuntimeError(f"{what}: {msg or 'CUDA error'} ({status})")


def call(name: str, *args) -> None:
    lib = load()
    check(getattr(lib, name)(*args), name)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def host_array(ctype, values):
    arr = (ctype * max(1, len(values)))(*values)
    return arr
