"""ctypes binding of the in-tree sm_100a library ``libgtree_b200.so``.

The library is the product: every share computation of the training and
inference path runs in its CUDA kernels (include/gtree_b200.h).  There is no
CPU fallback -- if the library is missing or no CUDA device is present, the
entry points raise instead of computing anything on the host.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgtree_b200.so")

GT_OK, GT_EINVAL, GT_ECUDA = 0, 1, 2
ABI_VERSION = 2


class ProtocolError(RuntimeError):
    """Device/launch failure inside a protocol run (reference exit code 2,
    cli.py:53-56: ShareError/MaterialError/TransportError class)."""


class gt_key(ctypes.Structure):
    _fields_ = [("k0", ctypes.c_uint32), ("k1", ctypes.c_uint32)]


class gt_keys(ctypes.Structure):
    _fields_ = [("dealer", gt_key), ("pair", gt_key * 3)]


class gt_train_cfg(ctypes.Structure):
    _fields_ = [
        ("depth", ctypes.c_int32),
        ("tau", ctypes.c_int32),
        ("score_width", ctypes.c_int32),
        ("nf", ctypes.c_int32),
        ("policy", ctypes.c_int32),
        ("heuristic", ctypes.c_int32),
        ("n_total", ctypes.c_uint64),
        ("n_local", ctypes.c_uint64),
        ("sample_base", ctypes.c_uint64),
        ("count_reshare", ctypes.c_int32),
        ("count_engine", ctypes.c_int32),
    ]


class gt_train_profile(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_uint32), ("n_prods", ctypes.c_uint32), ("n_partition", ctypes.c_uint32),
                ("n_count", ctypes.c_uint32), ("n_node_hc", ctypes.c_uint32), ("n_node_finish", ctypes.c_uint32),
                ("ms_prods", ctypes.c_float), ("ms_partition", ctypes.c_float), ("ms_count", ctypes.c_float),
                ("ms_node_hc", ctypes.c_float), ("ms_node_finish", ctypes.c_float), ("ms_total", ctypes.c_float),
                ("n_count_lanes", ctypes.c_uint32), ("n_count_contract", ctypes.c_uint32),
                ("ms_count_lanes", ctypes.c_float), ("ms_count_contract", ctypes.c_float)]


ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p)
HEURISTIC_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)

_u64p = ctypes.c_void_p
_SIGS = {
    "gt_abi_version": (ctypes.c_int, []),
    "gt_last_error": (ctypes.c_char_p, []),
    "gt_mul": (ctypes.c_int, [ctypes.c_int, _u64p, _u64p, _u64p, ctypes.c_uint64, ctypes.POINTER(gt_keys),
                              ctypes.c_uint32, ctypes.c_void_p]),
    "gt_eq": (ctypes.c_int, [ctypes.c_int, _u64p, _u64p, _u64p, _u64p, ctypes.c_uint64, ctypes.POINTER(gt_keys),
                             ctypes.c_uint32, ctypes.c_void_p]),
    "gt_lt": (ctypes.c_int, [ctypes.c_int, _u64p, _u64p, _u64p, _u64p, ctypes.c_uint64, ctypes.POINTER(gt_keys),
                             ctypes.c_uint32, ctypes.c_void_p]),
    "gt_b2a": (ctypes.c_int, [ctypes.c_int, _u64p, _u64p, ctypes.c_uint64, ctypes.POINTER(gt_keys), ctypes.c_uint32,
                              ctypes.c_void_p]),
    "gt_select": (ctypes.c_int, [ctypes.c_int, _u64p, _u64p, _u64p, _u64p, ctypes.c_uint64, ctypes.c_uint64,
                                 ctypes.POINTER(gt_keys), ctypes.c_uint32, ctypes.c_void_p]),
    "gt_truncate": (ctypes.c_int, [ctypes.c_int, _u64p, _u64p, ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(gt_keys),
                                   ctypes.c_uint32, ctypes.c_void_p]),
    "gt_division": (ctypes.c_int, [ctypes.c_int, _u64p, _u64p, _u64p, ctypes.c_uint64, ctypes.c_int,
                                   ctypes.POINTER(gt_keys), ctypes.c_uint32, ctypes.c_void_p]),
    "gt_argmin_scratch_words": (ctypes.c_uint64, [ctypes.c_uint64, ctypes.c_uint64]),
    "gt_argmin": (ctypes.c_int, [ctypes.c_int, _u64p, _u64p, _u64p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                 ctypes.POINTER(gt_keys), ctypes.c_uint32, _u64p, ctypes.c_void_p]),
    "gt_oaa": (ctypes.c_int, [ctypes.c_int, _u64p, ctypes.c_uint64, _u64p, _u64p, ctypes.c_uint64,
                              ctypes.POINTER(gt_keys), ctypes.c_uint32, ctypes.c_void_p]),
    "gt_row_lookup": (ctypes.c_int, [ctypes.c_int, _u64p, ctypes.c_uint64, _u64p, _u64p, ctypes.c_uint64,
                                     ctypes.POINTER(gt_keys), ctypes.c_uint32, ctypes.c_void_p]),
    "gt_train_workspace_bytes": (ctypes.c_uint64, [ctypes.POINTER(gt_train_cfg)]),
    "gt_train_host_workspace_bytes": (ctypes.c_uint64, [ctypes.POINTER(gt_train_cfg)]),
    "gt_train_host": (ctypes.c_int, [ctypes.POINTER(gt_train_cfg), _u64p, _u64p, _u64p, _u64p, _u64p,
                                     ctypes.POINTER(ctypes.c_int32), _u64p, ctypes.c_uint64, ctypes.POINTER(gt_keys),
                                     ALLREDUCE_FN, ctypes.c_void_p, ctypes.c_void_p]),
    "gt_train": (ctypes.c_int, [ctypes.POINTER(gt_train_cfg), _u64p, _u64p, _u64p, _u64p, _u64p,
                                ctypes.POINTER(ctypes.c_int32), ctypes.c_void_p, ctypes.c_uint64,
                                ctypes.POINTER(gt_keys), ALLREDUCE_FN, ctypes.c_void_p, ctypes.c_void_p]),
    "gt_train_ex": (ctypes.c_int, [ctypes.POINTER(gt_train_cfg), _u64p, _u64p, _u64p, _u64p, _u64p,
                                   ctypes.POINTER(ctypes.c_int32), ctypes.c_void_p, ctypes.c_uint64,
                                   ctypes.POINTER(gt_keys), ALLREDUCE_FN, ctypes.c_void_p, HEURISTIC_FN,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(gt_train_profile)]),
    "gt_infer": (ctypes.c_int, [ctypes.c_int, _u64p, _u64p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                _u64p, _u64p, ctypes.POINTER(gt_keys), ctypes.c_void_p]),
    "gt_diag_philox": (ctypes.c_int, [ctypes.c_uint32, ctypes.c_uint32, _u64p, ctypes.c_void_p]),
    "gt_diag_hc_timestamps": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "gt_diag_count_timestamps": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "gt_unpack_pairs": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p), ctypes.c_uint32,
                                       ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p]),
    "gt_party_eq_mask": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "gt_party_eq_planes": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]),
    "gt_party_and_half": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]),
    "gt_party_pack": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
    "gt_party_unpack": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
    "gt_party_b2a_mask": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]),
    "gt_party_b2a_finish": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]),
    "gt_party_select_mul": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]),
    "gt_party_lane_sum": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]),
    "gt_party_slot_step": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]),
    "gt_stage_pairs": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p), ctypes.c_uint64,
                                      ctypes.c_void_p, ctypes.c_int]),
}
EXPORTS = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the C ABI.  Raises ImportError if the library is
    not built -- there is deliberately no fallback path."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: build it with `make` or __graft_entry__.build() "
                              "(the B200 path has no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.gt_abi_version() != ABI_VERSION:
            raise ImportError(f"{path}: ABI version {lib.gt_abi_version()} != {ABI_VERSION}")
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc == GT_OK:
        return
    msg = (load().gt_last_error() or b"").decode(errors="replace")
    if rc == GT_EINVAL:
        raise ValueError(msg)
    raise ProtocolError(msg)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the B200 path needs a CUDA device; there is no CPU fallback")
    return torch
