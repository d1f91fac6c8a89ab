"""Standalone device gadgets (reference pkg/src/obtree/gadgets.py, oaa.py, rss.py).

Thin wrappers over the C ABI's single-gadget entry points, on
component-major device tensors: arithmetic shares ``[3, n]`` int64 (uint64
bits), boolean shares ``[3, n]`` uint8.  Training and inference use the same
per-lane device code fused into larger kernels; these entry points exist for
callers that compose their own protocols and for the parity tests.
"""

from __future__ import annotations

import ctypes

from . import _native
from .shares import ptr


def _stream(t, stream):
    torch = _native.require_cuda()
    s = stream if stream is not None else torch.cuda.current_stream(t.device)
    return ctypes.c_void_p(s.cuda_stream)


def _n(x) -> int:
    if x.dim() < 2 or x.shape[0] != 3:
        raise ValueError("share tensors are component-major [3, ...]")
    return int(x[0].numel())


def mul(width, x, y, keys, op, stream=None):
    """PartyEngine.mul (rss.py:386-400)."""
    torch = _native.require_cuda()
    z = torch.empty_like(x)
    _native.check(_native.load().gt_mul(width, ptr(x), ptr(y), ptr(z), _n(x), ctypes.byref(keys), op, _stream(x, stream)))
    return z


def eq(width, x, y=None, y_pub=None, *, keys, op, stream=None):
    """eq (gadgets.py:120-130): [x == y] boolean shares."""
    torch = _native.require_cuda()
    out = torch.empty((3, _n(x)), dtype=torch.uint8, device=x.device)
    _native.check(_native.load().gt_eq(width, ptr(x), ptr(y), ptr(y_pub), ptr(out), _n(x), ctypes.byref(keys), op,
                                       _stream(x, stream)))
    return out


def lt(width, x, y=None, y_pub=None, *, keys, op, stream=None):
    """lt (gadgets.py:188-216): [x < y] unsigned."""
    torch = _native.require_cuda()
    out = torch.empty((3, _n(x)), dtype=torch.uint8, device=x.device)
    _native.check(_native.load().gt_lt(width, ptr(x), ptr(y), ptr(y_pub), ptr(out), _n(x), ctypes.byref(keys), op,
                                       _stream(x, stream)))
    return out


def b2a(width, bits, *, keys, op, stream=None):
    """b2a (gadgets.py:223-231)."""
    torch = _native.require_cuda()
    out = torch.empty((3, bits.shape[1]), dtype=torch.int64, device=bits.device)
    _native.check(_native.load().gt_b2a(width, ptr(bits), ptr(out), int(bits.shape[1]), ctypes.byref(keys), op,
                                        _stream(bits, stream)))
    return out


def select_share(width, w1, w2, cond, *, keys, op, stream=None):
    """select_share (gadgets.py:238-253); payload [3, n_cond * group]."""
    torch = _native.require_cuda()
    n_cond = int(cond.shape[1])
    total = _n(w1)
    if n_cond == 0 or total % n_cond:
        raise ValueError("payload size must be a multiple of condition size")
    out = torch.empty_like(w1)
    _native.check(_native.load().gt_select(width, ptr(w1), ptr(w2), ptr(cond), ptr(out), n_cond, total // n_cond,
                                           ctypes.byref(keys), op, _stream(w1, stream)))
    return out


def truncate(width, x, k, *, keys, op, stream=None):
    """truncate (gadgets.py:260-288): exact floor(x / 2^k)."""
    torch = _native.require_cuda()
    out = torch.empty_like(x)
    _native.check(_native.load().gt_truncate(width, ptr(x), ptr(out), _n(x), int(k), ctypes.byref(keys), op,
                                             _stream(x, stream)))
    return out


def division(width, p, q, tau, *, keys, op, stream=None):
    """division (gadgets.py:310-349)."""
    torch = _native.require_cuda()
    out = torch.empty_like(p)
    _native.check(_native.load().gt_division(width, ptr(p), ptr(q), ptr(out), _n(p), int(tau), ctypes.byref(keys), op,
                                             _stream(p, stream)))
    return out


def argmin_masked(width, scores, avail, worst, *, keys, op, stream=None):
    """argmin_masked (gadgets.py:366-401): scores [3, n, m], avail [3, n, m] bits."""
    torch = _native.require_cuda()
    if scores.dim() != 3 or tuple(scores.shape) != tuple(avail.shape):
        raise ValueError("scores and mask must be matching 2-d arrays")
    n, m = int(scores.shape[1]), int(scores.shape[2])
    out = torch.empty((3, n), dtype=torch.int64, device=scores.device)
    lib = _native.load()
    scratch = torch.empty(int(lib.gt_argmin_scratch_words(n, m)), dtype=torch.int64, device=scores.device)
    _native.check(lib.gt_argmin(width, ptr(scores), ptr(avail), ptr(out), n, m, int(worst), ctypes.byref(keys), op,
                                ptr(scratch), _stream(scores, stream)))
    return out


def oaa(width, table, idx, *, keys, op, stream=None):
    """oaa (oaa.py:20-35)."""
    torch = _native.require_cuda()
    out = torch.empty_like(idx)
    _native.check(_native.load().gt_oaa(width, ptr(table), int(table.shape[1]), ptr(idx), ptr(out), _n(idx),
                                        ctypes.byref(keys), op, _stream(idx, stream)))
    return out


def row_lookup(width, rows, idx, *, keys, op, stream=None):
    """row_lookup (oaa.py:38-55): rows [3, n, m]."""
    torch = _native.require_cuda()
    if rows.dim() != 3:
        raise ValueError("rows must be two-dimensional")
    if int(rows.shape[1]) != _n(idx):
        raise ValueError("one index per row required")
    out = torch.empty_like(idx)
    _native.check(_native.load().gt_row_lookup(width, ptr(rows), int(rows.shape[2]), ptr(idx), ptr(out), _n(idx),
                                               ctypes.byref(keys), op, _stream(idx, stream)))
    return out
