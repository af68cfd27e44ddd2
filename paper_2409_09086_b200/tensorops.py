"""Drop-in for the reference's dense single-query numerics (tensorops.py).

``softmax_row``, ``attn_probs``, ``weighted_sum`` and ``rope_apply``
(reference tensorops.py:26-111) validate their inputs on the host exactly as
the reference does (same ValueError conditions) and compute on the device
(``skv_softmax_row`` / ``skv_attn_probs`` / ``skv_weighted_sum`` /
``skv_rope_apply``, csrc/tensorops.cu).  Host inputs give NumPy float32
results like the reference; CUDA tensors stay on the device.

``attend(keys, values, q)`` is ``Session._attend`` (reference engine.py:235-246)
-- equivalently ``tensorops.attn_probs`` + ``weighted_sum`` per head
(tensorops.py:86-111) -- run by the K1 split-KV decode kernel plus the probability
fold kernel.  Head dims below 64 (or between 64 and 128) are zero-padded to the
kernel's 64/128: padding adds exact zeros to every dot product and output.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import check


def attend(keys, values, q):
    """keys/values (H, n, D), q (H, D) -> probs (H, n) f32, out (H, D) f32."""
    host = not (isinstance(keys, torch.Tensor) and keys.is_cuda)
    k = torch.as_tensor(np.asarray(keys, np.float32) if not isinstance(keys, torch.Tensor) else keys)
    v = torch.as_tensor(np.asarray(values, np.float32) if not isinstance(values, torch.Tensor) else values)
    qq = torch.as_tensor(np.asarray(q, np.float32) if not isinstance(q, torch.Tensor) else q)
    k, v, qq = (t.to(device="cuda", dtype=torch.float32) for t in (k, v, qq))
    if k.ndim != 3 or k.shape[1] == 0:
        raise ValueError("keys must be a non-empty (heads, n, dim) block")
    H, n, D = k.shape
    if tuple(v.shape) != (H, n, D) or tuple(qq.shape) != (H, D):
        raise ValueError("shape mismatch between keys, values and q")
    Dp = 64 if D <= 64 else 128
    if D > 128:
        raise ValueError("head_dim > 128 is not supported by the device kernel")
    if Dp != D:
        pad = (0, Dp - D)
        k = torch.nn.functional.pad(k, pad)
        v = torch.nn.functional.pad(v, pad)
        qq = torch.nn.functional.pad(qq, pad)
    k, v, qq = k.contiguous(), v.contiguous(), qq.contiguous()
    probs = torch.empty((H, n), dtype=torch.float32, device="cuda")
    out = torch.empty((H, Dp), dtype=torch.float32, device="cuda")
    # the kernel scales by 1/sqrt(kernel head_dim); pre-scale q so the logits use 1/sqrt(D)
    if Dp != D:
        qq = qq * torch.tensor(np.float32(np.sqrt(Dp) / np.sqrt(D)), device="cuda")
    check(_lib.load().skv_attend(ctypes.c_void_p(k.data_ptr()), ctypes.c_void_p(v.data_ptr()), H, n, Dp, n * Dp,
                                 ctypes.c_void_p(qq.data_ptr()), ctypes.c_void_p(probs.data_ptr()),
                                 ctypes.c_void_p(out.data_ptr()),
                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    out = out[:, :D]
    if host:
        return probs.cpu().numpy(), out.cpu().numpy()
    return probs, out


def _vec(x, name="vector"):
    """The reference's _as_f32_vector (tensorops.py:17-23): 1-D, non-empty, finite."""
    if isinstance(x, torch.Tensor):
        t = x.detach().to(torch.float32)
        if t.ndim != 1 or t.numel() == 0:
            raise ValueError(f"{name} must be a non-empty 1-D vector")
        if not bool(torch.isfinite(t).all()):
            raise ValueError(f"{name} contains non-finite entries")
        return t.to("cuda").contiguous(), t.is_cuda
    v = np.asarray(x, dtype=np.float32)
    if v.ndim != 1 or v.size == 0:
        raise ValueError(f"{name} must be a non-empty 1-D vector")
    if not np.all(np.isfinite(v)):
        raise ValueError(f"{name} contains non-finite entries")
    return torch.from_numpy(np.ascontiguousarray(v)).to("cuda"), False


def _mat(x):
    if isinstance(x, torch.Tensor):
        return x.detach().to(device="cuda", dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32))).to("cuda")


def _out(t, on_device):
    return t if on_device else t.cpu().numpy()


def _sh():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


def softmax_row(logits):
    """Numerically stable softmax of one row (tensorops.py:26-35)."""
    _lib.require_cuda()
    z, dev = _vec(logits, "logits")
    out = torch.empty_like(z)
    check(_lib.load().skv_softmax_row(_p(z), z.numel(), _p(out), _sh()))
    return _out(out, dev)


def attn_probs(query, keys, scale=None):
    """softmax_row((keys @ query) * scale), scale = 1/sqrt(dim) by default (tensorops.py:86-102)."""
    _lib.require_cuda()
    q, dev = _vec(query, "query")
    k = _mat(keys)
    if k.ndim != 2 or k.shape[0] == 0:
        raise ValueError("keys must be a non-empty sequence of vectors")
    if k.shape[1] != q.numel():
        raise ValueError(f"key dim {k.shape[1]} does not match query dim {q.numel()}")
    if scale is None:
        scale = 1.0 / np.sqrt(q.numel())
    if scale <= 0:
        raise ValueError("scale must be positive")
    out = torch.empty(k.shape[0], dtype=torch.float32, device="cuda")
    check(_lib.load().skv_attn_probs(_p(q), _p(k), k.shape[0], k.shape[1], ctypes.c_float(np.float32(scale)),
                                     _p(out), _sh()))
    return _out(out, dev)


def weighted_sum(probs, values):
    """sum_i probs[i] * values[i] (tensorops.py:105-111)."""
    _lib.require_cuda()
    p, dev = _vec(probs, "probs")
    v = _mat(values)
    if v.ndim != 2 or v.shape[0] != p.numel():
        raise ValueError(f"expected {p.numel()} value vectors, got shape {tuple(v.shape)}")
    out = torch.empty(v.shape[1], dtype=torch.float32, device="cuda")
    if v.shape[1] > 0:
        check(_lib.load().skv_weighted_sum(_p(p), _p(v), v.shape[0], v.shape[1], _p(out), _sh()))
    return _out(out, dev)


def rope_apply(v, position: int, base: float = 10000.0):
    """Rotate consecutive pairs by position * base^(-2i/dim) (tensorops.py:38-64)."""
    _lib.require_cuda()
    x, dev = _vec(v, "v")
    if x.numel() % 2 != 0:
        raise ValueError("rope_apply requires an even-dimensional vector")
    if position < 0:
        raise ValueError("position must be non-negative")
    if base <= 1.0:
        raise ValueError("base must be > 1")
    out = torch.empty_like(x)
    check(_lib.load().skv_rope_apply(_p(x), x.numel(), int(position), float(base), _p(out), _sh()))
    return _out(out, dev)
