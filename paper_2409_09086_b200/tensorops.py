"""Drop-in for the attention half of the reference numerics.

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
