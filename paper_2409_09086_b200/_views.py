"""Device views that NumPy consumers can read.

The reference's ``KvCache.keys()`` & co. return NumPy views of the cache
(cache.py:93-108).  The drop-in keeps the cache on the GPU and returns torch
views of it; ``DeviceView`` is such a view that also implements the NumPy
array protocol: ``np.asarray(view)`` (and everything built on it, e.g.
``np.testing``) reads a host copy, while torch operations stay on the device
and slicing returns further views."""

from __future__ import annotations

import numpy as np
import torch


class DeviceView(torch.Tensor):
    def copy(self) -> "DeviceView":
        """ndarray.copy(): an independent copy (stays on the device)."""
        return self.clone()

    def __array__(self, dtype=None, copy=None):
        a = torch.Tensor.numpy(self.detach().as_subclass(torch.Tensor).cpu())
        return a if dtype is None else a.astype(dtype, copy=False)


def view(t: torch.Tensor) -> DeviceView:
    return t.as_subclass(DeviceView)
