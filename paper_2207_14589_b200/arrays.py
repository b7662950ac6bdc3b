"""Host <-> device block staging for the reference-facing API.

The reference API takes and returns numpy float64 arrays.  Here a numpy
input is cast to fp32 straight into a pinned staging buffer (one host pass),
copied H2D asynchronously, and results come back through pinned memory and
are returned as float64 numpy (API parity).  CUDA tensors pass through
untouched (fp32, contiguous) and results stay on the device.
"""

from __future__ import annotations

import numpy as np
import torch

__all__ = ["as_device_block", "from_device_block", "is_device_array"]


def is_device_array(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def as_device_block(x, device):
    """Return ``(fp32 contiguous CUDA tensor, back)``; ``back`` tells
    :func:`from_device_block` how to hand the result back."""
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            t = x
            if t.device != torch.device(device):
                t = t.to(device)
            if t.dtype != torch.float32:
                t = t.to(torch.float32)
            return t.contiguous(), ("torch", None)
        back = ("torch_cpu", x.dtype)
        if x.dtype == torch.float32 and x.is_pinned() and x.is_contiguous():
            return x.to(device, non_blocking=True), back  # zero-copy staging
        host = x.detach().numpy()
    else:
        host = np.asarray(x)
        back = ("numpy", None)
    if host.dtype == object:
        raise TypeError("object arrays are not supported")
    pinned = torch.empty(host.shape, dtype=torch.float32, pin_memory=True)
    np.copyto(pinned.numpy(), host, casting="unsafe")
    return pinned.to(device, non_blocking=True), back


def from_device_block(y: torch.Tensor, back):
    kind, dtype = back
    if kind == "torch":
        return y
    pinned = torch.empty(y.shape, dtype=torch.float32, pin_memory=True)
    pinned.copy_(y, non_blocking=True)
    torch.cuda.current_stream(y.device).synchronize()
    if kind == "torch_cpu":
        return pinned if dtype in (None, torch.float32) else pinned.to(dtype)
    return pinned.numpy().astype(np.float64)
