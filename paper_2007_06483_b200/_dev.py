"""Host<->device plumbing shared by the operator modules.

Every public operator accepts either numpy arrays (the reference's currency)
or torch CUDA tensors.  numpy in -> numpy out (after one device round trip);
CUDA tensor in -> CUDA tensor out (no host copies).  Device memory comes from
torch's caching allocator; kernels run on torch's current stream.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def torch_mod():
    return _lib.require_cuda()


def is_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def shape_of(x):
    return tuple(x.shape) if hasattr(x, "shape") else None


def ndim_of(x):
    return len(x.shape) if hasattr(x, "shape") else -1


def is_u8(x) -> bool:
    if isinstance(x, np.ndarray):
        return x.dtype == np.uint8
    if is_tensor(x):
        import torch

        return x.dtype == torch.uint8
    return False


def dtype_name(x) -> str:
    return str(getattr(x, "dtype", type(x).__name__))


def to_device(x, dtype=None):
    """Contiguous CUDA tensor holding x (numpy or torch); no copy if already so."""
    torch = torch_mod()
    if isinstance(x, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(x))
        if t.numel() * t.element_size() >= (1 << 20):
            t = t.pin_memory()
            t = t.to("cuda", non_blocking=True)
        else:
            t = t.to("cuda")
    elif is_tensor(x):
        t = x if x.is_cuda else x.to("cuda")
        t = t.contiguous()
    else:
        t = torch.as_tensor(np.asarray(x)).to("cuda")
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t


def like_input(t, original):
    """Return t as numpy if `original` was numpy, else as the CUDA tensor."""
    if isinstance(original, np.ndarray):
        return t.cpu().numpy()
    return t


def ptr(t) -> int:
    return int(t.data_ptr())


def stream() -> int:
    import torch

    return int(torch.cuda.current_stream().cuda_stream)


def readback_u64(t) -> int:
    """Host value of a 1-element device counter (synchronises the stream)."""
    return int(t.view(torch_mod().int64).item())
