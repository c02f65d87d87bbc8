"""Host/device plumbing shared by the public API.

numpy in -> numpy out (float64 inputs are rounded to fp32 for the device and
the result is returned as float64, matching the reference's dtype; float32 /
float16 arrays keep their dtype); CUDA tensors in -> CUDA tensors out, zero
copy.  torch is only plumbing here: device memory, streams, copies.
"""

from __future__ import annotations

import numpy as np

from . import _native as nat


def torch():
    import torch as _t
    return _t


def _storage(dtype):
    t = torch()
    if dtype in (t.float16, np.float16):
        return t.float16, nat.SKC_F16
    return t.float32, nat.SKC_F32


class Image:
    """An image argument resolved to a contiguous CUDA tensor (B, H, W, C)."""

    def __init__(self, img, batched: bool = False, device=None):
        t = torch()
        self.kind = "torch" if isinstance(img, t.Tensor) else "numpy"
        self.cpu_tensor = False
        if self.kind == "numpy":
            arr = np.asarray(img)
            if not np.issubdtype(arr.dtype, np.floating):
                arr = arr.astype(np.float64)
            self.np_dtype = arr.dtype
            host = arr.astype(np.float16 if arr.dtype == np.float16 else np.float32, copy=False)
            dev = t.device("cuda", t.cuda.current_device()) if device is None else t.device(device)
            ten = t.from_numpy(np.ascontiguousarray(host)).to(dev, non_blocking=False)
        else:
            ten = img
            self.cpu_tensor = not ten.is_cuda
            if not ten.is_cuda:
                dev = t.device("cuda", t.cuda.current_device()) if device is None else t.device(device)
                ten = ten.to(dev, non_blocking=ten.is_pinned())
            if ten.dtype not in (t.float32, t.float16):
                ten = ten.to(t.float32)
            ten = ten.contiguous()
        self.orig_ndim = ten.dim()
        if batched:
            if ten.dim() == 3:
                ten = ten.unsqueeze(-1)
            if ten.dim() != 4:
                raise ValueError(f"batched images must be (B, H, W) or (B, H, W, C), got {tuple(ten.shape)}")
        else:
            if ten.dim() == 2:
                ten = ten.unsqueeze(-1)
            if ten.dim() != 3:
                raise ValueError(f"image must be (H, W) or (H, W, C), got {tuple(ten.shape)}")
            ten = ten.unsqueeze(0)
        self.batched = batched
        self.tensor = ten
        self.dtype_id = nat.SKC_F16 if ten.dtype == t.float16 else nat.SKC_F32

    @property
    def dims(self):
        b, h, w, c = self.tensor.shape
        return int(b), int(h), int(w), int(c)

    def empty_like(self, dtype=None):
        t = torch()
        return t.empty_like(self.tensor, dtype=self.tensor.dtype if dtype is None else dtype)

    def restore(self, out, dest=None):
        """Undo the shape/kind normalisation on a result tensor (B, H, W, C).

        `dest` (optional torch tensor, e.g. pinned host memory) receives the
        result with a stream-ordered copy and is returned."""
        if not self.batched:
            out = out[0]
            if self.orig_ndim == 2:
                out = out[..., 0]
        elif self.orig_ndim == 3:
            out = out[..., 0]
        if dest is not None:
            dest.copy_(out.view(dest.shape), non_blocking=True)
            return dest
        if self.kind == "torch":
            return out.cpu() if self.cpu_tensor else out
        res = out.cpu().numpy()
        if self.np_dtype == np.float64:
            res = res.astype(np.float64)
        return res
