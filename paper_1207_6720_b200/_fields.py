"""Field conversion between the public API and the device layout.

Public fields follow the reference (1-D float64 arrays of one level) and
extend it with batches:

* ``(n,)``   -- one right-hand side (the reference's shape);
* ``(n, B)`` -- B independent right-hand sides, cells major, RHS fastest.

Inputs may be numpy arrays or torch tensors.  Everything computes on the
CUDA device in that ``[n][B]`` layout; numpy inputs are uploaded and the
result is handed back as numpy, so tests written against the reference read
the same.  Compute dtype: float64 unless every field argument is a float32
torch tensor.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native


@dataclass
class Field:
    t: torch.Tensor  # (n, B) contiguous, on CUDA
    one_d: bool
    numpy: bool

    @property
    def n(self) -> int:
        return self.t.shape[0]

    @property
    def B(self) -> int:
        return self.t.shape[1]

    @property
    def ld(self) -> int:
        return self.t.stride(0)

    def ptr(self) -> int:
        return self.t.data_ptr()


def _device():
    _native.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def length(x) -> int:
    return int(x.shape[0]) if hasattr(x, "shape") else len(x)


def pick_dtype(*xs) -> torch.dtype:
    ts = [x for x in xs if x is not None]
    if ts and all(isinstance(x, torch.Tensor) and x.dtype == torch.float32 for x in ts):
        return torch.float32
    return torch.float64


def to_field(x, dtype: torch.dtype = torch.float64, copy: bool = False) -> Field:
    """Upload / reshape ``x`` into a contiguous (n, B) CUDA tensor."""
    dev = _device()
    was_np = not isinstance(x, torch.Tensor)
    if was_np:
        t = torch.as_tensor(np.asarray(x, dtype=np.float64))
    else:
        t = x
    one_d = t.dim() == 1
    if t.dim() not in (1, 2):
        raise ValueError(f"fields must be (n,) or (n, B), got shape {tuple(t.shape)}")
    t = t.reshape(t.shape[0], 1) if one_d else t
    t = t.to(device=dev, dtype=dtype)
    if copy or not t.is_contiguous():
        t = t.contiguous().clone() if copy else t.contiguous()
    return Field(t, one_d, was_np)


def empty_like_rows(f: Field, rows: int) -> torch.Tensor:
    return torch.empty((rows, f.B), dtype=f.t.dtype, device=f.t.device)


def out(t: torch.Tensor, like: Field):
    """Return ``t`` in the caller's convention (1-D / numpy as given)."""
    r = t[:, 0] if like.one_d else t
    if like.numpy:
        return r.detach().cpu().numpy()
    return r


def same_batch(*fs: Field) -> None:
    B = fs[0].B
    for f in fs[1:]:
        if f.B != B:
            raise ValueError(f"batch sizes differ: {B} vs {f.B}")
