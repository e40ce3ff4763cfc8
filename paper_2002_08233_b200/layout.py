"""Object wrapper over the C-ABI (same operations, owned handle)."""
from __future__ import annotations

import numpy as np

from . import _bl


class BatchLayout:
    """Owns one bl_ctx (the device CSR of G)."""

    def __init__(self, n: int, rowptr, colidx):
        self.n = int(n)
        self.h = _bl.bl_create(self.n, rowptr, colidx)

    # -- host path: numpy in, numpy out (H2D + kernel + D2H inside bl_layout)
    def layout(self, xy, **params):
        xy = np.ascontiguousarray(np.asarray(xy, dtype=np.float32).reshape(self.n, 2)).copy()
        done = _bl.bl_layout(self.h, xy, _bl.bl_params_default(**params))
        return xy, done

    def _check_device_xy(self, d_xy):
        import torch
        if not (isinstance(d_xy, torch.Tensor) and d_xy.is_cuda and d_xy.dtype == torch.float32
                and d_xy.is_contiguous() and d_xy.numel() == 2 * self.n):
            raise TypeError("d_xy must be a contiguous float32 CUDA tensor with 2n elements")

    # -- device path: torch CUDA float32 (n, 2) tensor updated in place
    def layout_device(self, d_xy, stream=None, **params):
        import torch
        self._check_device_xy(d_xy)
        if stream is None:
            stream = torch.cuda.current_stream(d_xy.device)
        _bl.bl_layout_device(self.h, d_xy, _bl.bl_params_default(**params), stream)

    def energy(self, trace_len: int = 0):
        return _bl.bl_energy(self.h, trace_len)

    def forces(self, d_xy, first: int = 0, count: int | None = None, stream=None, **params):
        import torch
        self._check_device_xy(d_xy)
        if count is None:
            count = self.n - first
        out = torch.empty((max(count, 1), 2), dtype=torch.float32, device=d_xy.device)
        if stream is None:
            stream = torch.cuda.current_stream(d_xy.device)
        _bl.bl_forces(self.h, d_xy, first, count, out, _bl.bl_params_default(**params), stream)
        return out[:count]

    def close(self):
        if self.h:
            _bl.bl_destroy(self.h)
            self.h = 0

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
