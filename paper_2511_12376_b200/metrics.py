"""Quality metrics computed on the device.

`precision_device` is the reduction behind precision_report
(reference quantizer.py:280-296): MSE over all elements and MRE over the
elements with |o| > 1e-12, accumulated in float64 by csrc/quant.cu.
"""

from __future__ import annotations

import torch

from . import _lib
from . import _runtime as rt


def precision_device(original: torch.Tensor, restored: torch.Tensor) -> dict:
    o = original.reshape(-1).contiguous()
    r = restored.reshape(-1).contiguous()
    if o.dtype != torch.float32 or r.dtype != torch.float32 or o.numel() != r.numel():
        raise ValueError("precision_device needs two float32 tensors of equal size")
    acc = torch.empty(3, dtype=torch.float64, device=o.device)
    _lib.check(rt.lib().bsnp_precision_report(o.data_ptr(), r.data_ptr(), o.numel(),
                                              acc.data_ptr(), rt.stream_ptr(o.device)),
               "bsnp_precision_report")
    sse, rel, cnt = acc.cpu().tolist()
    n = o.numel()
    return {"mre": rel / cnt if cnt else 0.0, "mse": sse / n if n else 0.0}
