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
    lib = rt.lib()
    ws = rt.workspace(o.device, lib.bsnp_precision_ws_bytes(), "prec")
    _lib.check(lib.bsnp_precision_report(o.data_ptr(), r.data_ptr(), o.numel(), acc.data_ptr(),
                                         ws.data_ptr(), ws.numel(), rt.stream_ptr(o.device)),
               "bsnp_precision_report")
    sse, rel, cnt = acc.cpu().tolist()
    n = o.numel()
    return {"mre": rel / cnt if cnt else 0.0, "mse": sse / n if n else 0.0}


# ---------------------------------------------------------------------------
# Unified quality score (reference metrics.py) on the
# GPU codecs.  normalize / combine / build_report are the reference's host
# arithmetic (same floats); measure() runs the pipeline through
# store.CheckpointEncoder + decode_chain on the device.
# ---------------------------------------------------------------------------

import time
from dataclasses import asdict, dataclass

WEIGHT_TOLERANCE = 1e-9
DEFAULT_WEIGHTS = (0.2, 0.4, 0.4)


class MetricsError(ValueError):
    """metrics.py:31."""


@dataclass(frozen=True)
class QualityWeights:
    """metrics.py:35-48."""

    w1: float  # compression ratio
    w2: float  # speed
    w3: float  # precision

    def __post_init__(self):
        if min(self.w1, self.w2, self.w3) < 0:
            raise MetricsError("weights must be non-negative")
        if abs(self.w1 + self.w2 + self.w3 - 1.0) > WEIGHT_TOLERANCE:
            raise MetricsError(f"weights must sum to 1, got {self.w1 + self.w2 + self.w3}")


@dataclass(frozen=True)
class FactorBounds:
    """metrics.py:51-57: corpus min/max per raw factor."""

    cr: tuple
    cs: tuple
    ps: tuple


@dataclass(frozen=True)
class QualityReport:
    """metrics.py:60-73."""

    cr_raw: float  # original bytes / compressed bytes
    cs_raw: float  # codec wall time minus no-op baseline, seconds
    ps_raw: float  # MSE of restored optimizer states
    cr: float
    cs: float
    ps: float
    q: float
    weights: tuple
    bounds: dict

    def to_dict(self) -> dict:
        return asdict(self)


def normalize(value: float, lo: float, hi: float, higher_is_better: bool) -> float:
    """metrics.py:76-85: min-max score in [0, 1]; a degenerate bound scores 1."""
    if hi < lo:
        raise MetricsError(f"bounds out of order: ({lo}, {hi})")
    if hi == lo:
        return 1.0
    x = (value - lo) / (hi - lo)
    x = min(1.0, max(0.0, x))
    return x if higher_is_better else 1.0 - x


def combine(weights: QualityWeights, cr: float, cs: float, ps: float) -> float:
    """metrics.py:88-89."""
    return weights.w1 * cr + weights.w2 * cs + weights.w3 * ps


def build_report(cr_raw: float, cs_raw: float, ps_raw: float, weights: QualityWeights,
                 bounds: FactorBounds) -> QualityReport:
    """metrics.py:92-110."""
    cr = normalize(cr_raw, *bounds.cr, higher_is_better=True)
    cs = normalize(cs_raw, *bounds.cs, higher_is_better=False)
    ps = normalize(ps_raw, *bounds.ps, higher_is_better=False)
    return QualityReport(cr_raw=cr_raw, cs_raw=cs_raw, ps_raw=ps_raw, cr=cr, cs=cs, ps=ps,
                         q=combine(weights, cr, cs, ps),
                         weights=(weights.w1, weights.w2, weights.w3),
                         bounds={"cr": bounds.cr, "cs": bounds.cs, "ps": bounds.ps})


def _median_time(fn, warmup: int, repeats: int) -> float:
    """metrics.py:113-121."""
    import numpy as np
    for _ in range(warmup):
        fn()
    samples = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        fn()
        samples.append(time.perf_counter() - t0)
    return float(np.median(samples))


def measure(ckpt, base, weights: QualityWeights, bounds: FactorBounds, clusters: int = 16,
            warmup: int = 5, repeats: int = 20, device=None) -> QualityReport:
    """metrics.py:124-166 on the GPU codec: encode the checkpoint (model
    states RAW, or DELTA against `base`; optimizer states QUANT), decode it
    back on the device (deltas applied to the base's states), and score.
    cr_raw is the reference's (the encoded bytes are identical); ps_raw is
    the mean MSE of the restored optimizer states (float64 on the device);
    cs_raw is the median pipeline time minus the reference's host
    serialize/deserialize baseline (negative when the GPU pipeline beats
    that no-op).  Inputs may be TensorBlobs or store.DeviceTensors."""
    from . import store as S
    from .tensors import Checkpoint, deserialize_checkpoint, serialize_checkpoint
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    kind = S.KIND_BASE if base is None else S.KIND_DELTA
    enc = S.CheckpointEncoder(dev, clusters=clusters, keep_prev=False)
    buf = [None]

    def run_pipeline():
        manifest, out = enc.encode(ckpt, base, kind, out=buf[0])
        buf[0] = out
        restored = S.decode_chain([(manifest, out)], dev, to_host=False, base=base)
        return out.numel(), restored

    def host(t):
        return t.to_blob() if isinstance(t, S.DeviceTensor) else t

    host_ckpt = Checkpoint(iteration=ckpt.iteration,
                           model_states=tuple(host(t) for t in ckpt.model_states),
                           optimizer_states=tuple(host(t) for t in ckpt.optimizer_states))

    def run_baseline():
        deserialize_checkpoint(serialize_checkpoint(host_ckpt))

    compressed_bytes, restored = run_pipeline()
    original_bytes = sum(t.nbytes for t in ckpt.model_states) + \
        sum(t.nbytes for t in ckpt.optimizer_states)
    cr_raw = original_bytes / compressed_bytes if compressed_bytes else float("inf")
    pipeline_t = _median_time(run_pipeline, warmup, repeats)
    baseline_t = _median_time(run_baseline, warmup, repeats)
    cs_raw = pipeline_t - baseline_t
    if ckpt.optimizer_states:
        up = S._Uploader(dev, [t for t in ckpt.optimizer_states
                               if not isinstance(t, S.DeviceTensor)])
        mses = [precision_device(S._device_flat(o, up), r.flat())["mse"]
                for o, r in zip(ckpt.optimizer_states, restored.optimizer_states)]
        import numpy as np
        ps_raw = float(np.mean(mses))
    else:
        ps_raw = 0.0
    return build_report(cr_raw, cs_raw, ps_raw, weights, bounds)
