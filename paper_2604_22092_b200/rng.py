"""Counter-based uniforms addressed by (seed, step, stream).

``uniform_array`` is the reference's splitmix64-style mixer
(/root/reference/pkg/src/spreadsim/rng.py:48-67) evaluated by the same
device function the fused step calls; ``rng="philox"`` selects
Philox4x32-10 (key = seed, counter = (stream, step)).  ``derive_seed``
(rng.py:91-96) is integer seed bookkeeping and runs on the host.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib

__all__ = ["RngKey", "uniform", "uniform_array", "derive_seed", "RNG_KINDS"]

_M64 = (1 << 64) - 1
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB
_TRIAL_MULT = 0xD6E8FEB86659FD93
RNG_KINDS = {"splitmix": _lib.RNG_SPLITMIX, "philox": _lib.RNG_PHILOX}


@dataclass(frozen=True)
class RngKey:
    seed: int
    step: int
    stream: int


def _aval(x: int) -> int:
    x = ((x ^ (x >> 30)) * _MIX1) & _M64
    x = ((x ^ (x >> 27)) * _MIX2) & _M64
    return x ^ (x >> 31)


def derive_seed(seed: int, index: int) -> int:
    """Per-trial / per-purpose seed (rng.py:91-96)."""
    x = _aval((seed & _M64) ^ ((index * _TRIAL_MULT) & _M64))
    return _aval((x + _MIX1) & _M64)


def uniform_array(seed: int, step: int, streams=None, n: int | None = None, rng: str = "splitmix",
                  out: torch.Tensor | None = None):
    """Uniforms in [0, 1) for many streams of one (seed, step).

    ``streams`` may be a numpy array (result: numpy), a device tensor
    (result: device tensor) or None with ``n`` (streams = arange(n), result
    on device).
    """
    lib = _lib.load()
    dev = _device.device()
    kind = RNG_KINDS[rng]
    host = streams is not None and not isinstance(streams, torch.Tensor)
    if streams is None:
        s_t = None
        count = int(n)
    else:
        s_t = streams if isinstance(streams, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(np.asarray(streams, dtype=np.uint64)).view(np.int64)).to(dev)
        count = s_t.numel()
    if out is None:
        out = torch.empty(count, dtype=torch.float64, device=dev)
    _lib.check(lib.fs_uniform_fill(seed & _M64, step & _M64, _lib.ptr(s_t), count, kind, _lib.ptr(out),
                                   _device.stream_handle(dev)))
    return out.cpu().numpy() if host else out


def uniform(key: RngKey, rng: str = "splitmix") -> float:
    return float(uniform_array(key.seed, key.step, np.array([key.stream], dtype=np.uint64), rng=rng)[0])
