"""Device plumbing: the CUDA device, the current stream and host<->device
copies.  PyTorch is used only to own memory and name streams; every compute
call goes to libflashspread_b200.so.  No CUDA device -> FlashSpreadNativeError."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import FlashSpreadNativeError

_NP_TO_TORCH = {
    np.dtype(np.int8): torch.int8,
    np.dtype(np.int32): torch.int32,
    np.dtype(np.int64): torch.int64,
    np.dtype(np.uint64): torch.uint64,
    np.dtype(np.float16): torch.float16,
    np.dtype(np.float32): torch.float32,
    np.dtype(np.float64): torch.float64,
}


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise FlashSpreadNativeError("no CUDA device: the B200 engine has no CPU fallback")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(dev: torch.device | None = None) -> int | None:
    return torch.cuda.current_stream(dev).cuda_stream or None


def to_device(a: np.ndarray, dev: torch.device) -> torch.Tensor:
    """Host numpy -> device tensor (bf16 arrays travel as raw 16-bit words)."""
    a = np.ascontiguousarray(a)
    if a.dtype.name == "bfloat16":
        return torch.from_numpy(a.view(np.int16)).to(dev).view(torch.bfloat16)
    return torch.from_numpy(a).to(dev)


def to_host(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> host numpy (bf16 comes back as ml_dtypes.bfloat16)."""
    if t.dtype == torch.bfloat16:
        import ml_dtypes

        return t.view(torch.int16).cpu().numpy().view(ml_dtypes.bfloat16)
    return t.cpu().numpy()
