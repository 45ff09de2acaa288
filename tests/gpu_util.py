"""Host <-> device marshalling for the GPU tests (no arithmetic of the method)."""
import numpy as np
import torch

TORCH = {"int32": torch.int32, "float32": torch.float32, "bfloat16": torch.bfloat16}


def to_dev(x: np.ndarray, dtype: str, device="cuda:0") -> torch.Tensor:
    """numpy buffer (bf16 as uint16 bit patterns) -> CUDA tensor of the I/O dtype."""
    if dtype == "bfloat16":
        return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).to(device).view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(x)).to(device)


def to_host(t: torch.Tensor) -> np.ndarray:
    """CUDA tensor -> numpy (bf16 as uint16 bit patterns)."""
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def _nan_mask(a: np.ndarray):
    """NaN positions: fp32 by value, bf16 (uint16 bit patterns) when (bits & 0x7FFF) > 0x7F80."""
    if a.dtype == np.float32:
        return np.isnan(a)
    if a.dtype == np.uint16:
        return (a & 0x7FFF) > 0x7F80
    return None


def same_bits(a: np.ndarray, b: np.ndarray) -> bool:
    """Bitwise equality; all NaNs compare equal, fp32 and bf16 alike (SURVEY ledger 10)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    na, nb = _nan_mask(a), _nan_mask(b)
    if na is None:
        return bool(np.array_equal(a, b))
    ua = a.view(np.uint32) if a.dtype == np.float32 else a
    ub = b.view(np.uint32) if b.dtype == np.float32 else b
    return bool(np.array_equal(na, nb) and np.array_equal(ua[~na], ub[~nb]))


def first_diff(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    na, nb = _nan_mask(a), _nan_mask(b)
    if a.dtype == np.float32:
        a, b = a.view(np.uint32), b.view(np.uint32)
    diff = a != b
    if na is not None:
        diff &= ~(na & nb)
    idx = np.nonzero(diff)[0]
    return (int(idx[0]), a[idx[0]], b[idx[0]], len(idx)) if len(idx) else None
