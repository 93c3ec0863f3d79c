"""Helpers for the GPU parity tests: move seeded numpy workloads to the device in the kernel's
dtype, and round the oracle's inputs the same way."""
import numpy as np
import torch

from workloads import synth


def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)


def rel_per_instance(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    ax = tuple(range(1, a.ndim))
    return np.abs(a - b).max(axis=ax) / np.maximum(np.abs(b).max(axis=ax), 1e-30)


def np_dtype(tdtype):
    return np.float32 if tdtype == torch.float32 else np.float64


def to_device(d: dict, tdtype, device="cuda"):
    out = {}
    for k, v in d.items():
        if isinstance(v, np.ndarray):
            if v.dtype == np.uint8:
                out[k] = torch.from_numpy(np.ascontiguousarray(v)).to(device)
            else:
                out[k] = torch.from_numpy(np.ascontiguousarray(v.astype(np_dtype(tdtype)))).to(device)
        else:
            out[k] = v
    return out


def rounded(d: dict, tdtype):
    return synth.round_to(d, np_dtype(tdtype))


def to_np(t):
    return t.detach().cpu().numpy().astype(np.float64) if t.dtype.is_floating_point else t.detach().cpu().numpy()
