"""Helpers for the GPU parity tests: torch is used only for device memory (plumbing)."""
import numpy as np
import torch


def pad4(d):
    return (d + 3) // 4 * 4


def dev_tile(rp, ci, v):
    """Uploads a CSR tile in the device format of mg_dev_spmm: int32 row_ptr, {int32 col, f32 val}."""
    rp32 = torch.tensor(np.asarray(rp, np.int32), device="cuda")
    ed = np.empty((max(len(ci), 1), 2), np.int32)
    if len(ci):
        ed[:, 0] = np.asarray(ci, np.int32)
        ed[:, 1] = np.asarray(v, np.float32).view(np.int32)
    return rp32, torch.tensor(ed, device="cuda")


def dev_padded(a, ld=None):
    a = np.asarray(a, np.float32)
    rows, w = a.shape
    ld = pad4(w) if ld is None else ld
    buf = np.zeros((rows, ld), np.float32)
    buf[:, :w] = a
    return torch.tensor(buf, device="cuda")


def bits_equal(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def normwise(a, ref):
    a = np.asarray(a, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.max(np.abs(a - ref)) / max(np.max(np.abs(ref)), 1e-30))
