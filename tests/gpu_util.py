"""Helpers for the GPU parity tests: numpy <-> torch transfer (bit-preserving) and
an element-by-element comparison that reports the first mismatching index."""

import ml_dtypes
import numpy as np


def to_dev(x, device="cuda"):
    import torch
    x = np.ascontiguousarray(x)
    if x.dtype == ml_dtypes.bfloat16:
        return torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).to(device)
    return torch.from_numpy(x).to(device)


def to_host(t):
    import torch
    t = t.detach().cpu().contiguous()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(ml_dtypes.bfloat16)
    return t.numpy()


def bits_view(a):
    a = np.asarray(a)
    if a.dtype.itemsize == 1:
        return a.view(np.uint8)
    if a.dtype.itemsize == 2:
        return a.view(np.uint16)
    if a.dtype.itemsize == 4:
        return a.view(np.uint32)
    return a


def assert_bitwise(got, want, what=""):
    g, w = bits_view(got), bits_view(want)
    assert g.shape == w.shape, f"{what}: shape {g.shape} != {w.shape}"
    bad = np.nonzero(g != w)[0]
    if bad.size:
        i = int(bad[0])
        raise AssertionError(f"{what}: {bad.size} mismatches, first at {i}: got {got[i]!r} want {want[i]!r}")


def assert_close_rel(got, want, block_absmax, rel, what=""):
    """|got - want| <= rel * (block absmax of the oracle's value), elementwise."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    err = np.abs(got - want)
    tol = rel * np.asarray(block_absmax, np.float64)
    bad = np.nonzero(err > tol)[0]
    if bad.size:
        i = int(bad[0])
        raise AssertionError(f"{what}: {bad.size} beyond tol, first at {i}: got {got[i]} want {want[i]} tol {tol[i]}")
