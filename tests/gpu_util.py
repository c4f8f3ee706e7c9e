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


GUARD_BYTES = 4096          # sentinel band on each side (keeps 4 KB alignment of the view)
SENTINEL = 0xA5


class Guarded:
    """A device buffer of ``numel`` elements inside sentinel bands (compute-sanitizer is
    not available on the GPU pool): ``.t`` is the view handed to the library (its own
    bytes are pre-filled with the sentinel too, so an element the kernel forgets to
    write fails the parity check), ``check()`` asserts that nothing was written
    outside it.  ``alloc(n, dtype)`` overrides the allocator (e.g. ``ctx.sym_alloc``
    for peer-visible buffers: the same offsets on every rank keep it symmetric)."""

    def __init__(self, numel, dtype, alloc=None, device="cuda", guard_bytes=GUARD_BYTES):
        import torch
        self.item = torch.empty(0, dtype=dtype).element_size()
        self.pad = guard_bytes // self.item
        self.numel = numel
        n = numel + 2 * self.pad
        self.raw = alloc(n, dtype) if alloc is not None else torch.empty(n, dtype=dtype, device=device)
        self.raw.view(torch.uint8).fill_(SENTINEL)
        self.t = self.raw[self.pad:self.pad + numel]

    def check(self, what=""):
        import torch
        b = self.raw.view(torch.uint8)
        lo = self.pad * self.item
        hi = lo + self.numel * self.item
        head = b[:lo].cpu().numpy()
        tail = b[hi:].cpu().numpy()
        for name, band in (("before", head), ("after", tail)):
            bad = np.nonzero(band != SENTINEL)[0]
            if bad.size:
                raise AssertionError(f"{what}: {bad.size} bytes written {name} the buffer "
                                     f"(first at band offset {int(bad[0])})")


def assert_unchanged(t, host_copy, what=""):
    """An input the library only reads must be bit-identical after the call."""
    assert_bitwise(to_host(t), host_copy, f"{what} (input modified)")
