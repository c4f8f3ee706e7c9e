"""Thin ctypes binding of libhz.so (include/hz.h).  Argument marshalling only:
every step of the hot path runs in the library's CUDA kernels and NCCL calls.

Importing this module loads ``libhz.so`` from the package directory and raises
``ImportError`` if it is missing: there is no CPU fallback.  Tensor arguments
are torch CUDA tensors (PyTorch provides device memory, streams and process
groups only); raw integer device pointers are accepted too.
"""

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, os.environ.get("HZ_LIB", "libhz.so"))   # HZ_LIB: experimental builds only

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_2501_04266_b200.build` "
        "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

MAX_LEVELS = 4
F32, BF16, F16 = 0, 1, 2
OK, ERR_INVALID, ERR_CUDA, ERR_NCCL, ERR_NONFINITE, ERR_UNSUPPORTED, ERR_ABORTED = range(7)
_STATUS = {1: "HZ_ERR_INVALID", 2: "HZ_ERR_CUDA", 3: "HZ_ERR_NCCL", 4: "HZ_ERR_NONFINITE",
           5: "HZ_ERR_UNSUPPORTED", 6: "HZ_ERR_ABORTED"}


class HZError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class Partition(ctypes.Structure):
    _fields_ = [
        ("numel", ctypes.c_int64), ("padded_numel", ctypes.c_int64),
        ("block", ctypes.c_int32), ("levels", ctypes.c_int32), ("world", ctypes.c_int32),
        ("rank", ctypes.c_int32), ("w", ctypes.c_int32), ("s", ctypes.c_int32),
        ("gl", ctypes.c_int32),
        ("group", ctypes.c_int32 * MAX_LEVELS), ("digit", ctypes.c_int32 * MAX_LEVELS),
        ("off", ctypes.c_int64 * (MAX_LEVELS + 1)), ("len", ctypes.c_int64 * (MAX_LEVELS + 1)),
        ("nhops", ctypes.c_int32), ("hop_last", ctypes.c_int32 * MAX_LEVELS),
    ]

    def range(self, level):
        return int(self.off[level]), int(self.len[level])

    def set_hops(self, hop_last):
        """hz_partition_set_hops: qgZ hop grouping, e.g. (2, 3) on a 3-level hierarchy =
        levels 1..2 in one all-to-all, then level 3; None / () = one hop per level."""
        hl = list(hop_last or ())
        arr = (ctypes.c_int * max(len(hl), 1))(*hl)
        _check(_lib.hz_partition_set_hops(ctypes.byref(self), len(hl), arr))
        return self

    def hops(self):
        """The hop grouping as a list of (first level, last level)."""
        if self.nhops == 0:
            return [(l, l) for l in range(1, self.levels + 1)]
        out, a = [], 1
        for k in range(self.nhops):
            out.append((a, int(self.hop_last[k])))
            a = int(self.hop_last[k]) + 1
        return out

    def as_dict(self):
        L = self.levels
        return {
            "numel": self.numel, "padded_numel": self.padded_numel, "block": self.block,
            "levels": L, "world": self.world, "rank": self.rank, "w": self.w, "s": self.s,
            "gl": self.gl, "group": list(self.group[:L]), "digit": list(self.digit[:L]),
            "off": list(self.off[:L + 1]), "len": list(self.len[:L + 1]),
            "nhops": self.nhops, "hop_last": list(self.hop_last[:self.nhops]),
        }


class Uid(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_ubyte * 128)]


class TraceRec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_char_p), ("level", ctypes.c_int32), ("bits", ctypes.c_int32),
                ("elems", ctypes.c_int64), ("bytes", ctypes.c_int64), ("remote_bytes", ctypes.c_int64),
                ("ms", ctypes.c_float),
                ("wait_ms", ctypes.c_float), ("work_ms", ctypes.c_float), ("publish_ms", ctypes.c_float),
                ("stamp_ms", ctypes.c_float)]


class CommStep(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("level", ctypes.c_int32), ("level_last", ctypes.c_int32),
                ("group", ctypes.c_int32),
                ("peer", ctypes.c_int32), ("peer_rank", ctypes.c_int32), ("bits", ctypes.c_int32),
                ("elems", ctypes.c_int64), ("send_off", ctypes.c_int64), ("recv_off", ctypes.c_int64),
                ("code_bytes", ctypes.c_int64), ("scale_bytes", ctypes.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


PLAN_ALLGATHER, PLAN_SENDRECV = 1, 2

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int


def _sig(name, argtypes, restype=ctypes.c_int):
    f = getattr(_lib, name)
    f.argtypes = argtypes
    f.restype = restype
    return f


_sig("hz_version", [], ctypes.c_char_p)
_sig("hz_last_error", [], ctypes.c_char_p)
_sig("hz_num_symbols", [], ctypes.c_int)
_sig("hz_symbol_name", [_int], ctypes.c_char_p)
_sig("hz_partition_ex", [_int, _int, ctypes.POINTER(ctypes.c_int), _i64, _int, _int, _int, _int,
                         ctypes.POINTER(Partition)])
_sig("hz_quantize", [_vp, _int, _i64, _int, _int, _vp, _vp, _vp])
_sig("hz_dequantize", [_vp, _vp, _i64, _int, _int, _vp, _int, _vp])
_sig("hz_reduce_chunks", [_int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i64, _int, _int, _int,
                          _vp, _vp, _vp, _int, _vp])
_sig("hz_get_uid", [ctypes.POINTER(Uid)])
_sig("hz_init", [ctypes.POINTER(_vp), _int, _int, ctypes.POINTER(Uid), _int,
                 ctypes.POINTER(ctypes.c_int), _int, ctypes.c_size_t])
_sig("hz_finalize", [_vp])
_sig("hz_partition", [_vp, _i64, _int, _int, _int, _int, ctypes.POINTER(Partition)])
_sig("hz_allgather_params", [_vp, ctypes.POINTER(Partition), _int, _vp, _int, _int, _vp, _vp, _vp,
                             _int, _vp])
_sig("hz_reduce_scatter_grads", [_vp, ctypes.POINTER(Partition), _vp, _int, _int, _int,
                                 ctypes.POINTER(ctypes.c_int), _vp, _int, _vp])
_sig("hz_allgather_params_next", [_vp, ctypes.POINTER(Partition), _vp, _int, _int, _vp, _vp, _vp, _int,
                                  ctypes.POINTER(Partition), _vp, _vp, _vp, _vp])
_sig("hz_backward_step", [_vp, ctypes.POINTER(Partition), _vp, _int, _int, _int, ctypes.POINTER(ctypes.c_int), _vp,
                          _int, ctypes.POINTER(Partition), _vp, _vp, _int, _vp, _int, _vp])
class AdamWParams(ctypes.Structure):
    _fields_ = [(n, ctypes.c_float) for n in ("b1", "omb1", "b2", "omb2", "lr_wd", "sqrt_bc2", "eps", "step")]


_sig("hz_adamw_params", [ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                         _i64, ctypes.POINTER(AdamWParams)])


def adamw_params(lr, b1, b2, eps, wd, t):
    """hz_adamw_params: the hz_adamw_t of step t (t >= 1), computed by the library
    (reading R19: double, rounded once to fp32)."""
    hp = AdamWParams()
    _check(_lib.hz_adamw_params(float(lr), float(b1), float(b2), float(eps), float(wd), int(t), ctypes.byref(hp)))
    return hp


_sig("hz_adamw_step", [_vp, ctypes.POINTER(Partition), _vp, _vp, _vp, _vp, ctypes.POINTER(AdamWParams), _vp, _int,
                       _vp])
_sig("hz_set_sm_budget", [_int])
_sig("hz_allreduce_select", [_vp, _vp, _vp, _int, _int, _vp, _vp])
_sig("hz_flat_allgather", [_vp, _vp, _vp, _i64, _int, _vp])


class StepHostArgs:
    """Marshalled hz_step_host arguments (keeps the partitions and tensors alive)."""

    def __init__(self, io, n, dt, bits, keep):
        self.io, self.n, self.dt, self.bits, self._keep = io, n, dt, bits, keep


class TensorIO(ctypes.Structure):
    """hz_tensor_io: one tensor of an hz_step_host call (host + device buffers)."""
    _fields_ = [("p", ctypes.POINTER(Partition)), ("h_primary", _vp), ("d_primary", _vp), ("h_grad", _vp),
                ("d_grad", _vp), ("sec_codes", _vp), ("sec_scales", _vp), ("d_shard", _vp), ("h_shard", _vp)]


_sig("hz_step_host", [_vp, _int, ctypes.POINTER(TensorIO), _int, _int, ctypes.POINTER(ctypes.c_int), _vp, _vp,
                      _int, _vp])
_sig("hz_flat_reduce_scatter", [_vp, _vp, _vp, _i64, _int, _vp])
_sig("hz_trace_begin", [_int, _int])
_sig("hz_trace_end", [])
_sig("hz_trace_read", [ctypes.POINTER(TraceRec), _int, ctypes.POINTER(ctypes.c_int)])
_sig("hz_enable_p2p", [_vp, ctypes.c_size_t])
_sig("hz_init_virtual", [ctypes.POINTER(_vp), _int, _int, ctypes.POINTER(ctypes.c_int), _int, ctypes.c_size_t])
_sig("hz_init_virtual_ex", [ctypes.POINTER(_vp), _int, _int, ctypes.POINTER(ctypes.c_int),
                            ctypes.POINTER(ctypes.c_int), ctypes.c_size_t])
_sig("hz_set_wait_timeout", [_vp, ctypes.c_double])
_sig("hz_abort", [_vp])
_sig("hz_nvlink_probe", [_vp, _int, ctypes.c_size_t, _int, ctypes.POINTER(ctypes.c_float), _vp])
_sig("hz_check", [_vp])
_sig("hz_flush", [_vp, _vp])
_sig("hz_partition_set_hops", [ctypes.POINTER(Partition), _int, ctypes.POINTER(ctypes.c_int)])
_sig("hz_p2p_enabled", [_vp, ctypes.POINTER(ctypes.c_int)])
_sig("hz_sym_alloc", [_vp, ctypes.c_size_t, ctypes.POINTER(_vp)])
_sig("hz_p2p_capture_begin", [_vp])
_sig("hz_p2p_capture_end", [_vp, _vp, ctypes.POINTER(ctypes.c_ulonglong)])
_sig("hz_p2p_replayed", [_vp, ctypes.c_ulonglong])
_sig("hz_plan_allgather", [ctypes.POINTER(Partition), _int, _int, ctypes.POINTER(CommStep), _int,
                           ctypes.POINTER(ctypes.c_int)])
_sig("hz_plan_reduce_scatter", [ctypes.POINTER(Partition), _int, _int, ctypes.POINTER(ctypes.c_int),
                                ctypes.POINTER(CommStep), _int, ctypes.POINTER(ctypes.c_int)])


def _check(status):
    if status != OK:
        raise HZError(status, _lib.hz_last_error().decode())


def version():
    return _lib.hz_version().decode()


def exported_symbols():
    return [_lib.hz_symbol_name(i).decode() for i in range(_lib.hz_num_symbols())]


def lib_handle():
    return _lib


# ------------------------------------------------------------------ marshalling
def _ptr(t):
    """Device pointer of a torch tensor (or an int / None)."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _need(t, name, numel=None, dtypes=None):
    """Host-side guard for a tensor argument (the C side cannot know buffer sizes):
    a contiguous CUDA tensor of an accepted dtype with at least ``numel`` elements.
    Raw integer pointers and None pass through unchecked."""
    if t is None or isinstance(t, int):
        return
    if not t.is_cuda:
        raise HZError(ERR_INVALID, f"{name}: not a CUDA tensor")
    if not t.is_contiguous():
        raise HZError(ERR_INVALID, f"{name}: not contiguous")
    if dtypes is not None and t.dtype not in dtypes:
        raise HZError(ERR_INVALID, f"{name}: dtype {t.dtype} not in {dtypes}")
    if numel is not None and t.numel() < numel:
        raise HZError(ERR_INVALID, f"{name}: {t.numel()} elements, needs {numel}")


def _float_dtypes():
    import torch
    return (torch.float32, torch.bfloat16, torch.float16)


def _dtype_code(t):
    import torch
    return {torch.float32: F32, torch.bfloat16: BF16, torch.float16: F16}[t.dtype]


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _groups(group):
    g = list(group)
    return (ctypes.c_int * len(g))(*g), len(g)


# ---------------------------------------------------------------- host-only API
def partition_ex(rank, group, numel, block=256, w=1, s=1, gl=None, hops=None):
    """hz_partition_ex: the O1-O3 map for one rank (pure host, no GPU); ``hops``: the
    qgZ hop grouping as hz_partition_set_hops's hop_last list (None = per level)."""
    arr, L = _groups(group)
    p = Partition()
    _check(_lib.hz_partition_ex(rank, L, arr, numel, block, w, s, L if gl is None else gl,
                                ctypes.byref(p)))
    if hops:
        p.set_hops(hops)
    return p


def _plan(call, *args):
    n = ctypes.c_int(0)
    _check(call(*args, None, 0, ctypes.byref(n)))
    steps = (CommStep * max(n.value, 1))()
    _check(call(*args, steps, n.value, ctypes.byref(n)))
    return [s.as_dict() for s in steps[:n.value]]


def plan_allgather(p, backward=False, bits=8):
    """hz_plan_allgather: the NCCL all-gathers this rank issues (host only)."""
    return _plan(_lib.hz_plan_allgather, ctypes.byref(p), int(bool(backward)), bits)


def plan_reduce_scatter(p, bits_per_level, from_level=1, to_level=None):
    """hz_plan_reduce_scatter: the NCCL send/recv pairs this rank issues (host only)."""
    L = p.levels
    bpl = list(bits_per_level) + [4] * (L - len(bits_per_level))
    arr = (ctypes.c_int * L)(*bpl)
    return _plan(_lib.hz_plan_reduce_scatter, ctypes.byref(p), from_level,
                 L if to_level is None else to_level, arr)


# ------------------------------------------------------------------- codec ops
def code_nbytes(n, bits):
    return n * bits // 8


def quantize(x, bits=8, block=256, codes=None, scales=None, stream=None):
    """hz_quantize on a contiguous CUDA tensor x (fp32/bf16/fp16)."""
    import torch
    n = x.numel()
    if codes is None:
        codes = torch.empty(code_nbytes(n, bits), dtype=torch.uint8, device=x.device)
    if scales is None:
        scales = torch.empty(n // block, dtype=torch.float32, device=x.device)
    _check(_lib.hz_quantize(_ptr(x), _dtype_code(x), n, bits, block, _ptr(codes), _ptr(scales),
                            _stream(stream)))
    return codes, scales


def dequantize(codes, scales, n, bits=8, block=256, out_dtype=None, out=None, stream=None):
    import torch
    if out is None:
        out = torch.empty(n, dtype=out_dtype or torch.bfloat16, device=codes.device)
    _check(_lib.hz_dequantize(_ptr(codes), _ptr(scales), n, bits, block, _ptr(out),
                              _dtype_code(out), _stream(stream)))
    return out


def reduce_chunks(codes_list, scales_list, n, bits_in=4, block=256, bits_out=0, out_codes=None,
                  out_scales=None, out_f32=None, accumulate=False, stream=None):
    """hz_reduce_chunks: sum of g coded chunks (ascending p), requantized (bits_out 4/8)
    or written / accumulated as fp32 (bits_out 0)."""
    import torch
    g = len(codes_list)
    dev = codes_list[0].device
    if bits_out:
        if out_codes is None:
            out_codes = torch.empty(code_nbytes(n, bits_out), dtype=torch.uint8, device=dev)
        if out_scales is None:
            out_scales = torch.empty(n // block, dtype=torch.float32, device=dev)
    elif out_f32 is None:
        out_f32 = torch.empty(n, dtype=torch.float32, device=dev)
    cp = (_vp * g)(*[_ptr(c) for c in codes_list])
    sp = (_vp * g)(*[_ptr(s) for s in scales_list])
    _check(_lib.hz_reduce_chunks(g, cp, sp, n, bits_in, block, bits_out, _ptr(out_codes),
                                 _ptr(out_scales), _ptr(out_f32), int(bool(accumulate)),
                                 _stream(stream)))
    return (out_codes, out_scales) if bits_out else out_f32


# ---------------------------------------------------------------------- tracing
TRACE_EVENTS, TRACE_STAMPS = 1, 2


def trace_begin(capacity=4096, events=True, stamps=True):
    _check(_lib.hz_trace_begin(capacity, (TRACE_EVENTS if events else 0) | (TRACE_STAMPS if stamps else 0)))


def trace_end():
    _check(_lib.hz_trace_end())


def trace_read(max_records=1 << 16):
    n = ctypes.c_int(0)
    _check(_lib.hz_trace_read(None, 0, ctypes.byref(n)))
    cnt = min(n.value, max_records)
    recs = (TraceRec * max(cnt, 1))()
    _check(_lib.hz_trace_read(recs, cnt, ctypes.byref(n)))
    return [{"kind": r.kind.decode(), "level": r.level, "bits": r.bits, "elems": r.elems,
             "bytes": r.bytes, "remote_bytes": r.remote_bytes, "ms": r.ms, "wait_ms": r.wait_ms, "work_ms": r.work_ms,
             "publish_ms": r.publish_ms, "stamp_ms": r.stamp_ms}
            for r in recs[:n.value]]


_TYPESTR = {"torch.uint8": "|u1", "torch.float32": "<f4", "torch.bfloat16": "<V2", "torch.float16": "<f2"}


class _CudaArray:
    def __init__(self, ptr, numel, typestr):
        self.__cuda_array_interface__ = {"shape": (numel,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def _wrap_device_ptr(ptr, numel, dtype, device):
    """Zero-copy torch tensor over library-owned device memory."""
    import torch
    if dtype == torch.bfloat16:
        t = torch.as_tensor(_CudaArray(ptr, numel, "<i2"), device=f"cuda:{device}")
        return t.view(torch.bfloat16)
    return torch.as_tensor(_CudaArray(ptr, numel, _TYPESTR[str(dtype)]), device=f"cuda:{device}")


# ------------------------------------------------------------------ collectives
def set_sm_budget(sms):
    """hz_set_sm_budget: size every libhz grid for `sms` SMs (0 = all SMs)."""
    _check(_lib.hz_set_sm_budget(int(sms)))


def get_uid():
    u = Uid()
    _check(_lib.hz_get_uid(ctypes.byref(u)))
    return bytes(u.bytes)


class Context:
    """One rank's hz context: NCCL communicators per hierarchy level + workspace.

    group: relative group sizes innermost first, e.g. (2, 2, 2); the cumulative form
    (2, 4, 8) of the north star is accepted with ``cumulative=True``."""

    def __init__(self, rank, world, uid, group, device, workspace_bytes=0, cumulative=False):
        g = list(group)
        if cumulative:
            rel, prev = [], 1
            for c in g:
                if c % prev:
                    raise ValueError("cumulative group sizes must divide each other")
                rel.append(c // prev)
                prev = c
            g = rel
        self.group = tuple(g)
        self.rank, self.world, self.device = rank, world, device
        u = Uid()
        ctypes.memmove(ctypes.byref(u), bytes(uid), 128)
        arr, L = _groups(g)
        h = _vp()
        _check(_lib.hz_init(ctypes.byref(h), rank, world, ctypes.byref(u), L, arr, device,
                            workspace_bytes))
        self._h = h

    @classmethod
    def _wrap(cls, handle, rank, world, group, device):
        self = cls.__new__(cls)
        self.group, self.rank, self.world, self.device = tuple(group), rank, world, device
        self._h = handle
        return self

    def set_wait_timeout(self, seconds):
        """hz_set_wait_timeout: longest cross-GPU wait before the context aborts."""
        _check(_lib.hz_set_wait_timeout(self._h, float(seconds)))

    def abort(self):
        """hz_abort: abort the context (waiting kernels return; later calls fail)."""
        _check(_lib.hz_abort(self._h))

    def nvlink_probe(self, peer, nbytes, reps=5, stream=None):
        """hz_nvlink_probe: ms per read of nbytes of rank peer's pool (SM loads)."""
        ms = ctypes.c_float(0.0)
        _check(_lib.hz_nvlink_probe(self._h, int(peer), int(nbytes), int(reps), ctypes.byref(ms), _stream(stream)))
        return ms.value

    def check(self):
        """hz_check: raises HZError(ERR_ABORTED / ERR_NCCL) if the context is dead."""
        _check(_lib.hz_check(self._h))

    def flush(self, stream=None):
        """hz_flush: complete deferred P2P work (a deferred last qgZ hop of backward_step,
        a prefetched quantize's phase) on the stream."""
        _check(_lib.hz_flush(self._h, _stream(stream)))

    @property
    def levels(self):
        return len(self.group)

    def close(self):
        if self._h:
            _check(_lib.hz_finalize(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def enable_p2p(self, pool_bytes):
        """hz_enable_p2p (collective): NVLink peer-memory transport with a symmetric
        pool of pool_bytes on every rank."""
        _check(_lib.hz_enable_p2p(self._h, int(pool_bytes)))

    @property
    def p2p(self):
        v = ctypes.c_int(0)
        _check(_lib.hz_p2p_enabled(self._h, ctypes.byref(v)))
        return bool(v.value)

    def p2p_capture_begin(self):
        _check(_lib.hz_p2p_capture_begin(self._h))

    def p2p_capture_end(self, stream=None):
        span = ctypes.c_ulonglong(0)
        _check(_lib.hz_p2p_capture_end(self._h, _stream(stream), ctypes.byref(span)))
        return span.value

    def p2p_replayed(self, n):
        _check(_lib.hz_p2p_replayed(self._h, int(n)))

    def sym_alloc(self, numel, dtype):
        """hz_sym_alloc: a torch view of a symmetric pool allocation (same sequence of
        calls on every rank).  The memory belongs to the context."""
        import torch
        itemsize = torch.empty(0, dtype=dtype).element_size()
        ptr = _vp()
        _check(_lib.hz_sym_alloc(self._h, numel * itemsize, ctypes.byref(ptr)))
        return _wrap_device_ptr(ptr.value, numel, dtype, self.device)

    def partition(self, numel, block=256, w=1, s=1, gl=None, hops=None):
        p = Partition()
        _check(_lib.hz_partition(self._h, numel, block, w, s, self.levels if gl is None else gl,
                                 ctypes.byref(p)))
        if hops:
            p.set_hops(hops)
        return p

    def allgather_params(self, p, primary, sec_codes, sec_scales, full_out, bits=8,
                         backward=False, stream=None):
        """Forward (backward=False): quantize ``primary`` (the rank's range_w), gather,
        fill the secondary buffers, dequantize into ``full_out`` (Np elements).
        Backward: gather from the secondary buffers and dequantize."""
        import torch
        B, Np = p.block, p.padded_numel
        _, len_w = p.range(p.w)
        _, len_s = p.range(p.s)
        if not backward:
            _need(primary, "primary", len_w, _float_dtypes())
        _need(sec_codes, "sec_codes", len_s * bits // 8, (torch.uint8,))
        _need(sec_scales, "sec_scales", len_s // B, (torch.float32,))
        _need(full_out, "full_out", Np, _float_dtypes())
        dt = _dtype_code(primary) if primary is not None else BF16
        _check(_lib.hz_allgather_params(self._h, ctypes.byref(p), int(bool(backward)),
                                        _ptr(primary), dt, bits, _ptr(sec_codes),
                                        _ptr(sec_scales), _ptr(full_out), _dtype_code(full_out),
                                        _stream(stream)))
        return full_out

    def allgather_params_next(self, p, primary, sec_codes, sec_scales, full_out, bits=8, p_next=None,
                              next_primary=None, next_sec_codes=None, next_sec_scales=None, stream=None):
        """hz_allgather_params_next: forward gather of ``p`` with the quantize of the next
        layer's primary (``p_next``) prefetched into the same launch (same bits / dtype)."""
        import torch
        _need(primary, "primary", p.range(p.w)[1], _float_dtypes())
        _need(sec_codes, "sec_codes", p.range(p.s)[1] * bits // 8, (torch.uint8,))
        _need(sec_scales, "sec_scales", p.range(p.s)[1] // p.block, (torch.float32,))
        _need(full_out, "full_out", p.padded_numel, _float_dtypes())
        if p_next is not None:
            _need(next_primary, "next_primary", p_next.range(p_next.w)[1], _float_dtypes())
            _need(next_sec_codes, "next_sec_codes", p_next.range(p_next.s)[1] * bits // 8, (torch.uint8,))
            _need(next_sec_scales, "next_sec_scales", p_next.range(p_next.s)[1] // p_next.block, (torch.float32,))
        _check(_lib.hz_allgather_params_next(
            self._h, ctypes.byref(p), _ptr(primary), _dtype_code(primary), bits, _ptr(sec_codes), _ptr(sec_scales),
            _ptr(full_out), _dtype_code(full_out), ctypes.byref(p_next) if p_next is not None else None,
            _ptr(next_primary), _ptr(next_sec_codes), _ptr(next_sec_scales), _stream(stream)))
        return full_out

    def backward_step(self, p, grad, shard, bits_per_level=None, p_prev=None, prev_sec_codes=None,
                      prev_sec_scales=None, prev_full_out=None, prev_bits=8, from_level=1, to_level=None,
                      accumulate=False, stream=None):
        """hz_backward_step: qgZ reduce-scatter of ``p``'s gradient and the backward gather
        of the previous layer ``p_prev`` (fused in one launch where possible)."""
        import torch
        L = self.levels
        to = L if to_level is None else to_level
        _need(grad, "grad", p.range(from_level - 1)[1], _float_dtypes())
        _need(shard, "shard", p.range(to)[1], (torch.float32,))
        if p_prev is not None:
            _need(prev_sec_codes, "prev_sec_codes", p_prev.range(p_prev.s)[1] * prev_bits // 8, (torch.uint8,))
            _need(prev_sec_scales, "prev_sec_scales", p_prev.range(p_prev.s)[1] // p_prev.block, (torch.float32,))
            _need(prev_full_out, "prev_full_out", p_prev.padded_numel, _float_dtypes())
        bpl = list(bits_per_level) if bits_per_level is not None else [4] * L
        bpl = bpl + [4] * (L - len(bpl))
        arr = (ctypes.c_int * L)(*bpl)
        _check(_lib.hz_backward_step(
            self._h, ctypes.byref(p), _ptr(grad), _dtype_code(grad), from_level, L if to_level is None else to_level,
            arr, _ptr(shard), int(bool(accumulate)), ctypes.byref(p_prev) if p_prev is not None else None,
            _ptr(prev_sec_codes), _ptr(prev_sec_scales), prev_bits, _ptr(prev_full_out),
            _dtype_code(prev_full_out) if prev_full_out is not None else BF16, _stream(stream)))
        return shard

    def reduce_scatter_grads(self, p, grad, shard, bits_per_level=None, from_level=1,
                             to_level=None, accumulate=False, stream=None):
        import torch
        L = self.levels
        _need(grad, "grad", p.range(from_level - 1)[1], _float_dtypes())
        _need(shard, "shard", p.range(L if to_level is None else to_level)[1], (torch.float32,))
        bpl = list(bits_per_level) if bits_per_level is not None else [4] * L
        bpl = bpl + [4] * (L - len(bpl))
        arr = (ctypes.c_int * L)(*bpl)
        _check(_lib.hz_reduce_scatter_grads(self._h, ctypes.byref(p), _ptr(grad), _dtype_code(grad),
                                            from_level, L if to_level is None else to_level, arr,
                                            _ptr(shard), int(bool(accumulate)), _stream(stream)))
        return shard

    def allreduce_select(self, p, shard_in, out, from_level, to_level=None, stream=None):
        """hz_allreduce_select: the paper-literal A10 step (fp32 allreduce over levels
        from..to, ascending digit, then this rank's range_to slice into ``out``)."""
        import torch
        _need(shard_in, "shard_in", p.range(from_level - 1)[1], (torch.float32,))
        _need(out, "out", p.range(self.levels if to_level is None else to_level)[1], (torch.float32,))
        _check(_lib.hz_allreduce_select(self._h, ctypes.byref(p), _ptr(shard_in), int(from_level),
                                        self.levels if to_level is None else int(to_level), _ptr(out),
                                        _stream(stream)))
        return out

    def adamw_step(self, p, grad_shard, master, m, v, hp, primary, stream=None):
        """hz_adamw_step: AdamW on range_L, then the post-update all-gather into primary."""
        import torch
        nL = p.range(p.levels)[1]
        for t, name in ((grad_shard, "grad_shard"), (master, "master"), (m, "m"), (v, "v")):
            _need(t, name, nL, (torch.float32,))
        _need(primary, "primary", p.range(p.w)[1], _float_dtypes())
        _check(_lib.hz_adamw_step(self._h, ctypes.byref(p), _ptr(grad_shard), _ptr(master), _ptr(m), _ptr(v),
                                  ctypes.byref(hp), _ptr(primary), _dtype_code(primary), _stream(stream)))
        return primary

    def step_host(self, tensors, full_out, qwz_bits=8, qgz_bits=None, stream=None):
        """hz_step_host: one step (forward gather, backward gather, qgZ of every tensor)
        with host inputs and host fp32 shards.  ``tensors``: list of dicts with keys
        p, h_primary, d_primary, h_grad, d_grad, sec_codes, sec_scales, d_shard, h_shard
        (torch tensors; h_* pinned CPU tensors).  ``full_out``: two device buffers.
        Build the argument array once with :meth:`step_host_args` and pass it back to
        reuse it across steps."""
        args = tensors if isinstance(tensors, StepHostArgs) else self.step_host_args(tensors, qgz_bits)
        _check(_lib.hz_step_host(self._h, args.n, args.io, args.dt, qwz_bits, args.bits, _ptr(full_out[0]),
                                 _ptr(full_out[1]), _dtype_code(full_out[0]), _stream(stream)))

    def step_host_args(self, tensors, qgz_bits=None):
        L = self.levels
        bpl = list(qgz_bits) if qgz_bits is not None else [4] * L
        bpl = bpl + [4] * (L - len(bpl))
        io = (TensorIO * len(tensors))()
        for k, t in enumerate(tensors):
            io[k].p = ctypes.pointer(t["p"])
            for f in ("h_primary", "d_primary", "h_grad", "d_grad", "sec_codes", "sec_scales", "d_shard",
                      "h_shard"):
                setattr(io[k], f, _ptr(t[f]))
        return StepHostArgs(io, len(tensors), _dtype_code(tensors[0]["d_primary"]), (ctypes.c_int * L)(*bpl),
                            tensors)

    def flat_allgather(self, chunk, out, stream=None):
        _check(_lib.hz_flat_allgather(self._h, _ptr(chunk), _ptr(out), out.numel(),
                                      _dtype_code(out), _stream(stream)))
        return out

    def flat_reduce_scatter(self, inp, out_chunk, stream=None):
        _check(_lib.hz_flat_reduce_scatter(self._h, _ptr(inp), _ptr(out_chunk), inp.numel(),
                                           _dtype_code(inp), _stream(stream)))
        return out_chunk


def virtual_world(group, device=0, pool_bytes=64 << 20, cumulative=False, devices=None):
    """hz_init_virtual: one Context per rank of hierarchy ``group``, all in this process
    on GPU ``device``, P2P-enabled with each other's pools as peers.  Drive each from
    its own thread (tests/vworld.py).  ``devices`` (one ordinal per rank):
    hz_init_virtual_ex, rank r on GPU devices[r] (peer access over NVLink)."""
    g = list(group)
    if cumulative:
        rel, prev = [], 1
        for c in g:
            rel.append(c // prev)
            prev = c
        g = rel
    world = 1
    for x in g:
        world *= x
    arr, L = _groups(g)
    hs = (_vp * world)()
    if devices is None:
        _check(_lib.hz_init_virtual(hs, world, L, arr, device, int(pool_bytes)))
        return [Context._wrap(_vp(hs[r]), r, world, g, device) for r in range(world)]
    devs = [int(d) for d in devices]
    if len(devs) != world:
        raise ValueError(f"devices: {len(devs)} ordinals for a world of {world}")
    _check(_lib.hz_init_virtual_ex(hs, world, L, arr, (ctypes.c_int * world)(*devs), int(pool_bytes)))
    return [Context._wrap(_vp(hs[r]), r, world, g, devs[r]) for r in range(world)]
