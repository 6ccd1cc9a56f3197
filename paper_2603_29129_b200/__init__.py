"""paper_2603_29129_b200 -- fp64-accurate DFT of any length from 32-bit NTTs on B200.

Thin ctypes binding over libozfft.so, whose C ABI is declared in include/ozfft.h.
Argument marshalling only: every step of the transform runs in the library's sm_100a
kernels.  PyTorch provides device memory (the plan's persistent and workspace
buffers are torch.uint8 tensors) and streams.  There is no CPU fallback: importing
this package without the built library, or using it without a CUDA device, raises.

    import torch, paper_2603_29129_b200 as oz
    plan = oz.Plan(n=1 << 18, batch=16)            # K=3, L=3, paper primes
    y = plan.forward(x)                            # x: cuda complex128 [16, n]
    x2 = plan.inverse(y)

Method: arXiv 2603.29129 (Bluestein + Ozaki split + two-prime NTT + CRT); see
DESIGN.md and the header for citations.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libozfft.so")

P0 = 2130706433
P1 = 2113929217

_STATUS = {0: "OZFFT_OK", 1: "INVALID_ARGUMENT", 2: "UNSUPPORTED_LENGTH", 3: "BAD_PRIMES",
           4: "ALPHA", 5: "NOT_BOUND", 6: "MISALIGNED", 7: "CUDA", 8: "SHARD",
           9: "BUFFER_TOO_SMALL"}


class OzfftError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"ozfft {_STATUS.get(status, status)}: {msg}")
        self.status = status


class PlanDesc(C.Structure):
    _fields_ = [("n", C.c_int64), ("batch", C.c_int64), ("K", C.c_int32), ("L", C.c_int32),
                ("p0", C.c_uint32), ("p1", C.c_uint32), ("device", C.c_int32),
                ("conv_mode", C.c_int32), ("accum_mode", C.c_int32), ("precision", C.c_int32),
                ("max_workspace_bytes", C.c_uint64)]


class PlanInfo(C.Structure):
    _fields_ = [("n", C.c_int64), ("m", C.c_int64), ("batch", C.c_int64), ("chunk", C.c_int64),
                ("K", C.c_int32), ("L", C.c_int32), ("alpha", C.c_int32), ("rho", C.c_int32),
                ("log2_rows", C.c_int32), ("log2_cols", C.c_int32),
                ("persistent_bytes", C.c_uint64), ("workspace_bytes", C.c_uint64),
                ("cached_ntts", C.c_int32), ("conv_mode", C.c_int32), ("accum_mode", C.c_int32),
                ("precision", C.c_int32)]


class ExecStats(C.Structure):
    _fields_ = [("k", C.c_int32 * 4), ("fwd_ntts", C.c_int64), ("inv_ntts", C.c_int64),
                ("cached_ntts", C.c_int64), ("groups", C.c_int64), ("nonfinite", C.c_int64),
                ("flags", C.c_uint32), ("reserved", C.c_int32)]


class Taps(C.Structure):
    _fields_ = [(f, C.c_void_p) for f in ("digits", "E", "kv", "X", "sched", "Z", "res", "crt", "W")]


# Symbols declared in include/ozfft.h (checked by tests/test_abi.py without a GPU).
EXPORTS = ["ozfft_plan_create", "ozfft_plan_get_info", "ozfft_plan_bind", "ozfft_execute",
           "ozfft_execute_host", "ozfft_execute_taps", "ozfft_last_stats",
           "ozfft_shard_residue_bytes", "ozfft_shard_partial", "ozfft_shard_finish",
           "ozfft_plan_destroy", "ozfft_status_string", "ozfft_last_error_string",
           "ozfft_version", "ozfft_profile_enable", "ozfft_profile_read", "ozfft_kernel_launches",
           "ozfft_host_subbatches", "ozfft_shard_partial_p2p", "ozfft_ipc_get_handle",
           "ozfft_ipc_open_handle", "ozfft_ipc_close"]

STAGES = ["split_max", "split_digits", "col_fwd", "row_fused", "col_inv", "crt_finish"]

_lib = None


def load_library() -> C.CDLL:
    """Load libozfft.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: run `python -m paper_2603_29129_b200.build` "
                          "(or __graft_entry__.build()); ozfft has no CPU fallback")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, u64 = C.c_void_p, C.c_int, C.c_int64, C.c_uint64
    L.ozfft_plan_create.argtypes = [C.POINTER(PlanDesc), C.POINTER(vp)]
    L.ozfft_plan_get_info.argtypes = [vp, C.POINTER(PlanInfo)]
    L.ozfft_plan_bind.argtypes = [vp, vp, C.c_size_t, vp, C.c_size_t, vp]
    L.ozfft_execute.argtypes = [vp, vp, vp, i32, vp]
    L.ozfft_execute_host.argtypes = [vp, vp, vp, i32, vp]
    L.ozfft_execute_taps.argtypes = [vp, vp, vp, i32, vp, C.POINTER(Taps)]
    L.ozfft_last_stats.argtypes = [vp, C.POINTER(ExecStats), vp]
    L.ozfft_shard_residue_bytes.argtypes = [vp, C.c_int32]
    L.ozfft_shard_residue_bytes.restype = u64
    L.ozfft_shard_partial.argtypes = [vp, i32, i32, vp, i32, vp, C.POINTER(C.c_int32), vp]
    L.ozfft_shard_finish.argtypes = [vp, vp, C.c_int32, vp, i32, vp]
    L.ozfft_shard_partial_p2p.argtypes = [vp, i32, i32, vp, i32, C.POINTER(vp), C.POINTER(C.c_int32), vp]
    L.ozfft_ipc_get_handle.argtypes = [vp, vp, C.POINTER(u64)]
    L.ozfft_ipc_open_handle.argtypes = [vp, u64, C.POINTER(vp)]
    L.ozfft_ipc_close.argtypes = [vp, u64]
    L.ozfft_plan_destroy.argtypes = [vp]
    L.ozfft_profile_enable.argtypes = [vp, i32]
    L.ozfft_profile_read.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_int64), vp]
    L.ozfft_host_subbatches.argtypes = [vp, C.POINTER(C.c_int64), i64]
    L.ozfft_host_subbatches.restype = i64
    L.ozfft_kernel_launches.argtypes = []
    L.ozfft_kernel_launches.restype = u64
    for f in ("ozfft_plan_create", "ozfft_plan_get_info", "ozfft_plan_bind", "ozfft_execute",
              "ozfft_execute_host", "ozfft_execute_taps", "ozfft_last_stats",
              "ozfft_shard_partial", "ozfft_shard_finish", "ozfft_plan_destroy",
              "ozfft_shard_partial_p2p", "ozfft_ipc_get_handle", "ozfft_ipc_open_handle",
              "ozfft_ipc_close",
              "ozfft_profile_enable", "ozfft_profile_read"):
        getattr(L, f).restype = C.c_int
    L.ozfft_status_string.argtypes = [C.c_int]
    L.ozfft_status_string.restype = C.c_char_p
    L.ozfft_last_error_string.argtypes = []
    L.ozfft_last_error_string.restype = C.c_char_p
    L.ozfft_version.argtypes = []
    L.ozfft_version.restype = C.c_char_p
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        raise OzfftError(status, load_library().ozfft_last_error_string().decode())


def version() -> str:
    return load_library().ozfft_version().decode()


def ipc_handle(t: torch.Tensor) -> bytes:
    """CUDA IPC handle of a tensor's device memory: 64 handle bytes + the 8-byte offset of the
    tensor inside its allocation (a caching allocator's tensor need not start it)."""
    buf = C.create_string_buffer(64)
    off = C.c_uint64(0)
    with torch.cuda.device(t.device):
        _check(load_library().ozfft_ipc_get_handle(t.data_ptr(), buf, C.byref(off)))
    return buf.raw + int(off.value).to_bytes(8, "little")


def ipc_open(handle: bytes, device=None) -> int:
    """Map another process's tensor (ipc_handle) into this process: its device pointer."""
    ptr = C.c_void_p(0)
    off = int.from_bytes(handle[64:72], "little")
    with torch.cuda.device(_normalize_device(device)):
        _check(load_library().ozfft_ipc_open_handle(C.create_string_buffer(handle[:64], 64), off, C.byref(ptr)))
    return int(ptr.value)


def ipc_close(ptr: int, handle: bytes, device=None):
    """Release a mapping made by ipc_open(handle)."""
    off = int.from_bytes(handle[64:72], "little")
    with torch.cuda.device(_normalize_device(device)):
        _check(load_library().ozfft_ipc_close(C.c_void_p(ptr), off))


def kernel_launches() -> int:
    """Process-wide number of kernels libozfft.so has launched."""
    return int(load_library().ozfft_kernel_launches())


def _normalize_device(device) -> torch.device:
    """torch.device('cuda', i) with an explicit index: None / 'cuda' mean the current device,
    so the C plan, its buffers and the inputs' device checks all name the same GPU."""
    d = torch.device("cuda") if device is None else torch.device(device)
    if d.type != "cuda":
        raise ValueError(f"ozfft runs on CUDA devices only, got {d}")
    return torch.device("cuda", torch.cuda.current_device() if d.index is None else d.index)


def _stream_ptr(stream, device=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


class Plan:
    """Plan for `batch` complex fp64 DFTs of length n (any n, 1 <= n <= 2^23: m <= 2^24, the paper primes' limit).

    K: split cap per real vector; L: NTT-domain accumulation bound
    (P:940-946).  p0, p1: NTT primes (default: the paper's).
    conv: "padded" (m = 2^ceil(log2(2n-1)), any n; the north star's path) or "cyclic"
    (m = n for power-of-two n; bitwise-identical results at half the NTT length).
    accum: "real" (the paper's four real convolutions) or "image" (complex-image
    accumulation: 32 instead of 52 runtime NTTs; different digits and bits).
    precision: "dd" (double-double O(n) steps, the default) or "ts" (the paper's
    triple-single arithmetic; accum="real" only).
    """

    CONV = {"padded": 0, "cyclic": 1}
    ACCUM = {"real": 0, "image": 1}
    PREC = {"dd": 0, "ts": 1}

    def __init__(self, n: int, batch: int = 1, K: int = 3, L: int = 3, p0: int = 0, p1: int = 0,
                 device=None, max_workspace_bytes: int = 0, stream=None, conv: str = "padded",
                 accum: str = "real", precision: str = "dd"):
        if not torch.cuda.is_available():
            raise RuntimeError("ozfft needs a CUDA device (sm_100a); there is no CPU fallback")
        self._lib = load_library()
        self.device = dev = _normalize_device(device)
        if conv not in self.CONV:
            raise ValueError(f"conv must be one of {sorted(self.CONV)}")
        if accum not in self.ACCUM:
            raise ValueError(f"accum must be one of {sorted(self.ACCUM)}")
        if precision not in self.PREC:
            raise ValueError(f"precision must be one of {sorted(self.PREC)}")
        d = PlanDesc(n=n, batch=batch, K=K, L=L, p0=p0, p1=p1, device=dev.index,
                     conv_mode=self.CONV[conv], accum_mode=self.ACCUM[accum],
                     precision=self.PREC[precision], max_workspace_bytes=max_workspace_bytes)
        h = C.c_void_p()
        _check(self._lib.ozfft_plan_create(C.byref(d), C.byref(h)))
        self._h = h
        info = PlanInfo()
        _check(self._lib.ozfft_plan_get_info(h, C.byref(info)))
        self.n, self.batch, self.K, self.L = n, batch, info.K, info.L
        self.m, self.alpha, self.rho, self.chunk = info.m, info.alpha, info.rho, info.chunk
        self.log2_rows, self.log2_cols = info.log2_rows, info.log2_cols
        self.conv, self.accum, self.precision = conv, accum, precision
        with torch.cuda.device(dev):
            self.persistent = torch.empty(max(info.persistent_bytes, 256), dtype=torch.uint8, device=dev)
            self.workspace = torch.empty(max(info.workspace_bytes, 256), dtype=torch.uint8, device=dev)
            _check(self._lib.ozfft_plan_bind(h, self.persistent.data_ptr(), self.persistent.numel(),
                                             self.workspace.data_ptr(), self.workspace.numel(),
                                             _stream_ptr(stream, dev)))
        info2 = PlanInfo()
        _check(self._lib.ozfft_plan_get_info(h, C.byref(info2)))
        self.cached_ntts = info2.cached_ntts

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.ozfft_plan_destroy(h)
            self._h = None

    # ------------------------------------------------------------------ execution
    def _check_io(self, x: torch.Tensor, out: torch.Tensor | None):
        if x.device != self.device or x.dtype != torch.complex128 or not x.is_contiguous():
            raise ValueError("input must be a contiguous complex128 tensor on the plan's device")
        if x.numel() != self.batch * self.n:
            raise ValueError(f"input must hold batch*n = {self.batch * self.n} elements")
        if out is None:
            out = torch.empty_like(x)
        elif out.device != self.device or out.dtype != torch.complex128 or not out.is_contiguous() \
                or out.numel() != x.numel():
            raise ValueError("out must match the input")
        return out

    def execute(self, x: torch.Tensor, direction: int = -1, out=None, stream=None) -> torch.Tensor:
        out = self._check_io(x, out)
        if torch.cuda.current_device() == self.device.index:
            _check(self._lib.ozfft_execute(self._h, x.data_ptr(), out.data_ptr(), direction,
                                           _stream_ptr(stream, self.device)))
        else:
            with torch.cuda.device(self.device):  # the library launches on the current device
                _check(self._lib.ozfft_execute(self._h, x.data_ptr(), out.data_ptr(), direction,
                                               _stream_ptr(stream, self.device)))
        return out

    def forward(self, x, out=None, stream=None):
        """y = DFT(x), omega_n = e^{-2 pi i/n} (eq:dft)."""
        return self.execute(x, -1, out, stream)

    def inverse(self, y, out=None, stream=None):
        """x = DFT^{-1}(y) = conj(DFT(conj(y)))/n (eq:idft P:158-160; ruling 16)."""
        return self.execute(y, +1, out, stream)

    def execute_host(self, x_host: torch.Tensor, direction: int = -1, out_host=None, stream=None):
        """End-to-end call on HOST buffers (pinned CPU complex128 tensors): H2D, pipeline, D2H."""
        if x_host.device.type != "cpu" or x_host.dtype != torch.complex128 or not x_host.is_contiguous():
            raise ValueError("x_host must be a contiguous CPU complex128 tensor")
        if out_host is None:
            out_host = torch.empty_like(x_host, pin_memory=x_host.is_pinned())
        with torch.cuda.device(self.device):
            _check(self._lib.ozfft_execute_host(self._h, x_host.data_ptr(), out_host.data_ptr(),
                                                direction, _stream_ptr(stream, self.device)))
        return out_host

    def execute_taps(self, x: torch.Tensor, direction: int = -1, stream=None):
        """Test-only: run once and return every stage output in the oracle's layout."""
        B, n, m, K, L = self.batch, self.n, self.m, self.K, self.L
        G = K * K
        stride = 1 + G * (2 + 2 * L)
        dev = self.device
        z = lambda *s, dt: torch.zeros(*s, dtype=dt, device=dev)  # noqa: E731
        t = dict(digits=z(B, 2, K, n, dt=torch.int32), E=z(B, 2, K, dt=torch.int32),
                 kv=z(B, 2, dt=torch.int32), X=z(B, 2, K, 2, m, dt=torch.int32),
                 sched=z(B, 4, stride, dt=torch.int32), Z=z(B, 4, G, 2, m, dt=torch.int32),
                 res=z(B, 4, G, 2, n, dt=torch.int32), crt=z(B, 4, G, n, dt=torch.int64),
                 W=z(2, K, 2, m, dt=torch.int32))
        tp = Taps(*[t[f].data_ptr() for f, _ in Taps._fields_])
        out = torch.empty_like(x)
        with torch.cuda.device(dev):
            _check(self._lib.ozfft_execute_taps(self._h, x.data_ptr(), out.data_ptr(), direction,
                                                _stream_ptr(stream, dev), C.byref(tp)))
        torch.cuda.synchronize(dev)
        for k in ("X", "Z", "res", "W"):  # uint32 payloads carried in int32 tensors
            t[k] = t[k].to(torch.int64) & 0xFFFFFFFF
        return out, t

    def stats(self, stream=None) -> dict:
        s = ExecStats()
        with torch.cuda.device(self.device):
            _check(self._lib.ozfft_last_stats(self._h, C.byref(s), _stream_ptr(stream, self.device)))
        return dict(k=list(s.k), fwd_ntts=s.fwd_ntts, inv_ntts=s.inv_ntts,
                    cached_ntts=s.cached_ntts, groups=s.groups, nonfinite=s.nonfinite,
                    flags=s.flags)

    # ------------------------------------------------------------------ profiling
    def profile(self, on: bool = True):
        """Enable/disable per-stage CUDA-event timers (OZFFT_STAGE_*)."""
        _check(self._lib.ozfft_profile_enable(self._h, 1 if on else 0))

    def profile_read(self, stream=None) -> dict:
        """{stage: (total_ms, launches)} since enable / last read (synchronizes)."""
        ms = (C.c_double * len(STAGES))()
        ln = (C.c_int64 * len(STAGES))()
        with torch.cuda.device(self.device):
            _check(self._lib.ozfft_profile_read(self._h, ms, ln, _stream_ptr(stream, self.device)))
        return {s: (ms[i], ln[i]) for i, s in enumerate(STAGES)}

    # ------------------------------------------------------------------ sharding
    def shard_residue_bytes(self, groups: int = 0) -> int:
        """Bytes of the [8 units][groups][n] residue exchange buffer (groups <= 0: the K*K
        capacity, the size to allocate)."""
        return int(self._lib.ozfft_shard_residue_bytes(self._h, groups))

    def shard_partial(self, x: torch.Tensor, shard: int, nshards: int, residues: torch.Tensor,
                      direction: int = -1, stream=None) -> int:
        """This shard's units of transform 0 into their place of `residues`; returns the
        group count g of the buffer layout (see include/ozfft.h)."""
        g = C.c_int32(0)
        with torch.cuda.device(self.device):
            _check(self._lib.ozfft_shard_partial(self._h, shard, nshards, x.data_ptr(), direction,
                                                 residues.data_ptr(), C.byref(g),
                                                 _stream_ptr(stream, self.device)))
        return int(g.value)

    def shard_partial_p2p(self, x: torch.Tensor, shard: int, nshards: int, buffers: list,
                          direction: int = -1, stream=None) -> int:
        """shard_partial with the exchange fused into the producing kernels: this shard's
        residues are stored into every rank's buffer; buffers[r] = rank r's exchange buffer as
        a device pointer valid here (int, e.g. from ipc_open) or a tensor (include/ozfft.h)."""
        ptrs = (C.c_void_p * nshards)(*[b.data_ptr() if isinstance(b, torch.Tensor) else int(b)
                                        for b in buffers])
        g = C.c_int32(0)
        with torch.cuda.device(self.device):
            _check(self._lib.ozfft_shard_partial_p2p(self._h, shard, nshards, x.data_ptr(), direction,
                                                     ptrs, C.byref(g), _stream_ptr(stream, self.device)))
        return int(g.value)

    def shard_finish(self, residues: torch.Tensor, groups: int, out: torch.Tensor, direction: int = -1,
                     stream=None):
        with torch.cuda.device(self.device):
            _check(self._lib.ozfft_shard_finish(self._h, residues.data_ptr(), groups, out.data_ptr(),
                                                direction, _stream_ptr(stream, self.device)))
        return out
