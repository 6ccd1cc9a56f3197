"""ctypes wrapper around the CPU oracle (oracle/ozfft_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The product
package ``paper_2603_29129_b200`` never imports it and shares no code with it.

Function-level citations live in ozfft_oracle.c (PAPER.md lines "P:N").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ozfft_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

P0 = 2130706433
P1 = 2113929217


def build(force: bool = False) -> str:
    """Compile the oracle with plain IEEE semantics (no contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
             "-shared", "-o", _LIB, _SRC, "-lquadmath", "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.orc_sym_mod.restype = C.c_int64
        L.orc_sym_mod.argtypes = [C.c_int64, C.c_int64]
        L.orc_powmod.restype = C.c_uint32
        L.orc_powmod.argtypes = [C.c_uint32, C.c_uint64, C.c_uint32]
        L.orc_invmod.restype = C.c_uint32
        L.orc_invmod.argtypes = [C.c_uint32, C.c_uint32]
        L.orc_is_prime.restype = C.c_int
        L.orc_is_prime.argtypes = [C.c_uint64]
        L.orc_primitive_root.restype = C.c_uint32
        L.orc_primitive_root.argtypes = [C.c_uint32]
        L.orc_root_of_unity.restype = C.c_uint32
        L.orc_root_of_unity.argtypes = [C.c_uint32, C.c_uint64]
        L.orc_alpha.restype = C.c_int
        L.orc_alpha.argtypes = [C.c_int64, C.c_int64, C.c_uint32, C.c_uint32]
        L.orc_garner2.restype = C.c_int64
        L.orc_garner2.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                  C.POINTER(C.c_int)]
        L.orc_ntt.restype = None
        L.orc_ntt.argtypes = [C.c_void_p, C.c_int64, C.c_uint32, C.c_int]
        L.orc_chirp.restype = None
        L.orc_chirp.argtypes = [C.c_int64, C.c_void_p, C.c_void_p]
        L.orc_premul.restype = None
        L.orc_premul.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_split.restype = C.c_int
        L.orc_split.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                C.c_void_p, C.c_void_p]
        L.orc_sched_stride.restype = C.c_int
        L.orc_sched_stride.argtypes = [C.c_int, C.c_int]
        L.orc_schedule.restype = C.c_int
        L.orc_schedule.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                   C.c_int, C.c_void_p]
        L.orc_plan_create.restype = C.c_void_p
        L.orc_plan_create.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_uint32, C.c_uint32]
        L.orc_plan_create_ts.restype = C.c_void_p
        L.orc_plan_create_ts.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_uint32, C.c_uint32,
                                         C.c_int, C.c_int, C.c_int]
        for fn in ("orc_ts_add", "orc_ts_mul"):
            getattr(L, fn).restype = TS
            getattr(L, fn).argtypes = [TS, TS]
        L.orc_ts_neg.restype = TS
        L.orc_ts_neg.argtypes = [TS]
        L.orc_ts_from_double.restype = TS
        L.orc_ts_from_double.argtypes = [C.c_double]
        L.orc_ts_from_int64.restype = TS
        L.orc_ts_from_int64.argtypes = [C.c_int64]
        L.orc_ts_to_double.restype = C.c_double
        L.orc_ts_to_double.argtypes = [TS]
        L.orc_split_ts.restype = C.c_int
        L.orc_split_ts.argtypes = [C.c_int64, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_plan_create_ex.restype = C.c_void_p
        L.orc_plan_create_ex.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_uint32, C.c_uint32,
                                         C.c_int, C.c_int]
        L.orc_plan_create_conv.restype = C.c_void_p
        L.orc_plan_create_conv.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_uint32, C.c_uint32,
                                           C.c_int]
        L.orc_plan_destroy.restype = None
        L.orc_plan_destroy.argtypes = [C.c_void_p]
        L.orc_plan_m.restype = C.c_int64
        L.orc_plan_m.argtypes = [C.c_void_p]
        L.orc_plan_alpha.restype = C.c_int
        L.orc_plan_alpha.argtypes = [C.c_void_p]
        L.orc_plan_wsplit.restype = None
        L.orc_plan_wsplit.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_plan_copy.restype = None
        L.orc_plan_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p]
        L.orc_execute.restype = C.c_int
        L.orc_execute.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                  C.POINTER(Taps)]
        L.orc_execute_batch.restype = C.c_int
        L.orc_execute_batch.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                        C.c_int, C.c_int]
        L.orc_dft_f128.restype = None
        L.orc_dft_f128.argtypes = [C.c_int64, C.c_void_p, C.c_int, C.c_void_p, C.c_int64,
                                   C.c_void_p]
    return _lib


class TS(C.Structure):
    """Triple-single number x0 + x1 + x2 (fp32 words), as orc_ts."""
    _fields_ = [("x0", C.c_float), ("x1", C.c_float), ("x2", C.c_float)]

    def words(self):
        return (self.x0, self.x1, self.x2)


class Taps(C.Structure):
    _fields_ = [("digits", C.c_void_p), ("E", C.c_void_p), ("kv", C.c_void_p),
                ("X", C.c_void_p), ("sched", C.c_void_p), ("Z", C.c_void_p),
                ("res", C.c_void_p), ("crt", C.c_void_p), ("xdd", C.c_void_p),
                ("counts", C.c_void_p), ("flags", C.c_void_p)]


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- scalar helpers
def sym_mod(a: int, m: int) -> int:
    return lib().orc_sym_mod(a, m)


def alpha(n: int, L: int, p0: int = P0, p1: int = P1) -> int:
    return lib().orc_alpha(n, L, p0, p1)


def garner2(z0: int, z1: int, p0: int = P0, p1: int = P1) -> tuple[int, bool]:
    fix = C.c_int(0)
    v = lib().orc_garner2(z0, z1, p0, p1, C.byref(fix))
    return v, bool(fix.value)


def primitive_root(p: int) -> int:
    return lib().orc_primitive_root(p)


def root_of_unity(p: int, m: int) -> int:
    return lib().orc_root_of_unity(p, m)


def ntt(a, p: int, inverse: bool = False) -> np.ndarray:
    v = np.ascontiguousarray(np.asarray(a, dtype=np.uint32)).copy()
    lib().orc_ntt(_p(v), v.size, p, 1 if inverse else 0)
    return v


def chirp(n: int) -> tuple[np.ndarray, np.ndarray]:
    Cc = np.empty(n, np.float64)
    S = np.empty(n, np.float64)
    lib().orc_chirp(n, _p(Cc), _p(S))
    return Cc, S


def premul(x: np.ndarray, Cc: np.ndarray, S: np.ndarray, conj: bool = False):
    x = np.ascontiguousarray(x, dtype=np.complex128)
    n = x.size
    out = [np.empty(n, np.float64) for _ in range(4)]
    lib().orc_premul(n, _p(x), _p(np.ascontiguousarray(Cc)), _p(np.ascontiguousarray(S)),
                     1 if conj else 0, *[_p(o) for o in out])
    return out  # hi_re, lo_re, hi_im, lo_im


def split(hi: np.ndarray, lo: np.ndarray, alpha_: int, K: int):
    hi = np.ascontiguousarray(hi, dtype=np.float64).copy()
    lo = np.ascontiguousarray(lo, dtype=np.float64).copy()
    n = hi.size
    dig = np.zeros((K, n), np.int32)
    E = np.zeros(K, np.int32)
    k = lib().orc_split(n, _p(hi), _p(lo), alpha_, K, _p(dig), _p(E))
    return k, dig, E, hi, lo


def schedule(sx, sy, K: int, L: int):
    sx = np.ascontiguousarray(sx, dtype=np.int32)
    sy = np.ascontiguousarray(sy, dtype=np.int32)
    out = np.zeros(lib().orc_sched_stride(K, L), np.int32)
    ng = lib().orc_schedule(sx.size, _p(sx), sy.size, _p(sy), K, L, _p(out))
    groups = []
    for g in range(ng):
        base = 1 + g * (2 + 2 * L)
        cexp, npairs = int(out[base]), int(out[base + 1])
        pairs = [(int(out[base + 2 + 2 * e]), int(out[base + 3 + 2 * e])) for e in range(npairs)]
        groups.append((cexp, pairs))
    return groups, out


def parse_sched(row: np.ndarray, L: int):
    ng = int(row[0])
    groups = []
    for g in range(ng):
        base = 1 + g * (2 + 2 * L)
        cexp, npairs = int(row[base]), int(row[base + 1])
        pairs = [(int(row[base + 2 + 2 * e]), int(row[base + 3 + 2 * e])) for e in range(npairs)]
        groups.append((cexp, pairs))
    return groups


def dft_f128(x: np.ndarray, inverse: bool = False, bins=None) -> np.ndarray:
    """Reference DFT in __float128 (eq:dft); returns (hi + lo) as two arrays."""
    x = np.ascontiguousarray(x, dtype=np.complex128)
    n = x.size
    if bins is None:
        nb, bp = n, None
    else:
        b = np.ascontiguousarray(bins, dtype=np.int64)
        nb, bp = b.size, _p(b)
    out = np.empty((nb, 4), np.float64)
    lib().orc_dft_f128(n, _p(x), 1 if inverse else -1, bp, nb if bins is not None else 0, _p(out))
    hi = out[:, 0] + 1j * out[:, 2]
    lo = out[:, 1] + 1j * out[:, 3]
    return hi, lo


class Plan:
    """Oracle plan: chirp, omega~* split, and the cached W spectra."""

    def __init__(self, n: int, K: int = 3, L: int = 3, p0: int = P0, p1: int = P1,
                 cyclic: bool = False, image: bool = False, ts: bool = False):
        """cyclic: m = n for power-of-two n instead of m >= 2n-1.
        image: complex-image accumulation (orc_execute_image).
        ts: triple-single working precision for a1, a2, a7."""
        self.n, self.K, self.L, self.p, self.cyclic, self.image = n, K, L, (p0, p1), cyclic, image
        self.ts = ts
        self._h = lib().orc_plan_create_ts(n, K, L, p0, p1, 1 if cyclic else 0, 1 if image else 0,
                                           1 if ts else 0)
        if not self._h:
            raise ValueError("orc_plan_create failed")
        self.m = lib().orc_plan_m(self._h)
        self.alpha = lib().orc_plan_alpha(self._h)
        self.stride = lib().orc_sched_stride(K, L)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.orc_plan_destroy(h)
            self._h = None

    def tables(self):
        n, m, K = self.n, self.m, self.K
        Cc = np.empty(n, np.float64)
        S = np.empty(n, np.float64)
        wdig = np.empty((2, K, m), np.int32)
        W = np.empty((2, K, 2, m), np.uint32)
        lib().orc_plan_copy(self._h, _p(Cc), _p(S), _p(wdig), _p(W))
        kw = np.empty(2, np.int32)
        Ew = np.empty((2, K), np.int32)
        lib().orc_plan_wsplit(self._h, _p(kw), _p(Ew))
        return dict(C=Cc, S=S, wdig=wdig, W=W, kw=kw, Ew=Ew)

    def execute(self, x: np.ndarray, inverse: bool = False, taps: bool = False):
        """One transform. Returns y (complex128) and, if taps, a dict of stage outputs."""
        n, m, K = self.n, self.m, self.K
        x = np.ascontiguousarray(x, dtype=np.complex128)
        assert x.size == n
        y = np.empty(n, np.complex128)
        if not taps:
            lib().orc_execute(self._h, _p(x), _p(y), 1 if inverse else -1, None)
            return y
        G = K * K
        t = dict(digits=np.zeros((2, K, n), np.int32), E=np.zeros((2, K), np.int32),
                 kv=np.zeros(2, np.int32), X=np.zeros((2, K, 2, m), np.uint32),
                 sched=np.zeros((4, self.stride), np.int32),
                 Z=np.zeros((4, G, 2, m), np.uint32), res=np.zeros((4, G, 2, n), np.uint32),
                 crt=np.zeros((4, G, n), np.int64), xdd=np.zeros((4, n), np.float64),
                 counts=np.zeros(3, np.int64), flags=np.zeros(1, np.int32))
        tp = Taps(*[_p(t[f]) for f, _ in Taps._fields_])
        lib().orc_execute(self._h, _p(x), _p(y), 1 if inverse else -1, C.byref(tp))
        return y, t

    def execute_batch(self, x: np.ndarray, inverse: bool = False, nthreads: int = 0):
        x = np.ascontiguousarray(x, dtype=np.complex128)
        B = x.shape[0]
        y = np.empty_like(x)
        used = lib().orc_execute_batch(self._h, B, _p(x), _p(y), 1 if inverse else -1, nthreads)
        return y, used


# --------------------------------------------------------------------------- Fig. 1 alpha
def alpha_formulas(n: int, u_log2_inv: int = 24, p0: int = P0, p1: int = P1) -> dict:
    """The four split widths compared in the paper's Fig. 1, evaluated with
    mpmath at 100 digits in the precision u = 2^-u_log2_inv (single precision: 24):
      ozaki   eq:ozaki-scheme-alpha          floor((log2 u^-1 - log2 n) / 2)
      fft     eq:ozaki-scheme-conv-fft-alpha floor(-(1 + log2 n + log2{(1+u)^3n
              (1+u sqrt5)^(3n+1) (1+u/sqrt2)^3n - 1}) / 2)
      ntt     eq:ozaki-scheme-conv-ntt-alpha floor((log2(p/2) - log2 n) / 2), p = p0
      crt     eq:ozaki-scheme-conv-ntt-crt-alpha floor((log2(p0 p1/2) - log2 n) / 2)
    (TEST INFRASTRUCTURE: tools/sweep.py and tests only.)"""
    import mpmath
    mpmath.mp.dps = 100
    u = mpmath.mpf(2) ** -u_log2_inv
    N = mpmath.mpf(n)
    lg = lambda v: mpmath.log(v, 2)  # noqa: E731
    growth = (1 + u) ** (3 * N) * (1 + u * mpmath.sqrt(5)) ** (3 * N + 1) * \
        (1 + u / mpmath.sqrt(2)) ** (3 * N) - 1
    return {
        "ozaki": int(mpmath.floor((lg(1 / u) - lg(N)) / 2)),
        "fft": int(mpmath.floor(-(1 + lg(N) + lg(growth)) / 2)),
        "ntt": int(mpmath.floor((lg(mpmath.mpf(p0) / 2) - lg(N)) / 2)),
        "crt": int(mpmath.floor((lg(mpmath.mpf(p0) * p1 / 2) - lg(N)) / 2)),
    }


# --------------------------------------------------------------------------- TS helpers
def ts_from_double(d: float) -> TS:
    return lib().orc_ts_from_double(d)


def ts_from_int64(v: int) -> TS:
    return lib().orc_ts_from_int64(v)


def ts_to_double(t: TS) -> float:
    return lib().orc_ts_to_double(t)


def ts_add(a: TS, b: TS) -> TS:
    return lib().orc_ts_add(a, b)


def ts_mul(a: TS, b: TS) -> TS:
    return lib().orc_ts_mul(a, b)


def split_ts(r: np.ndarray, alpha_: int, K: int):
    """orc_split_ts on a [3][len] float32 TS vector (modified in place). Returns (k, digits, E)."""
    r = np.ascontiguousarray(r, dtype=np.float32)
    n = r.shape[1]
    dig = np.zeros((K, n), np.int32)
    E = np.zeros(K, np.int32)
    k = lib().orc_split_ts(n, _p(r), alpha_, K, _p(dig), _p(E))
    return k, dig, E, r
