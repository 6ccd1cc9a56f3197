"""The C-ABI library builds, loads and exports every symbol include/ozfft.h declares.
No compute calls (this runs on the CPU-only container)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "ozfft.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ozfft_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2603_29129_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_exports_match_header(lib):
    import paper_2603_29129_b200 as oz
    syms = header_symbols()
    assert len(syms) >= 13
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(oz.EXPORTS) == syms


def test_status_strings_and_version(lib):
    lib.ozfft_status_string.restype = ctypes.c_char_p
    lib.ozfft_version.restype = ctypes.c_char_p
    assert lib.ozfft_status_string(0) == b"OZFFT_OK"
    assert lib.ozfft_status_string(7) == b"OZFFT_ERR_CUDA"
    assert lib.ozfft_version().startswith(b"ozfft sm_100a")


def test_sass_is_sm100a():
    """The shared object carries sm_100a SASS (cuobjdump runs without a GPU)."""
    import subprocess
    from paper_2603_29129_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.build()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_plan_create_validation(lib):
    """Host-side argument checks of ozfft_plan_create (no device memory touched)."""
    import paper_2603_29129_b200 as oz
    L = oz.load_library()

    def create(**kw):
        d = oz.PlanDesc(**{"n": 1024, "batch": 1, "K": 3, "L": 3, "p0": 0, "p1": 0,
                           "device": 0, "conv_mode": 0, "accum_mode": 0, "precision": 0,
                           "max_workspace_bytes": 0, **kw})
        h = ctypes.c_void_p()
        st = L.ozfft_plan_create(ctypes.byref(d), ctypes.byref(h))
        if st == 0:
            info = oz.PlanInfo()
            assert L.ozfft_plan_get_info(h, ctypes.byref(info)) == 0
            L.ozfft_plan_destroy(h)
            return st, info
        return st, None

    st, info = create()
    assert st == 0 and info.m == 2048 and info.alpha == 24 and info.rho == 29
    st, info = create(n=1 << 18, batch=16)
    assert st == 0 and info.m == 1 << 19 and info.alpha == 20
    assert info.log2_rows + info.log2_cols == 19
    st, info = create(n=100003, batch=32)
    assert st == 0 and info.m == 1 << 18 and info.alpha == 21
    assert create(n=0)[0] == 1
    assert create(batch=0)[0] == 1
    assert create(K=9)[0] == 1
    assert create(p0=2130706433, p1=2130706433)[0] == 3
    assert create(p0=2130706431)[0] == 3          # not prime
    assert create(n=(1 << 23) + 1)[0] == 2        # m = 2^25 > the primes' limit 2^24
    st, info = create(n=1)
    assert st == 0 and info.m == 1
    # cyclic Bluestein: m = n for power-of-two n, same alpha as the padded plan
    st, info = create(n=1 << 18, batch=16, conv_mode=1)
    assert st == 0 and info.m == 1 << 18 and info.alpha == 20 and info.conv_mode == 1
    st, info = create(n=1 << 20, conv_mode=1)     # m = 2^20
    assert st == 0 and info.m == 1 << 20
    st, info = create(n=1 << 21)                  # m = 2^22 = 2^10 x 2^12
    assert st == 0 and info.m == 1 << 22 and info.log2_rows == 10 and info.log2_cols == 12
    st, info = create(n=(1 << 21) + 1)            # m = 2^23 = 2^11 x 2^12
    assert st == 0 and info.m == 1 << 23 and info.log2_rows == 11 and info.log2_cols == 12
    st, info = create(n=1 << 23)                  # m = 2^24 = 2^12 x 2^12: the primes' limit
    assert st == 0 and info.m == 1 << 24 and info.log2_rows == 12 and info.log2_cols == 12
    assert create(n=1 << 22, conv_mode=1)[0] == 0
    assert create(n=100003, conv_mode=1)[0] == 2  # not a power of two
    assert create(n=1024, conv_mode=2)[0] == 1    # unknown mode
    # complex-image accumulation: alpha from the bound 2 L n 4^alpha < P/2
    st, info = create(n=1 << 18, accum_mode=1)
    assert st == 0 and info.alpha == 20 and info.accum_mode == 1
    st, info = create(n=1 << 17, accum_mode=1)
    assert st == 0 and info.alpha == 20           # the real-mode value at 2n
    assert create(n=1024, accum_mode=2)[0] == 1
    assert create(n=1024, precision=2)[0] == 1
    st, info = create(n=1024, precision=1)
    assert st == 0 and info.precision == 1 and info.alpha == 24
    assert create(n=1024, precision=1, accum_mode=1)[0] == 1  # TS with the real mode only
    assert create(n=1024, accum_mode=1, p0=2130706433, p1=2013265921)[0] == 0  # 15*2^27+1
    assert create(n=1024, accum_mode=1, p0=2130706433, p1=2147483647)[0] == 3  # 2^31-1 = 3 mod 4


def test_entry_point_errors_without_device(lib):
    """Synchronous argument errors of the execute / bind / shard / stats entry points (no
    device memory is touched before these checks)."""
    import paper_2603_29129_b200 as oz
    L = oz.load_library()
    d = oz.PlanDesc(n=1000, batch=2, K=3, L=3, p0=0, p1=0, device=0, conv_mode=0, accum_mode=0,
                    precision=0, max_workspace_bytes=0)
    h = ctypes.c_void_p()
    assert L.ozfft_plan_create(ctypes.byref(d), ctypes.byref(h)) == 0
    buf = ctypes.c_void_p(1 << 20)  # never dereferenced: the checks fail first
    assert L.ozfft_execute(h, buf, buf, -1, None) == 5          # NOT_BOUND
    assert L.ozfft_execute_host(h, buf, buf, -1, None) == 5
    g = ctypes.c_int32(0)
    assert L.ozfft_shard_partial(h, 0, 2, buf, -1, buf, ctypes.byref(g), None) == 5
    assert L.ozfft_shard_residue_bytes(h, 0) == 8 * 9 * 1000 * 4   # K*K capacity
    assert L.ozfft_shard_residue_bytes(h, 5) == 160 * 1000          # 8 g n words
    st = oz.ExecStats()
    assert L.ozfft_last_stats(h, ctypes.byref(st), None) == 5
    assert L.ozfft_plan_bind(h, None, 0, None, 0, None) == 1    # null buffers
    assert L.ozfft_plan_bind(h, ctypes.c_void_p(257), 1 << 30, ctypes.c_void_p(512), 1 << 30, None) == 6
    info = oz.PlanInfo()
    assert L.ozfft_plan_get_info(h, ctypes.byref(info)) == 0
    assert L.ozfft_plan_bind(h, ctypes.c_void_p(256), info.persistent_bytes - 1, ctypes.c_void_p(512),
                             info.workspace_bytes, None) == 9   # BUFFER_TOO_SMALL
    assert L.ozfft_execute(None, buf, buf, -1, None) == 1
    assert b"null plan" in L.ozfft_last_error_string()
    assert L.ozfft_status_string(9) == b"OZFFT_ERR_BUFFER_TOO_SMALL"
    assert L.ozfft_plan_destroy(h) == 0
    assert L.ozfft_plan_destroy(None) == 0


def _raw_plan(L, **kw):
    import paper_2603_29129_b200 as oz
    d = oz.PlanDesc(**{"n": 1024, "batch": 1, "K": 3, "L": 3, "p0": 0, "p1": 0, "device": 0,
                       "conv_mode": 0, "accum_mode": 0, "precision": 0,
                       "max_workspace_bytes": 0, **kw})
    h = ctypes.c_void_p()
    st = L.ozfft_plan_create(ctypes.byref(d), ctypes.byref(h))
    return st, h


def test_host_subbatches_fit_the_chunk(lib):
    """ozfft_execute_host's sub-batches: every one fits a workspace chunk and they cover the
    batch.  Regression: the m <= 2^16 schedule B/8, B/4, ... gave a middle
    sub-batch of ceil(rest/3) > chunk for B = 8k + 7 with chunk = 2k + 2 (e.g. B = 15,
    chunk 4 -> 5), overrunning the workspace slot."""
    import paper_2603_29129_b200 as oz
    L = oz.load_library()
    info = oz.PlanInfo()

    def ok(n, B, cap):
        st, h = _raw_plan(L, n=n, batch=B, max_workspace_bytes=cap)
        if st == 0:
            L.ozfft_plan_destroy(h)
        return st == 0

    for n, Bs in ((1000, list(range(1, 70)) + [127, 199, 1024]), (3000, [7, 15, 23, 31, 64]),
                  (20000, [7, 15, 23])):
        st, h = _raw_plan(L, n=n, batch=1)
        assert st == 0
        assert L.ozfft_plan_get_info(h, ctypes.byref(info)) == 0
        L.ozfft_plan_destroy(h)
        per = info.workspace_bytes  # >= one transform's chunked regions
        for B in Bs:
            lo, hi = 0, per + 64 * B * 1300 + (1 << 20)  # smallest cap that takes one transform
            assert ok(n, B, hi)
            while hi - lo > per // 16:
                mid = (lo + hi) // 2
                lo, hi = (lo, mid) if ok(n, B, mid) else (mid, hi)
            for chunk_target in sorted({1, 2, 3, 4, 6, max(1, B // 4 + 1), B}):
                cap = hi + per * (chunk_target - 1) + per // 2  # about chunk_target transforms
                st, h = _raw_plan(L, n=n, batch=B, max_workspace_bytes=cap)
                assert st == 0, (n, B, chunk_target)
                assert L.ozfft_plan_get_info(h, ctypes.byref(info)) == 0
                assert info.workspace_bytes <= cap, (n, B, info.workspace_bytes, cap)
                cnt = L.ozfft_host_subbatches(h, None, 0)
                sizes = (ctypes.c_int64 * cnt)()
                assert L.ozfft_host_subbatches(h, sizes, cnt) == cnt
                sz = list(sizes)
                L.ozfft_plan_destroy(h)
                assert sum(sz) == B and min(sz) >= 1, (n, B, sz)
                assert max(sz) <= info.chunk, (n, B, info.chunk, sz)


def test_workspace_cap_too_small(lib):
    """A max_workspace_bytes below one transform's workspace is refused (BUFFER_TOO_SMALL)
    instead of silently exceeding the cap."""
    import paper_2603_29129_b200 as oz
    L = oz.load_library()
    st, h = _raw_plan(L, n=1 << 14, batch=4, max_workspace_bytes=4096)
    assert st == 9
    assert L.ozfft_host_subbatches(None, None, 0) == -1
