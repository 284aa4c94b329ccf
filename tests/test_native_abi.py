"""CPU-side checks of the C-ABI library: it loads without a GPU and exports
every symbol declared in include/quakescan_b200.h (no compute calls)."""

import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "quakescan_b200.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qs_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "qs_minmax_signatures" in syms and "qs_lsh_pairs" in syms
    assert len(syms) >= 20


def test_library_exports_every_declared_symbol():
    from paper_1803_09835_b200 import _native
    lib = _native.lib()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert missing == []
    assert set(declared_symbols()) <= set(_native.SIGNATURES)
    assert lib.qs_version().decode().startswith("quakescan-b200")


def test_library_is_sm100a_only():
    import subprocess
    from paper_1803_09835_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


def test_host_pack_helpers():
    """Host-side staging helpers (csrc/qs_host.cu): the saturating uint32 ->
    uint16 narrow and the float64 -> float32 narrow with its exactness flag."""
    import ctypes

    import numpy as np
    from paper_1803_09835_b200 import _native
    lib = _native.lib()
    rng = np.random.default_rng(3)
    for count in (0, 1, 15, 16, 17, 1000, 4099):
        src = rng.integers(0, 4096, count, dtype=np.uint32)
        if count > 2:
            src[1] = 70000
            src[count - 1] = 0xFFFFFFFF
        dst = np.zeros(count, np.uint16)
        assert lib.qs_host_pack_u16(ctypes.c_void_p(src.ctypes.data), ctypes.c_void_p(dst.ctypes.data),
                                    count) == 0
        assert np.array_equal(dst, np.minimum(src, 65535).astype(np.uint16))
    # 12-bit fields: value i in bits [12 i, 12 i + 12) of the byte stream
    for count in (0, 1, 2, 7, 8, 15, 16, 17, 24, 31, 1000, 4099):
        src = rng.integers(0, 4096, count, dtype=np.uint32)
        nbytes = (count * 12 + 7) // 8
        dst = np.full(nbytes + 8, 0xAA, np.uint8)  # the guard bytes must stay untouched
        ok = ctypes.c_int(-1)
        assert lib.qs_host_pack_u12(ctypes.c_void_p(src.ctypes.data), ctypes.c_void_p(dst.ctypes.data),
                                    count, ctypes.byref(ok)) == 0
        assert ok.value == 1
        want = np.zeros(nbytes + 2, np.uint8)
        for i, v in enumerate(src.tolist()):
            bit = 12 * i
            word = int(v) << (bit & 7)
            want[bit >> 3] |= word & 0xFF
            want[(bit >> 3) + 1] |= (word >> 8) & 0xFF
            if word >> 16:
                want[(bit >> 3) + 2] |= word >> 16
        assert np.array_equal(dst[:nbytes], want[:nbytes]), count
        assert np.all(dst[nbytes:] == 0xAA), count
        if count:
            for pos in {0, count // 2, count - 1}:
                bad = src.copy()
                bad[pos] = 4096
                lib.qs_host_pack_u12(ctypes.c_void_p(bad.ctypes.data), ctypes.c_void_p(dst.ctypes.data),
                                     count, ctypes.byref(ok))
                assert ok.value == 0, (count, pos)
    for count in (0, 1, 7, 8, 9, 1000, 4099):
        x = rng.standard_normal(count).astype(np.float32).astype(np.float64)
        out = np.zeros(count, np.float32)
        ok = ctypes.c_int(-1)
        lib.qs_host_pack_f32(ctypes.c_void_p(x.ctypes.data), ctypes.c_void_p(out.ctypes.data), count,
                             ctypes.byref(ok))
        assert ok.value == 1 and np.array_equal(out.astype(np.float64), x)
        if count:
            for bad in (0.1, np.nan, 1e300):
                y = x.copy()
                y[count // 2] = bad
                lib.qs_host_pack_f32(ctypes.c_void_p(y.ctypes.data), ctypes.c_void_p(out.ctypes.data),
                                     count, ctypes.byref(ok))
                assert ok.value == 0
    buf = np.zeros(16, np.uint8)
    assert lib.qs_host_ptr_pinned(ctypes.c_void_p(buf.ctypes.data)) == 0
    assert lib.qs_host_ptr_pinned(None) == 0
