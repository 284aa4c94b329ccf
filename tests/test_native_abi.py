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
