"""CPU-side checks of the native boundary (no GPU needed)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2305_09493_b200" / "libskgpu.so"
HEADER = ROOT / "include" / "skgpu.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(skg_[a-z_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("skg_tables_create", "skg_disasm", "skg_validate", "skg_decode", "skg_workspace_bytes"):
        assert s in syms


@pytest.mark.skipif(not LIB.exists(), reason="library not built (run __graft_entry__.build())")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(LIB))
    for s in declared_symbols():
        assert hasattr(lib, s), s
    lib.skg_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.skg_version()


def test_tables_pack_roundtrip_lookups():
    """The device blob encodes the same lookups as the grammar dicts."""
    import numpy as np
    from paper_2305_09493_b200 import grammar, tables
    spec = grammar.load_pinned()
    t = tables.pack(spec)
    b = t.blob
    h = b[:64]
    inst, opidx_off, max_op = h[3], h[5], h[4]
    opidx = b[opidx_off: opidx_off + (max_op + 2) // 2 + 1].view(np.uint16)
    strings = b[h[12]: h[12] + (h[13] + 3) // 4].tobytes()[: h[13]]
    for op in range(max_op + 1):
        i = int(opidx[op])
        if spec.has_instruction(op):
            rec = b[inst + 8 * i: inst + 8 * i + 8]
            name = strings[rec[0]: rec[0] + (rec[1] & 0xFFFF)].decode()
            assert name == spec.instruction(op).name
        else:
            assert i == 0xFFFF
