"""Binary codec types + ``decode_module`` on the GPU boundary pass.

Mirrors the decode side of the reference codec (``spirvkit/codec.py``):
``ModuleHeader`` / ``RawInstruction`` (:23-41), ``TypedInt`` / ``TypedFloat``
(:44-58) and ``decode_module`` (:199-231).  The instruction-boundary walk,
magic/endianness normalisation and every error message come from the CUDA
``skg_decode`` kernel; Python only wraps the offsets into the reference's
objects.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _native

MAGIC = 0x07230203
WORD_MASK = 0xFFFFFFFF
HEADER_WORDS = 5


@dataclass(frozen=True)
class ModuleHeader:
    major_version: int
    minor_version: int
    generator_magic: int
    bound: int
    schema: int = 0


@dataclass(frozen=True)
class RawInstruction:
    opcode: int
    operands: tuple = ()

    @property
    def word_count(self) -> int:
        return 1 + len(self.operands)


@dataclass(frozen=True)
class TypedInt:
    value: int
    width: int
    signed: bool = False


@dataclass(frozen=True)
class TypedFloat:
    value: float
    width: int


def decode_module(data: bytes):
    """Split a binary module into (ModuleHeader, [RawInstruction]) on the GPU."""
    header, words, starts = _native.run_decode(bytes(data))
    wl = words.tolist()
    insts = []
    for s in starts.tolist():
        wc = wl[s] >> 16
        insts.append(RawInstruction(wl[s] & 0xFFFF, tuple(wl[s + 1:s + wc])))
    return ModuleHeader(*header), insts
