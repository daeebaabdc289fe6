"""Assembler API (reference ``spirvkit/asm.py``) on the CUDA batch kernel.

``assemble_module`` / ``Assembler.assemble`` keep the reference signatures
(asm.py:123-180, 365-368); ``assemble_batch`` is the batch entry point.  The
whole pipeline -- splitlines, tokenizer, symbol table, header comments, width
scans, Encoder slot walk, builder routing and serialization, every diagnostic
-- runs in ``skg_asm`` (csrc/skg_asm.cu).  Results are the module bytes or the
exception the reference raises (AssemblyError with its AsmDiagnostic list,
ValueError, OverflowError, StructureError, SerializationError, CodecError).
"""

from __future__ import annotations

from . import _native


def assemble_batch(texts, spec=None, ext=None, default_version=(1, 2)):
    """list[str] -> list[bytes | Exception] (exception instances, not raised)."""
    return _native.run_asm(list(texts), spec, ext, default_version)


class Assembler:
    def __init__(self, spec=None, ext=None, default_version=(1, 2)):
        self.spec, self.ext = spec, ext
        self.default_version = default_version

    def assemble(self, text: str) -> bytes:
        out = assemble_batch([text], self.spec, self.ext, self.default_version)[0]
        if isinstance(out, BaseException):
            raise out
        return out


def assemble_module(text: str, spec=None, ext=None) -> bytes:
    return Assembler(spec=spec, ext=ext).assemble(text)
