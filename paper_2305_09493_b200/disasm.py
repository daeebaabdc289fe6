"""Disassembler API (reference ``spirvkit/disasm.py``) on the CUDA batch kernel.

``disassemble_module`` / ``Disassembler`` keep the reference signatures
(disasm.py:97-127, 392-398); ``disassemble_batch`` is the batch entry point
the bench and batch users call.  All work -- decode, friendly names, float
repr, layout -- happens in ``skg_disasm`` (csrc/skg_disasm.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _native


@dataclass
class DisassemblerOptions:
    highlight: bool = False
    inline_names: bool = True
    no_indent: bool = False
    group: bool = False
    no_header: bool = False


def option_bits(options, strict=False) -> int:
    o = options if options is not None else DisassemblerOptions()
    bits = 0
    bits |= _native.OPT_HIGHLIGHT if o.highlight else 0
    bits |= _native.OPT_INLINE if o.inline_names else 0
    bits |= _native.OPT_NO_INDENT if o.no_indent else 0
    bits |= _native.OPT_GROUP if o.group else 0
    bits |= _native.OPT_NO_HEADER if o.no_header else 0
    bits |= _native.OPT_STRICT if strict else 0
    return bits


def disassemble_batch(modules, options=None, spec=None, ext=None, strict=False):
    """list[bytes] -> list[str | Exception] (exception instances, not raised)."""
    batch = modules if isinstance(modules, _native.DeviceBatch) else \
        _native.DeviceBatch.from_modules([bytes(m) for m in modules])
    res = _native.run_disasm(batch, option_bits(options, strict), spec, ext)
    return [r if isinstance(r, BaseException) else r.decode("utf-8")
            for r in _native.fetch_texts(res, batch.n)]


class Disassembler:
    def __init__(self, spec=None, ext=None, options=None, strict=False):
        self.spec, self.ext = spec, ext
        self.options = options if options is not None else DisassemblerOptions()
        self.strict = strict

    def to_text(self, data: bytes) -> str:
        out = disassemble_batch([data], self.options, self.spec, self.ext, self.strict)[0]
        if isinstance(out, BaseException):
            raise out
        return out

    def disassemble(self, data: bytes, sink) -> int:
        text = self.to_text(data)
        sink.write(text)
        return text.count("\n")


def disassemble_module(data: bytes, options=None, sink=None, spec=None, ext=None,
                       strict: bool = False):
    tool = Disassembler(spec=spec, ext=ext, options=options, strict=strict)
    return tool.to_text(data) if sink is None else tool.disassemble(data, sink)
