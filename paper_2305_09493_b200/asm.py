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


class RoundTripSession:
    """Host-buffer batch API for binary -> text -> binary (disassemble + assemble).

    ``stage(data, offsets, lengths)`` fills pinned staging buffers (outside any
    timed region); ``run_staged()`` copies the modules to the device, runs
    ``skg_disasm`` and then ``skg_asm`` directly on the disassembler's text
    arena (its interleaved spans are read with stride 2, no host work in
    between), and copies back both results: the text arena with its spans and
    the re-assembled binaries with their spans and statuses.
    """

    def __init__(self, options=None, spec=None, ext=None):
        from .disasm import DisasmSession
        self.dis = DisasmSession(options, spec, ext)
        self.spec, self.ext = spec, ext
        self.plan = None

    def stage(self, data, offsets, lengths):
        self.dis.stage(data, offsets, lengths)
        self.total_in = int(lengths.sum())

    def _asm_plan(self, max_text):
        import torch
        d = self.dis.plan
        n = d.batch.n
        tb = _native.DeviceBatch(d.text, d.span[0::2], d.span[1::2], (max_text + 3) // 4, 0)
        tb.n = n
        if self.plan is None or self.plan.batch.n != n or self.plan.slot < _native.lib().skg_asm_slot_hint(
                max_text + 16):
            self.plan = _native.AsmPlan(tb, self.spec, self.ext, out_cap=self.total_in + 64 * n + 4096,
                                        stride=2)
            self.h_out = torch.empty(self.plan.cap, dtype=torch.uint8).pin_memory()
            self.h_span = torch.empty(2 * n, dtype=torch.int64).pin_memory()
            self.h_status = torch.empty(n, dtype=torch.int32).pin_memory()
        self.plan.batch = tb
        return self.plan

    def run_staged(self, max_text=None):
        import torch
        text, spans, status = self.dis.run_staged()
        if max_text is None:
            max_text = int(spans[:, 1].max()) if len(spans) else 0
        p = self._asm_plan(max_text)
        p.launch()
        counts = torch.empty(8, dtype=torch.int32).pin_memory()
        counts.copy_(p.ws[:32].view(torch.int32), non_blocking=True)
        n = p.batch.n
        self.h_span.copy_(p.span[: 2 * n], non_blocking=True)
        self.h_status.copy_(p.status[:n], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        c = counts.numpy()
        used = int(c[4]) & 0xFFFFFFFF | (int(c[5]) & 0xFFFFFFFF) << 32
        if c[2]:
            p.grow(used)
            self.h_out = torch.empty(p.cap, dtype=torch.uint8).pin_memory()
            p.launch()
            self.h_span.copy_(p.span[: 2 * n], non_blocking=True)
            self.h_status.copy_(p.status[:n], non_blocking=True)
        self.h_out[:used].copy_(p.out[:used], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return (text, spans, status, self.h_out[:used].numpy(),
                self.h_span[: 2 * n].numpy().reshape(n, 2), self.h_status[:n].numpy())
