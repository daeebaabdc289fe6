"""Disassembler API (reference ``spirvkit/disasm.py``) on the CUDA batch kernel.

``disassemble_module`` / ``Disassembler`` keep the reference signatures
(disasm.py:97-127, 392-398); ``disassemble_batch`` is the batch entry point
the bench and batch users call.  All work -- decode, friendly names, float
repr, layout -- happens in ``skg_disasm`` (csrc/skg_disasm.cu).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

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
    return [r if isinstance(r, BaseException) else r.decode("utf-8")
            for r in _native.run_texts("disasm", batch, option_bits(options, strict), spec, ext)]


@dataclass
class RenderContext:
    """disasm.py:57-79: the per-module maps the per-instruction renderer draws from."""
    refs: dict = field(default_factory=dict)          # id -> %ref text
    type_info: dict = field(default_factory=dict)     # type id -> (width, signed, floating)
    value_type: dict = field(default_factory=dict)    # value id -> type id
    import_sets: dict = field(default_factory=dict)   # set id -> import name

    def ref(self, ident: int) -> str:
        return self.refs.get(ident) or f"%{ident}"

    def literal_resolver(self, opdef, decoded):
        if opdef.name == "OpSwitch":
            if not decoded:
                return None
            return self.type_info.get(self.value_type.get(decoded[0].value, -1))
        for operand in decoded:
            if operand.role == "result_type":
                return self.type_info.get(operand.value)
        return None


def _u32(v) -> bool:
    return isinstance(v, int) and 0 <= v <= 0xFFFFFFFF


def _str_words(text: str):
    data = text.encode("utf-8") + b"\0"
    data += b"\0" * (-len(data) % 4)
    return list(struct.unpack(f"<{len(data) // 4}I", data))


def disassemble_validate_batch(modules, options=None, spec=None, ext=None, strict=False):
    """Fused decode -> validate -> disassemble: every module is read and
    decoded once (skg_disasm_validate) for both results.  -> list of (text | exception,
    list[Diagnostic] | exception) pairs, each element exactly what
    disassemble_batch / validate_batch return for the module."""
    from .validate import _parse
    batch = modules if isinstance(modules, _native.DeviceBatch) else \
        _native.DeviceBatch.from_modules([bytes(m) for m in modules])
    texts, diags = _native.run_texts_pipeline(batch, option_bits(options, strict), spec, ext)
    return [(t if isinstance(t, BaseException) else t.decode("utf-8"),
             d if isinstance(d, BaseException) else _parse(d.decode("utf-8"))) for t, d in zip(texts, diags)]


def format_instruction(spec, inst, context=None, ext=None) -> str:
    """One raw instruction as one plain-text line (reference disasm.py:380-389).

    Rendered by skg_disasm on a synthesized module: the instruction, preceded by
    the declarations that make the kernel's own prescan reproduce the context's
    maps -- OpTypeInt / OpTypeFloat per ``type_info`` entry, OpUndef per
    ``value_type`` entry and an OpExtInstImport "OpenCL.std" per such
    ``import_sets`` entry (only when an ``ext`` grammar is given, as the reference
    names extended instructions only then) -- with no header, no indentation and
    numeric ids, except that the context's ``refs`` are passed to the kernel as
    explicit ref texts (skg_disasm_refs).  Decode errors raise the reference's
    exceptions."""
    import numpy as np
    from . import grammar as _grammar
    spec = spec if spec is not None else _grammar.load_pinned()
    spec.instruction(inst.opcode)          # NotFoundError outside the grammar, as the reference
    ops = [int(w) & 0xFFFFFFFF for w in inst.operands]
    if len(ops) + 1 > 0xFFFF:
        raise ValueError("format_instruction: more than 65534 operand words")
    ctx = context if context is not None else RenderContext()
    pre, ids = [], list(ops)
    for tid, info in ctx.type_info.items():
        if not _u32(tid) or info is None:
            continue
        width, signed, floating = info
        if floating:
            pre += [(3 << 16) | 22, tid, int(width) & 0xFFFFFFFF]                       # OpTypeFloat
        else:
            pre += [(4 << 16) | 21, tid, int(width) & 0xFFFFFFFF, 1 if signed else 0]    # OpTypeInt
        ids.append(tid)
    for vid, tid in ctx.value_type.items():
        if _u32(vid) and _u32(tid):
            pre += [(3 << 16) | 1, tid, vid]                                            # OpUndef
            ids += [vid, tid]
    if ext is not None:
        for sid, name in ctx.import_sets.items():
            if _u32(sid) and name == "OpenCL.std":
                w = _str_words(name)
                pre += [((2 + len(w)) << 16) | 11, sid, *w]                              # OpExtInstImport
                ids.append(sid)
    bound = min(max(ids, default=0) + 1, 0xFFFFFFFF)
    words = [0x07230203, 0x00010200, 0, bound, 0, *pre, ((len(ops) + 1) << 16) | (int(inst.opcode) & 0xFFFF), *ops]
    module = struct.pack(f"<{len(words)}I", *words)
    refs = sorted((k, v.encode("utf-8", "surrogatepass")) for k, v in ctx.refs.items() if _u32(k) and v)
    opts = DisassemblerOptions(inline_names=False, no_indent=True, no_header=True)
    batch = _native.DeviceBatch.from_modules([module])
    dev_refs = None
    if refs:
        blob = b"".join(r for _, r in refs)
        tab = np.zeros((len(refs), 3), dtype=np.uint32)
        pos = 0
        for k, (i, r) in enumerate(refs):
            tab[k] = (i, pos, len(r))
            pos += len(r)
        dev_refs = (_native._dev(tab.reshape(-1), np.uint32), _native._dev(np.frombuffer(blob, np.uint8), np.uint8),
                    len(refs))
    res = _native.run_texts("disasm", batch, option_bits(opts), spec, ext, refs=dev_refs)[0]
    if isinstance(res, BaseException):
        raise res
    out = res.decode("utf-8")
    return out.rsplit("\n", 2)[-2] if out.endswith("\n") else out


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


class DisasmSession:
    """Host-buffer batch API: packed modules in, packed text out.

    ``run(data, offsets, lengths)`` takes a host byte arena (module starts
    16-byte aligned) with int64 offsets/lengths, copies it to the device from
    pinned memory, disassembles every module and copies the used text arena,
    the per-module (offset, length) spans and statuses back (pinned).  Buffers
    are reused across calls of the same shape.  Returns (text uint8[],
    spans int64[n, 2], status int32[n]); module m's text is
    text[spans[m, 0] : spans[m, 0] + spans[m, 1]].  Failing modules have
    status != 0 and an empty span; ``errors()`` maps them to exceptions.
    """

    def __init__(self, options=None, spec=None, ext=None, strict=False):
        self.opts = option_bits(options, strict)
        self.spec, self.ext = spec, ext
        self._key = None

    def _prepare(self, data, offsets, lengths):
        import torch
        key = (data.nbytes, len(offsets), int(lengths.max()) if len(lengths) else 0)
        if key == self._key:
            return
        n = len(offsets)
        self.h_data = torch.empty(data.nbytes, dtype=torch.uint8).pin_memory()
        self.h_meta = torch.empty(2 * n, dtype=torch.int64).pin_memory()
        self.d_data = torch.empty(data.nbytes, dtype=torch.uint8, device="cuda")
        self.d_meta = torch.empty(2 * n, dtype=torch.int64, device="cuda")
        self.batch = _native.DeviceBatch(self.d_data, self.d_meta[:n], self.d_meta[n:],
                                         key[2] // 4, int(lengths.sum()))
        self.plan = _native.DisasmPlan(self.batch, self.opts, self.spec, self.ext,
                                       text_cap=6 * int(lengths.sum()) + 4096)
        self.h_span = torch.empty(2 * max(n, 1), dtype=torch.int64).pin_memory()
        self.h_status = torch.empty(max(n, 1), dtype=torch.int32).pin_memory()
        self.h_counts = torch.empty(8, dtype=torch.int32).pin_memory()
        self.h_text = torch.empty(0, dtype=torch.uint8).pin_memory()
        self._key = key

    def stage(self, data, offsets, lengths):
        """Host arrays -> pinned staging buffers (outside any timed region)."""
        import numpy as np
        self._prepare(data, offsets, lengths)
        n = len(offsets)
        self.h_data.numpy()[:] = np.frombuffer(memoryview(data).cast("B"), dtype=np.uint8)
        self.h_meta.numpy()[:n] = offsets
        self.h_meta.numpy()[n:] = lengths

    def run_staged(self):
        """H2D of the staged inputs, kernel, D2H of text + spans + status."""
        import torch
        self.d_data.copy_(self.h_data, non_blocking=True)
        self.d_meta.copy_(self.h_meta, non_blocking=True)
        self.plan.launch()
        n = self.batch.n
        self.h_span.copy_(self.plan.span, non_blocking=True)
        self.h_status.copy_(self.plan.status, non_blocking=True)
        self.h_counts.copy_(self.plan.ws[:32].view(torch.int32), non_blocking=True)
        torch.cuda.current_stream().synchronize()
        c = self.h_counts.numpy()
        used = int(c[4]) & 0xFFFFFFFF | (int(c[5]) & 0xFFFFFFFF) << 32
        if c[2]:   # arena overflow: grow and rerun
            self.plan.grow(used)
            self.plan.launch()
            self.h_span.copy_(self.plan.span, non_blocking=True)
        if self.h_text.numel() < used:
            self.h_text = torch.empty(used, dtype=torch.uint8).pin_memory()
        self.h_text[:used].copy_(self.plan.text[:used], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return (self.h_text[:used].numpy(), self.h_span[: 2 * n].numpy().reshape(n, 2),
                self.h_status[:n].numpy())

    def run(self, data, offsets, lengths):
        self.stage(data, offsets, lengths)
        return self.run_staged()

    def errors(self):
        """module index -> exception instance for the last run."""
        info = self.plan.check()
        ne = min(info["errors"], self.plan.ecap)
        return _native.decode_errors(self.plan.errs[: ne * 256].cpu().numpy()) if ne else {}
