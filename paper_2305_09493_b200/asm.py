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

from dataclasses import dataclass

from . import _native
from .errors import AsmDiagnostic, AssemblyError


@dataclass(frozen=True)
class Token:
    """asm.py:34-38."""
    text: str
    column: int  # 1-based (code points)
    is_string: bool = False


@dataclass
class TextInstruction:
    """asm.py:41-48: one parsed source line."""
    result: Token | None
    opname: Token
    operands: list
    line: int


def tokenize_lines(lines, first_lineno: int = 1):
    """Batch tokenize_line over many lines on the GPU (skg_tokenize, one thread per
    line): list[str] -> list[TextInstruction | None | AssemblyError] (line numbers
    first_lineno, first_lineno + 1, ...; exception instances, not raised)."""
    raws = [ln.encode("utf-8", "surrogatepass") for ln in lines]
    out = []
    for k, (kind, toks, col) in enumerate(_native.run_tokenize(raws)):
        lineno = first_lineno + k
        if kind == 3:
            out.append(AssemblyError([AsmDiagnostic(lineno, col, "unterminated string literal")]))
            continue
        if kind == 0:
            out.append(None)
            continue
        tokens = [Token(b.decode("utf-8", "surrogatepass"), c, s) for b, c, s in toks]
        result = None
        if kind == 2:
            result, tokens = tokens[0], tokens[2:]
        out.append(TextInstruction(result=result, opname=tokens[0], operands=tokens[1:], line=lineno))
    return out


def tokenize_line(line: str, lineno: int = 1):
    """asm.py:51-90 on the GPU: None for blank / comment lines, AssemblyError for an
    unterminated string literal (column of the opening quote)."""
    r = tokenize_lines([line], lineno)[0]
    if isinstance(r, BaseException):
        raise r
    return r


class SymbolTable:
    """asm.py:93-120: names <-> ids of a builder module.  Numeric names (%13) pin
    their value (module.reserve_id), symbolic names take module.new_id() at first
    mention.  The assembler kernel runs this logic on the device for whole
    documents (skg_asm phase D: a name hash map, the reservation bitmap and a
    select over unreserved ids); this class is the reference's per-name interface
    over a caller-owned builder module."""

    def __init__(self, module):
        self.module = module
        self.by_name = {}
        self.by_id = {}

    def resolve(self, name: str):
        if not name.startswith("%") or len(name) == 1:
            raise ValueError(f"expected an id like %name, got {name!r}")
        hit = self.by_name.get(name)
        if hit is not None:
            return hit
        body = name[1:]
        ident = self.module.reserve_id(int(body)) if body.isdigit() else self.module.new_id()
        self.by_name[name] = ident
        self.by_id[int(ident)] = name
        return ident


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

    ``stage(data, offsets, lengths)`` copies the host batch (module starts
    16-byte aligned in one byte arena, int64 offsets/lengths) into pinned
    staging buffers and sizes the device plans with one untimed pass.
    ``run_staged()`` then runs the whole round trip as a pipeline over
    ``chunks`` contiguous module ranges on three CUDA streams: the H2D copy of
    chunk k+1 and the D2H copies of chunk k-1's text and binaries overlap
    ``skg_disasm`` + ``skg_asm`` of chunk k (the assembler reads the
    disassembler's text arena directly, spans with stride 2).  Returns
    (text uint8[], text spans int64[n, 2], disasm status int32[n],
    binaries uint8[], binary spans int64[n, 2], asm status int32[n]) with spans
    relative to the returned arenas.
    """

    def __init__(self, options=None, spec=None, ext=None, chunks=8):
        from .disasm import DisassemblerOptions, option_bits
        self.opts = option_bits(options if options is not None else DisassemblerOptions())
        self.spec, self.ext = spec, ext
        self.nchunks = max(1, int(chunks))
        self.chunks = None

    def stage(self, data, offsets, lengths):
        import numpy as np
        import torch
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        lengths = np.ascontiguousarray(lengths, dtype=np.int64)
        n = len(offsets)
        self.n = n
        self.h_data = torch.empty(max(data.nbytes, 16), dtype=torch.uint8).pin_memory()
        self.h_data.numpy()[: data.nbytes] = np.frombuffer(memoryview(data).cast("B"), dtype=np.uint8)
        self.h_meta = torch.empty(2 * max(n, 1), dtype=torch.int64).pin_memory()
        self.h_meta.numpy()[:n] = offsets
        self.h_meta.numpy()[n: 2 * n] = lengths
        self.d_data = torch.empty(max(data.nbytes, 16), dtype=torch.uint8, device="cuda")
        self.d_meta = torch.empty(2 * max(n, 1), dtype=torch.int64, device="cuda")
        self.d_meta.copy_(self.h_meta)
        self.d_data.copy_(self.h_data)
        # contiguous module ranges by bytes; the first and last chunks are half size, so the
        # copy-in before the first kernel and the copy-out after the last one are short
        cum = np.cumsum(lengths) if n else np.zeros(0, dtype=np.int64)
        total = int(cum[-1]) if n else 0
        w = np.ones(self.nchunks)
        if self.nchunks >= 3:
            w[0] = w[-1] = 0.5
        frac = np.cumsum(w) / w.sum()
        cuts = [0]
        for k in range(1, self.nchunks):
            cuts.append(int(np.searchsorted(cum, total * frac[k - 1])))
        cuts.append(n)
        cuts = sorted(set(cuts))
        self.chunks = []
        dis_ws = asm_ws = None
        for a, b in zip(cuts[:-1], cuts[1:]):
            if b <= a:
                continue
            c = _Chunk(self, a, b, offsets, lengths, dis_ws, asm_ws)
            dis_ws, asm_ws = c.dplan.ws, c.aplan.ws
            self.chunks.append(c)
        torch.cuda.synchronize()
        self.h_text = torch.empty(max(sum(c.text_used for c in self.chunks), 16), dtype=torch.uint8).pin_memory()
        self.h_out = torch.empty(max(sum(c.out_used for c in self.chunks), 16), dtype=torch.uint8).pin_memory()
        self.h_tspan = torch.empty(2 * max(n, 1), dtype=torch.int64).pin_memory()
        self.h_bspan = torch.empty(2 * max(n, 1), dtype=torch.int64).pin_memory()
        self.h_tst = torch.empty(max(n, 1), dtype=torch.int32).pin_memory()
        self.h_bst = torch.empty(max(n, 1), dtype=torch.int32).pin_memory()
        self.h_counts = torch.empty(max(len(self.chunks), 1) * 16, dtype=torch.int32).pin_memory()
        self.d_counts = torch.zeros(max(len(self.chunks), 1) * 16, dtype=torch.int32, device="cuda")
        tb = ob = 0
        for c in self.chunks:
            c.text_base, c.out_base = tb, ob
            tb += c.text_used
            ob += c.out_used
        self.s_in, self.s_out = torch.cuda.Stream(), torch.cuda.Stream()

    def run_staged(self, max_text=None):
        import numpy as np
        import torch
        if self.chunks is None:
            raise RuntimeError("stage() first")
        if self.n == 0 or not self.chunks:
            z8, z32 = np.zeros(0, np.uint8), np.zeros(0, np.int32)
            zs = np.zeros((0, 2), np.int64)
            return z8, zs, z32, z8.copy(), zs.copy(), z32.copy()
        comp = torch.cuda.current_stream()
        cs = _native.ctypes.c_void_p(comp.cuda_stream)
        evs = []
        for k, c in enumerate(self.chunks):
            ev_in, ev_dis, ev_asm = torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event()
            with torch.cuda.stream(self.s_in):
                self.d_data[c.b0:c.b1].copy_(self.h_data[c.b0:c.b1], non_blocking=True)
                ev_in.record(self.s_in)
            comp.wait_event(ev_in)
            c.dplan.launch(cs)
            self.d_counts[16 * k: 16 * k + 8].copy_(c.dplan.ws[:32].view(torch.int32), non_blocking=True)
            ev_dis.record(comp)
            c.aplan.launch(cs)
            self.d_counts[16 * k + 8: 16 * k + 16].copy_(c.aplan.ws[:32].view(torch.int32), non_blocking=True)
            ev_asm.record(comp)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(ev_dis)
                self.h_text[c.text_base:c.text_base + c.text_used].copy_(c.dplan.text[: c.text_used],
                                                                          non_blocking=True)
                self.h_tspan[2 * c.m0:2 * c.m1].copy_(c.dplan.span[: 2 * c.n], non_blocking=True)
                self.h_tst[c.m0:c.m1].copy_(c.dplan.status[: c.n], non_blocking=True)
                self.s_out.wait_event(ev_asm)
                self.h_out[c.out_base:c.out_base + c.out_used].copy_(c.aplan.out[: c.out_used], non_blocking=True)
                self.h_bspan[2 * c.m0:2 * c.m1].copy_(c.aplan.span[: 2 * c.n], non_blocking=True)
                self.h_bst[c.m0:c.m1].copy_(c.aplan.status[: c.n], non_blocking=True)
            evs.append(ev_asm)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(evs[-1])
            self.h_counts.copy_(self.d_counts, non_blocking=True)
        self.s_out.synchronize()
        cnt = self.h_counts.numpy().reshape(-1, 16)
        for k, c in enumerate(self.chunks):
            dused = int(cnt[k, 4]) & 0xFFFFFFFF | (int(cnt[k, 5]) & 0xFFFFFFFF) << 32
            aused = int(cnt[k, 12]) & 0xFFFFFFFF | (int(cnt[k, 13]) & 0xFFFFFFFF) << 32
            if cnt[k, 2] or cnt[k, 10] or dused != c.text_used or aused != c.out_used:
                raise RuntimeError("RoundTripSession: staged sizes changed; call stage() again")
        n = self.n
        tspan = self.h_tspan[: 2 * n].numpy().reshape(n, 2).copy()
        bspan = self.h_bspan[: 2 * n].numpy().reshape(n, 2).copy()
        for c in self.chunks:   # chunk-relative -> arena-relative offsets
            tspan[c.m0:c.m1, 0] += c.text_base
            bspan[c.m0:c.m1, 0] += c.out_base
        return (self.h_text[: sum(c.text_used for c in self.chunks)].numpy(), tspan,
                self.h_tst[:n].numpy(), self.h_out[: sum(c.out_used for c in self.chunks)].numpy(), bspan,
                self.h_bst[:n].numpy())


class _Chunk:
    """One contiguous module range of a RoundTripSession with its fitted plans."""

    def __init__(self, sess, m0, m1, offsets, lengths, dis_ws, asm_ws):
        self.m0, self.m1, self.n = m0, m1, m1 - m0
        self.b0 = int(offsets[m0])
        self.b1 = int((offsets[m1 - 1] + lengths[m1 - 1] + 15) // 16 * 16)
        mw = int(lengths[m0:m1].max()) // 4
        batch = _native.DeviceBatch(sess.d_data, sess.d_meta[m0:m1], sess.d_meta[sess.n + m0: sess.n + m1],
                                    mw, int(lengths[m0:m1].sum()))
        self.dplan = _native.DisasmPlan(batch, sess.opts, sess.spec, sess.ext, ws=dis_ws)
        info = self.dplan.fit()
        self.text_used = int(info["text_bytes"])
        max_text = int(self.dplan.span[1::2].max().item()) if self.n else 0
        tb = _native.DeviceBatch(self.dplan.text, self.dplan.span[0::2], self.dplan.span[1::2],
                                 (max_text + 3) // 4, 0)
        tb.n = self.n
        self.aplan = _native.AsmPlan(tb, sess.spec, sess.ext, out_cap=int(lengths[m0:m1].sum()) + 64 * self.n + 4096,
                                     stride=2, ws=asm_ws)
        ainfo = self.aplan.fit()
        self.out_used = int(ainfo["bytes"])
