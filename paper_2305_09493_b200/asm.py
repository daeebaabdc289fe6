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

import time
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

    ``run(data, offsets, lengths)`` takes a host batch (byte arena with module
    starts 16-byte aligned, int64 offsets / lengths; ``data`` may be a pinned
    torch uint8 tensor, otherwise it is copied into pinned staging first) and runs
    the round trip as a pipeline over ``chunks`` contiguous module ranges on three
    CUDA streams: the H2D copy of chunk k+1 and the D2H copies of chunk k-1's
    text and binaries overlap ``skg_disasm`` + ``skg_asm`` of chunk k (the
    assembler reads the disassembler's text arena directly, spans with stride 2).
    No sizing pass: the device arenas are capacity bounds (6x the chunk's input
    bytes for text, 1x + slack for binaries); after each chunk's kernels its
    counters are copied to pinned memory and the host, one chunk behind, issues
    D2H copies of exactly the bytes used (a chunk that overflows is re-run with
    grown arenas).  Returns (text uint8[], text spans int64[n, 2], disasm status
    int32[n], binaries uint8[], binary spans int64[n, 2], asm status int32[n])
    with spans relative to the returned arenas.  The arrays are views of the
    session's pinned host arenas (each chunk's D2H lands at its running offset,
    no host-side concatenation): they stay valid until the next call.
    ``stage()`` + ``run_staged()`` split the same call (pinned staging, then the
    pipeline).
    """

    TEXT_FACTOR = 6
    TAPER = (0.125, 0.25, 0.5, 0.75)   # relative sizes of the first / last chunks (short pipeline head / tail)

    def __init__(self, options=None, spec=None, ext=None, chunks=16):
        from .disasm import DisassemblerOptions, option_bits
        self.opts = option_bits(options if options is not None else DisassemblerOptions())
        self.spec, self.ext = spec, ext
        self.nchunks = max(1, int(chunks))
        self._buf = {}
        self._staged = None
        self._ratio = (4.0, 1.1)   # host arena sizes per input byte (grown from the runs seen)
        self.kernel_events = None  # a list: (start, disasm end, asm end) CUDA events per chunk launch

    def _get(self, name, n, dtype, pinned=False):
        """grow-only buffer (device, or pinned host)"""
        import torch
        b = self._buf.get(name)
        if b is None or b.numel() < n:
            n = max(int(n) * 9 // 8, 16)   # headroom: the next batch's chunks may be a little larger
            b = torch.empty(n, dtype=dtype).pin_memory() if pinned else \
                torch.empty(n, dtype=dtype, device="cuda")
            self._buf[name] = b
        return b

    def stage(self, data, offsets, lengths):
        """Pinned staging of the host inputs (what run() does first for non-pinned data)."""
        import numpy as np
        import torch
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        lengths = np.ascontiguousarray(lengths, dtype=np.int64)
        if isinstance(data, torch.Tensor) and data.is_pinned():
            h = data
        else:
            arr = np.frombuffer(memoryview(data).cast("B"), dtype=np.uint8) if not isinstance(data, np.ndarray) \
                else data.view(np.uint8).reshape(-1)
            h = self._get("h_data", arr.size + 16, torch.uint8, pinned=True)
            h.numpy()[: arr.size] = arr
        self._staged = (h, offsets, lengths)

    def run_staged(self, max_text=None):
        if self._staged is None:
            raise RuntimeError("stage() first")
        return self._pipeline(*self._staged)

    def run(self, data, offsets, lengths):
        self.stage(data, offsets, lengths)
        return self.run_staged()

    def _pipeline(self, h_data, offsets, lengths):
        import numpy as np
        import torch
        n = len(offsets)
        if self.kernel_events is not None:
            self.marks = [("start", time.perf_counter())]
        if n == 0:
            z8, z32 = np.zeros(0, np.uint8), np.zeros(0, np.int32)
            zs = np.zeros((0, 2), np.int64)
            return z8, zs, z32, z8.copy(), zs.copy(), z32.copy()
        nbytes = int(offsets[-1] + lengths[-1] + 15) // 16 * 16
        # contiguous module ranges by bytes; the first and last chunks are half size, so the
        # copy-in before the first kernel and the copy-out after the last one are short
        cum = np.cumsum(lengths)
        total = int(cum[-1])
        w = np.ones(self.nchunks)
        for j, t in enumerate(self.TAPER):          # short head and tail chunks
            if self.nchunks >= 2 * j + 3:
                w[j] = w[-1 - j] = t
        frac = np.cumsum(w) / w.sum()
        # integer targets: a float target would convert all of cum to float64 per search
        cuts = [0] + [int(np.searchsorted(cum, int(total * frac[k - 1]))) for k in range(1, self.nchunks)] + [n]
        cuts = sorted(set(cuts))
        chunks = [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
        if self.kernel_events is not None:
            self.marks.append(("chunks cut", time.perf_counter()))
        d_data = self._get("d_data", nbytes + 16, torch.uint8)
        # module offsets / lengths go up per chunk with the chunk's bytes (the host fills
        # chunk k's slice of the pinned staging while the GPU runs chunk k - 1)
        h_meta = self._get("h_meta", 2 * n, torch.int64, pinned=True)
        d_meta = self._get("d_meta", 2 * n, torch.int64)
        h_tspan = self._get("h_tspan", 2 * n, torch.int64, pinned=True)
        h_bspan = self._get("h_bspan", 2 * n, torch.int64, pinned=True)
        h_tst = self._get("h_tst", n, torch.int32, pinned=True)
        h_bst = self._get("h_bst", n, torch.int32, pinned=True)
        h_cnt = self._get("h_cnt", 16 * len(chunks), torch.int32, pinned=True)
        if self.kernel_events is not None:
            self.marks.append(("buffers", time.perf_counter()))
        comp = torch.cuda.current_stream()
        if "s_in" not in self._buf:
            self._buf["s_in"], self._buf["s_out"] = torch.cuda.Stream(), torch.cuda.Stream()
        s_in, s_out = self._buf["s_in"], self._buf["s_out"]
        cs = _native.ctypes.c_void_p(comp.cuda_stream)
        plans = []
        if self.kernel_events is not None:
            self.marks.append(("streams", time.perf_counter()))

        L = _native.lib()

        def store_counters(h, at, ws):
            # the chunk's allocator counters straight into pinned memory by a kernel: a
            # copy-engine D2H here would queue behind the previous chunk's text copy
            rc = L.skg_store_counters(_native.ctypes.c_void_p(h.data_ptr() + 4 * at),
                                      _native.ctypes.c_void_p(ws.data_ptr()), 8, cs)
            if rc:
                raise RuntimeError(f"skg_store_counters failed ({rc})")

        def launch(k, grow=None):
            a, b = chunks[k]
            b0 = int(offsets[a])
            b1 = int(offsets[b - 1] + lengths[b - 1] + 15) // 16 * 16
            cb = int(lengths[a:b].sum())
            mw = int(lengths[a:b].max()) // 4
            tcap, ocap = self.TEXT_FACTOR * cb + 4096, cb + 64 * (b - a) + 4096
            max_text = self.TEXT_FACTOR * mw * 4 + 4096      # per-module text bound: sizes the asm slots
            if grow:
                tcap, ocap = max(tcap, grow[0] + 16), max(ocap, grow[1] + 16)
                max_text = max(max_text, grow[2])
            batch = _native.DeviceBatch(d_data, d_meta[a:b], d_meta[n + a:n + b], mw, cb)
            # every device buffer is a grow-only pool of the session (per chunk slot): no
            # allocator traffic, which would synchronise the pipeline, once warmed up
            nb = b - a
            dbufs = {"text": self._get(f"text{k}", tcap, torch.uint8),
                     "span": self._get(f"dspan{k}", 2 * nb, torch.int64),
                     "status": self._get(f"dst{k}", nb, torch.int32),
                     "errs": self._get(f"derr{k}", 256 * max(16, min(nb, 1 << 16)), torch.uint8)}
            dp = _native.DisasmPlan(batch, self.opts, self.spec, self.ext, text_cap=tcap,
                                    ws=self._buf.get("ws_d"), bufs=dbufs)
            if dp.ws is not self._buf.get("ws_d"):
                self._buf["ws_d"] = dp.ws
            tb = _native.DeviceBatch(dp.text, dp.span[0::2], dp.span[1::2], 0, 0)
            tb.n = nb
            tb.max_words = (max_text + 3) // 4
            abufs = {"out": self._get(f"out{k}", ocap, torch.uint8),
                     "span": self._get(f"aspan{k}", 2 * nb, torch.int64),
                     "status": self._get(f"ast{k}", nb, torch.int32)}
            ap = _native.AsmPlan(tb, self.spec, self.ext, out_cap=ocap, stride=2, ws=self._buf.get("ws_a"),
                                 bufs=abufs)
            if ap.ws is not self._buf.get("ws_a"):
                self._buf["ws_a"] = ap.ws
            if grow is None:
                hm = h_meta.numpy()
                hm[a:b] = offsets[a:b]
                hm[n + a:n + b] = lengths[a:b]
                ev_in = torch.cuda.Event()
                with torch.cuda.stream(s_in):
                    d_meta[a:b].copy_(h_meta[a:b], non_blocking=True)
                    d_meta[n + a:n + b].copy_(h_meta[n + a:n + b], non_blocking=True)
                    d_data[b0:b1].copy_(h_data[b0:b1], non_blocking=True)
                    ev_in.record(s_in)
                comp.wait_event(ev_in)
            if self.kernel_events is not None:
                e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                e0.record(comp)
            dp.launch(cs)
            store_counters(h_cnt, 16 * k, dp.ws)
            if self.kernel_events is not None:
                e1.record(comp)
            ap.launch(cs)
            if self.kernel_events is not None:
                e2.record(comp)
                self.kernel_events.append((e0, e1, e2))
            store_counters(h_cnt, 16 * k + 8, ap.ws)
            ev = torch.cuda.Event()
            ev.record(comp)
            return dp, ap, ev

        def drain(k):
            dp, ap, ev = plans[k]
            ev.synchronize()
            c = h_cnt[16 * k: 16 * k + 16].numpy()
            tused = int(c[4]) & 0xFFFFFFFF | (int(c[5]) & 0xFFFFFFFF) << 32
            oused = int(c[12]) & 0xFFFFFFFF | (int(c[13]) & 0xFFFFFFFF) << 32
            if c[2] or c[10]:          # an arena overflowed: re-run this chunk with grown arenas
                plans[k] = launch(k, grow=(tused, oused, 0))
                return drain(k)
            a, b = chunks[k]
            # the results land in one host arena each, at running offsets (no host-side
            # concatenation: the returned arrays are views of the session's pinned arenas)
            ht = arena("h_text", pos[0], tused)
            ho = arena("h_out", pos[1], oused)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev)
                ht[pos[0]:pos[0] + tused].copy_(dp.text[:tused], non_blocking=True)
                h_tspan[2 * a:2 * b].copy_(dp.span[: 2 * (b - a)], non_blocking=True)
                h_tst[a:b].copy_(dp.status[: b - a], non_blocking=True)
                ho[pos[1]:pos[1] + oused].copy_(ap.out[:oused], non_blocking=True)
                h_bspan[2 * a:2 * b].copy_(ap.span[: 2 * (b - a)], non_blocking=True)
                h_bst[a:b].copy_(ap.status[: b - a], non_blocking=True)
            ev_copy = torch.cuda.Event()
            ev_copy.record(s_out)
            parts[k] = (pos[0], tused, pos[1], oused, ev_copy)
            rebased.discard(k)
            pos[0] += tused
            pos[1] += oused

        def rebase(k):
            """chunk k's spans -> offsets in the whole arenas (once its copies are done)"""
            a, b = chunks[k]
            tp, _, op, _, ev_copy = parts[k]
            ev_copy.synchronize()
            h_tspan[2 * a:2 * b:2].numpy()[:] += tp
            h_bspan[2 * a:2 * b:2].numpy()[:] += op
            if (h_bst[a:b].numpy() == _native.ST_INTERNAL).any():
                internal.add(k)
            rebased.add(k)

        def arena(name, used, need):
            """grow-only pinned host arena; growing keeps the bytes already copied"""
            h = self._buf.get(name)
            if h is None or h.numel() < used + need:
                s_out.synchronize()
                est = int(hint.get(name, 0) * 1.05) + 4096
                nh = torch.empty(max(est, 2 * (used + need)) if h is not None else max(est, used + need),
                                 dtype=torch.uint8).pin_memory()
                if h is not None and used:
                    nh[:used].copy_(h[:used])
                self._buf[name] = h = nh
            return h

        total_in = int(lengths.sum())
        hint = {"h_text": total_in * self._ratio[0], "h_out": total_in * self._ratio[1]}
        pos, parts, rebased, internal = [0, 0], {}, set(), set()
        for k in range(len(chunks)):
            plans.append(launch(k))
            if k == 0 and self.kernel_events is not None:
                self.marks.append(("chunk 0 queued", time.perf_counter()))
            if k >= 1:
                drain(k - 1)          # host one chunk behind: chunk k's kernels are queued
            if k >= 2:
                rebase(k - 2)         # its copies were queued a chunk ago: overlaps chunk k
        drain(len(chunks) - 1)
        if self.kernel_events is not None:
            self.marks.append(("last drain queued", time.perf_counter()))
        s_out.synchronize()
        if self.kernel_events is not None:
            self.marks.append(("copies done", time.perf_counter()))
        for k in range(len(chunks)):
            if k not in rebased:
                rebase(k)
        # a module whose text outgrew the per-module bound the assembler slots were sized
        # for reports an internal status: re-run its chunk with slots for the real maximum
        # (its results are appended to the arenas and its spans rebased again)
        for k in sorted(internal):
            a, b = chunks[k]
            mx = int(h_tspan[2 * a + 1:2 * b:2].numpy().max())
            _, tused, _, oused, _ = parts[k]
            plans[k] = launch(k, grow=(tused, max(oused, 4 * mx), mx))
            drain(k)
            s_out.synchronize()
            rebase(k)
        tspan = h_tspan[: 2 * n].numpy().reshape(n, 2)
        bspan = h_bspan[: 2 * n].numpy().reshape(n, 2)
        if total_in:
            self._ratio = (max(self._ratio[0], pos[0] / total_in), max(self._ratio[1], pos[1] / total_in))
        if self.kernel_events is not None:
            self.marks.append(("spans rebased", time.perf_counter()))
        text = self._buf["h_text"].numpy()[: pos[0]]
        binv = self._buf["h_out"].numpy()[: pos[1]]
        return text, tspan, h_tst[:n].numpy(), binv, bspan, h_bst[:n].numpy()
