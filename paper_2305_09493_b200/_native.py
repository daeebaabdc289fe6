"""ctypes binding of libskgpu.so (include/skgpu.h) + device buffer plumbing.

PyTorch is used only to own device memory and streams.  There is no CPU
fallback: if the library or a CUDA device is missing, every codec entry point
raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
import struct
from pathlib import Path

import numpy as np

from . import errors as _err

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("SKGPU_LIB", _HERE / "libskgpu.so"))

ST_OK, ST_TRUNCATED, ST_NOTSPIRV, ST_CORRUPT, ST_CODEC = 0, 1, 2, 3, 4
ST_UNICODE, ST_KEY, ST_VALUE, ST_INTERNAL = 5, 6, 7, 99

OPT_HIGHLIGHT, OPT_INLINE, OPT_NO_INDENT, OPT_GROUP, OPT_NO_HEADER, OPT_STRICT = 1, 2, 4, 8, 16, 32

ERR_DTYPE = np.dtype([("module", "<i4"), ("status", "<i4"), ("a", "<u4"), ("b", "<u4"),
                      ("c", "<u4"), ("d", "<u4"), ("len", "<i4"), ("msg", "S228")])
assert ERR_DTYPE.itemsize == 256

_UTF8_REASON = {1: "invalid start byte", 2: "invalid continuation byte", 3: "unexpected end of data"}


class NativeUnavailable(RuntimeError):
    """libskgpu.so could not be loaded or no CUDA device is present."""


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.is_file():
        raise NativeUnavailable(f"{LIB_PATH} is missing: run __graft_entry__.build()")
    L = ctypes.CDLL(str(LIB_PATH))
    P, U32, U64, I32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32
    L.skg_tables_create.argtypes = [P, U64, ctypes.POINTER(P)]
    L.skg_tables_destroy.argtypes = [P]
    L.skg_workspace_bytes.argtypes = [U32, U32]
    L.skg_workspace_bytes.restype = U64
    L.skg_disasm.argtypes = [P, P, P, P, U32, U32, U32, P, U64, P, P, P, U32, P, U64, P]
    L.skg_validate.argtypes = [P, P, P, P, U32, U32, P, U64, P, P, P, U32, P, U64, P]
    L.skg_decode.argtypes = [P, P, P, U32, P, P, P, P, P, P, P, P, U32, P, U64, P]
    L.skg_last_counts.argtypes = [P, ctypes.POINTER(U32), ctypes.POINTER(U32), ctypes.POINTER(U64), P]
    L.skg_decode_large_workspace_bytes.argtypes = [U64]
    L.skg_decode_large_workspace_bytes.restype = U64
    L.skg_decode_large.argtypes = [P, U64, U32, P, P, P, P, P, P, P, U64, P]
    L.skg_large_workspace_bytes.argtypes = [U64, U32]
    L.skg_large_workspace_bytes.restype = U64
    L.skg_validate_large.argtypes = [P, P, U64, P, U64, ctypes.POINTER(U64), P, P, P, U64, P, U32]
    L.skg_validate_large.restype = I32
    L.skg_disasm_large.argtypes = [P, P, U64, U32, P, U64, ctypes.POINTER(U64), P, P, P, U64, P, U32]
    L.skg_disasm_large.restype = I32
    L.skg_disasm_refs.argtypes = [P, P, P, P, U32, U32, U32, P, U64, P, P, P, U32, P, U64, P, P, P, U32]
    L.skg_disasm_refs.restype = I32
    L.skg_disasm_validate.argtypes = [P, P, P, P, U32, U32, U32, P, U64, P, P, P, U32, P, U64, P, P, P, U32,
                                      P, U64, P]
    L.skg_disasm_validate.restype = I32
    L.skg_selftest_repr_f32.argtypes = [P, U64, U64, P, P, P]
    L.skg_selftest_repr_f32.restype = I32
    L.skg_tokenize.argtypes = [P, P, P, U32, P, P, P, P, P, P, P, P, P]
    L.skg_encode_modules.argtypes = [P, U32, P, P, U64, P, P, U64, P, P, P]
    L.skg_pack_strings.argtypes = [P, P, P, P, U32, U64, P, P, P]
    L.skg_ctx_literals.argtypes = [P, P, P, U32, P, P, P, P]
    for f in (L.skg_tokenize, L.skg_encode_modules, L.skg_pack_strings, L.skg_ctx_literals):
        f.restype = I32
    L.skg_store_counters.argtypes = [P, P, U32, P]
    L.skg_store_counters.restype = I32
    L.skg_copy_to_host.argtypes = [P, P, U64, U32, P]
    L.skg_copy_to_host.restype = I32
    L.skg_version.restype = ctypes.c_char_p
    for f in (L.skg_tables_create, L.skg_disasm, L.skg_validate, L.skg_decode, L.skg_last_counts,
              L.skg_decode_large):
        f.restype = I32
    _lib = L
    return L


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the codec path runs on the GPU only")
    return torch


def _check(rc, what):
    if rc == -4:
        raise RuntimeError(f"libskgpu {what}: the output exceeds 4 GiB (32-bit text offsets)")
    if rc != 0:
        raise RuntimeError(f"libskgpu {what} failed with code {rc}")


def _device():
    """index of the current CUDA device: table handles and workspaces are per device"""
    return _torch().cuda.current_device()


# -- grammar tables --------------------------------------------------------------
_tables = {}


def tables_handle(spec, ext):
    """Device table handle for (spec, ext); packed + uploaded once per pair."""
    from . import grammar, tables
    spec = spec if spec is not None else grammar.load_pinned()
    ext = ext if ext is not None else grammar.load_pinned_extended()
    key = (id(spec), id(ext), _device())
    hit = _tables.get(key)
    if hit is not None and hit[1] is spec and hit[2] is ext:
        return hit[0]
    _torch()
    packed = tables.pack(spec, ext)
    blob = np.ascontiguousarray(packed.blob, dtype=np.uint32)
    handle = ctypes.c_void_p()
    _check(lib().skg_tables_create(blob.ctypes.data, blob.size, ctypes.byref(handle)), "tables_create")
    _tables[key] = (handle, spec, ext)
    return handle


# -- device batches ----------------------------------------------------------------
class DeviceBatch:
    """Modules resident in device memory: byte arena + int64 offsets/lengths."""

    def __init__(self, data, off, length, max_words, total_bytes):
        self.data, self.off, self.len = data, off, length
        self.n = int(off.numel())
        self.max_words = int(max_words)
        self.total_bytes = int(total_bytes)

    @classmethod
    def from_host(cls, data: np.ndarray, offsets: np.ndarray, lengths: np.ndarray, stream=None):
        torch = _torch()
        dev = torch.device("cuda")
        arr = np.ascontiguousarray(data, dtype=np.uint8)
        if not arr.flags.writeable:   # torch.from_numpy wants a writable array (read-only bytes views)
            arr = arr.copy()
        d = torch.from_numpy(arr).to(dev, non_blocking=False)
        o = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int64)).to(dev)
        ln = torch.from_numpy(np.ascontiguousarray(lengths, dtype=np.int64)).to(dev)
        mw = int(lengths.max()) // 4 if len(lengths) else 0
        return cls(d, o, ln, mw, int(lengths.sum()))

    @classmethod
    def from_modules(cls, modules):
        lengths = np.array([len(m) for m in modules], dtype=np.int64)
        padded = (lengths + 15) // 16 * 16
        offsets = np.zeros(len(modules), dtype=np.int64)
        if len(modules) > 1:
            offsets[1:] = np.cumsum(padded)[:-1]
        buf = bytearray(int(padded.sum()) + 16)
        for m, o in zip(modules, offsets):
            buf[o:o + len(m)] = m
        return cls.from_host(np.frombuffer(bytes(buf), dtype=np.uint8), offsets, lengths)


class _Workspace:
    """One grow-only device scratch buffer per CUDA device."""

    def __init__(self):
        self.bufs = {}

    def get(self, nbytes):
        torch = _torch()
        dev = _device()
        buf = self.bufs.get(dev)
        if buf is None or buf.numel() < nbytes:
            buf = self.bufs[dev] = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device="cuda")
        return buf


_ws = _Workspace()
_large_text = _Workspace()   # the large-module calls' text arena (grow-only, per device)
_large_vtext = _Workspace()  # the validation's, when it runs while a disassembly is copied out


class _PinnedStage:
    """Pinned host staging for large device -> host results (a pageable .cpu() copy of a
    ~1 GB text runs at a fraction of the link rate); grown on demand, reused."""

    def __init__(self):
        self.buf = None

    def to_bytes(self, dev_u8, view: bool = False):
        """bytes of a device uint8 tensor; view=True: a numpy view of the pinned staging
        buffer instead (no host-side copy into a new bytes object; valid until the next
        staged copy)"""
        torch = _torch()
        n = int(dev_u8.numel())
        if n < (16 << 20) or dev_u8.dtype != torch.uint8 or not dev_u8.is_contiguous():
            # small results: the plain copy is cheaper than pinning
            out = dev_u8.cpu().numpy()
            return out if view else out.tobytes()
        if self.buf is None or self.buf.numel() < n:
            self.buf = torch.empty(n + (n >> 3), dtype=torch.uint8).pin_memory()
        self.buf[:n].copy_(dev_u8, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self.buf[:n].numpy() if view else self.buf[:n].numpy().tobytes()

    def to_u32(self, dev_i32, count: int):
        """the first `count` elements of a device int32 tensor as a host uint32 array"""
        torch = _torch()
        n = 4 * count
        if n < (16 << 20):
            return dev_i32[:count].cpu().numpy().view(np.uint32)
        if self.buf is None or self.buf.numel() < n:
            self.buf = torch.empty(n + (n >> 3), dtype=torch.uint8).pin_memory()
        self.buf[:n].copy_(dev_i32[:count].view(torch.uint8), non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self.buf[:n].numpy().view(np.uint32).copy()


_pinned = _PinnedStage()
_pinned_v = _PinnedStage()   # a validation's results while _pinned receives a disassembly


def release_host_staging():
    """Free the pinned host staging buffers (they grow to the largest result fetched)."""
    _pinned.buf = None
    _pinned_v.buf = None


def _stream():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class TextResult:
    """Device-resident output of a batch call: module m's text is
    text[span[2m] : span[2m] + span[2m+1]]."""

    def __init__(self, text, span, status, errors):
        self.text, self.span, self.status, self.errors = text, span, status, errors


def last_counts(ws):
    nerr, over, used = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint64()
    _check(lib().skg_last_counts(ws.data_ptr(), ctypes.byref(nerr), ctypes.byref(over),
                                 ctypes.byref(used), _stream()), "counts")
    return int(nerr.value), bool(over.value), int(used.value)


def _run_text_kernel(kind, batch: DeviceBatch, opts, spec, ext, text_cap=None, err_cap=None, refs=None):
    torch = _torch()
    L = lib()
    th = tables_handle(spec, ext)
    n = batch.n
    ws_bytes = int(L.skg_workspace_bytes(n, max(batch.max_words, 1)))
    ws = _ws.get(ws_bytes)
    cap = text_cap if text_cap is not None else 6 * batch.total_bytes + 4096
    ecap = err_cap if err_cap is not None else max(16, min(n, 1 << 16))
    for _ in range(3):
        text = torch.empty(max(cap, 16), dtype=torch.uint8, device="cuda")
        span = torch.empty(2 * max(n, 1), dtype=torch.int64, device="cuda")
        status = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        errs = torch.empty(ecap * 256, dtype=torch.uint8, device="cuda")
        if kind == "disasm" and refs is not None:   # (ids u32[n, 3] device, text u8 device, n)
            rc = L.skg_disasm_refs(th, batch.data.data_ptr(), batch.off.data_ptr(), batch.len.data_ptr(), n,
                                   opts, batch.max_words, text.data_ptr(), cap, span.data_ptr(),
                                   status.data_ptr(), errs.data_ptr(), ecap, ws.data_ptr(), ws_bytes, _stream(),
                                   refs[0].data_ptr(), refs[1].data_ptr(), refs[2])
        elif kind == "disasm":
            rc = L.skg_disasm(th, batch.data.data_ptr(), batch.off.data_ptr(), batch.len.data_ptr(), n,
                              opts, batch.max_words, text.data_ptr(), cap, span.data_ptr(),
                              status.data_ptr(), errs.data_ptr(), ecap, ws.data_ptr(), ws_bytes, _stream())
        else:
            rc = L.skg_validate(th, batch.data.data_ptr(), batch.off.data_ptr(), batch.len.data_ptr(), n,
                                batch.max_words, text.data_ptr(), cap, span.data_ptr(),
                                status.data_ptr(), errs.data_ptr(), ecap, ws.data_ptr(), ws_bytes,
                                _stream())
        _check(rc, kind)
        nerr, over, used = last_counts(ws)
        if over or nerr > ecap:
            cap = max(cap, used + 16)
            ecap = max(ecap, nerr)
            continue
        return TextResult(text[:used], span[: 2 * n], status[:n], errs[: nerr * 256])
    raise RuntimeError(f"libskgpu {kind}: output capacity retry failed")


VAL_COUNTERS = 128   # byte offset of the fused validator's counters in the workspace


def run_pipeline(batch: DeviceBatch, opts, spec=None, ext=None):
    """skg_disasm_validate: one pass -> (disasm TextResult, validate TextResult)."""
    torch = _torch()
    L = lib()
    th = tables_handle(spec, ext)
    n = batch.n
    ws_bytes = int(L.skg_workspace_bytes(n, max(batch.max_words, 1)))
    ws = _ws.get(ws_bytes)
    cap, vcap = 6 * batch.total_bytes + 4096, batch.total_bytes + 4096
    ecap = max(16, min(n, 1 << 16))
    for _ in range(3):
        text = torch.empty(max(cap, 16), dtype=torch.uint8, device="cuda")
        vtext = torch.empty(max(vcap, 16), dtype=torch.uint8, device="cuda")
        span = torch.empty(2 * max(n, 1), dtype=torch.int64, device="cuda")
        vspan = torch.empty(2 * max(n, 1), dtype=torch.int64, device="cuda")
        status = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        vstatus = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        errs = torch.empty(ecap * 256, dtype=torch.uint8, device="cuda")
        verrs = torch.empty(ecap * 256, dtype=torch.uint8, device="cuda")
        _check(L.skg_disasm_validate(th, batch.data.data_ptr(), batch.off.data_ptr(), batch.len.data_ptr(), n, opts,
                                     batch.max_words, text.data_ptr(), cap, span.data_ptr(), status.data_ptr(),
                                     errs.data_ptr(), ecap, vtext.data_ptr(), vcap, vspan.data_ptr(),
                                     vstatus.data_ptr(), verrs.data_ptr(), ecap, ws.data_ptr(), ws_bytes,
                                     _stream()), "disasm_validate")
        nerr, over, used = last_counts(ws)
        vnerr, vover, vused = last_counts(ws[VAL_COUNTERS:])
        if over or vover or nerr > ecap or vnerr > ecap:
            cap, vcap = max(cap, used + 16), max(vcap, vused + 16)
            ecap = max(ecap, nerr, vnerr)
            continue
        return (TextResult(text[:used], span[: 2 * n], status[:n], errs[: nerr * 256]),
                TextResult(vtext[:vused], vspan[: 2 * n], vstatus[:n], verrs[: vnerr * 256]))
    raise RuntimeError("libskgpu disasm_validate: output capacity retry failed")


def run_texts_pipeline(batch: DeviceBatch, opts=0, spec=None, ext=None):
    """Fused disassembly + validation of a device batch -> (texts, diagnostics texts), each
    a list of (bytes | exception).  Batches with large modules (grid-wide kernels) or
    beyond the one-launch workspace budget take the two separate batch paths."""
    n = batch.n
    if n == 0:
        return [], []
    need = int(lib().skg_workspace_bytes(n, max(batch.max_words, 1)))
    if n == 1 and batch.max_words >= large_threshold(1):   # one large module: grid-wide, copy overlapped
        t, v = _disasm_validate_large(batch, 0, int(batch.len[0].item()), opts, spec, ext)
        if t is None:
            t = run_texts("disasm", batch, opts, spec, ext)[0]
        if v is None:
            v = run_texts("validate", batch, 0, spec)[0]
        return [t], [v]
    if batch.max_words >= large_threshold(n) or (n > 1 and need > WS_BUDGET):
        return run_texts("disasm", batch, opts, spec, ext), run_texts("validate", batch, 0, spec)
    d, v = run_pipeline(batch, opts, spec, ext)
    return fetch_texts(d, n), fetch_texts(v, n)


def run_disasm(batch, opts, spec=None, ext=None, **kw):
    return _run_text_kernel("disasm", batch, opts, spec, ext, **kw)


def run_validate(batch, spec=None, **kw):
    return _run_text_kernel("validate", batch, 0, spec, None, **kw)


def decode_errors(err_bytes: np.ndarray):
    """module index -> exception instance, from the device error records."""
    recs = np.frombuffer(err_bytes.tobytes(), dtype=ERR_DTYPE)
    out = {}
    for r in recs:
        msg = bytes(r["msg"])[: max(0, min(int(r["len"]), 227))].decode("utf-8", "replace")
        out[int(r["module"])] = make_exception(int(r["status"]), msg, int(r["a"]), int(r["b"]),
                                               int(r["c"]), int(r["d"]))
    return out


def make_exception(status, msg, a=0, b=0, c=0, d=0):
    if status == ST_TRUNCATED:
        return _err.TruncatedStreamError(msg)
    if status == ST_NOTSPIRV:
        return _err.NotSpirvError(msg)
    if status == ST_CORRUPT:
        return _err.CorruptStreamError(msg)
    if status == ST_CODEC:
        return _err.CodecError(msg)
    if status == ST_UNICODE:
        obj = bytes(a) + bytes([d]) + bytes(max(0, b - a - 1))
        return UnicodeDecodeError("utf-8", obj, a, b, _UTF8_REASON.get(c, "invalid start byte"))
    if status == ST_KEY:
        return KeyError(int(msg))
    if status == ST_VALUE:
        return ValueError(msg)
    return RuntimeError(f"libskgpu internal error: {msg}")


# Workspace budget of one launch: the per-warp scratch slot is sized for the
# largest module, so a batch mixing a few very large modules with many small
# ones runs the large ones in launches of their own (one warp each).
WS_BUDGET = 8 << 30


def run_texts(kind, batch: DeviceBatch, opts=0, spec=None, ext=None, refs=None):
    """disasm / validate of a device batch -> list of (text bytes | exception).
    refs: explicit id refs for skg_disasm_refs (format_instruction with a context)."""
    torch = _torch()
    n = batch.n
    if n == 0:
        return []
    run = (lambda b: run_disasm(b, opts, spec, ext, refs=refs)) if kind == "disasm" else \
        (lambda b: run_validate(b, spec))
    need = int(lib().skg_workspace_bytes(n, max(batch.max_words, 1)))
    big = large_threshold(n) if refs is None else 1 << 62   # explicit refs: the batch kernel only
    if (n == 1 or need <= WS_BUDGET) and batch.max_words < big:
        return fetch_texts(run(batch), n)
    lens = batch.len.cpu().numpy()
    words = lens // 4
    if batch.max_words >= big:   # single large modules: the whole GPU on one module
        out = [None] * n
        rest = []
        for i in range(n):
            r = None
            if words[i] >= big:
                r = _validate_large(batch, i, int(lens[i]), spec) if kind == "validate" else \
                    _disasm_large(batch, i, int(lens[i]), opts, spec, ext)
            if r is None:
                rest.append(i)
            else:
                out[i] = r
        if not rest:
            return out
        if len(rest) < n:
            idx = np.array(rest)
            ti = torch.from_numpy(idx.astype(np.int64)).to(batch.off.device)
            sub = DeviceBatch(batch.data, batch.off[ti], batch.len[ti], int(words[idx].max()), int(lens[idx].sum()))
            for k, r in zip(rest, run_texts(kind, sub, opts, spec, ext)):
                out[k] = r
            return out
    per_word = max(need // max(int(batch.max_words), 1), 1)        # workspace bytes per max-word
    w_small = max(int(WS_BUDGET // per_word), 1)
    out = [None] * n
    small = np.nonzero(words <= w_small)[0]
    groups = [small] if len(small) else []
    groups += [np.array([i]) for i in np.nonzero(words > w_small)[0]]
    for idx in groups:
        ti = torch.from_numpy(idx.astype(np.int64)).to(batch.off.device)
        sub = DeviceBatch(batch.data, batch.off[ti], batch.len[ti], int(words[idx].max()), int(lens[idx].sum()))
        for k, r in zip(idx, fetch_texts(run(sub), len(idx))):
            out[int(k)] = r
    return out


LARGE_MODULE_WORDS = 1 << 20   # modules this size and up in a batch run grid-wide (skg_*_large)
# A single-module call (n == 1) runs grid-wide from this size: one warp takes ~0.27 ms
# (disasm) / ~0.09 ms (validate) per 1000 words, the grid-wide path ~1 ms + ~0.01 ms per
# 1000 words (tools/large_threshold_probe.py on a B200: 13.6k words 3.8 vs 1.2 ms,
# 850k words 291 vs 3.3 ms; 1.8k words 0.64 vs 0.98 ms).  In a batch the other modules
# run beside the one warp, so only LARGE_MODULE_WORDS sends a module there.
SINGLE_LARGE_WORDS = 4096


def large_threshold(n: int) -> int:
    return min(SINGLE_LARGE_WORDS, LARGE_MODULE_WORDS) if n == 1 else LARGE_MODULE_WORDS
_DECODE_CODES = {ST_NOTSPIRV: "NotSpirv", ST_TRUNCATED: "TruncatedStream", ST_CORRUPT: "CorruptStream"}


def _header_bound(head: bytes) -> int:
    """the header bound as skg_*_large read it: byte-swapped only when the magic is"""
    if len(head) < 20:
        return 0
    w = np.frombuffer(head[:20], dtype="<u4")
    return int(np.frombuffer(head[:20], dtype=">u4")[3]) if w[0] == 0x03022307 else int(w[3])


def _large_call(fn, batch: DeviceBatch, i: int, nbytes: int, *args, cap=None, view=False, pool=None,
                fetch=True, stage=None):
    """Shared driver of skg_validate_large / skg_disasm_large -> (rc, text bytes, errs);
    view=True: the text as a numpy view of the pinned staging buffer (see _PinnedStage);
    pool: the device text arena (default _large_text); fetch=False: the text stays a
    device tensor (a slice of the arena)."""
    torch = _torch()
    L = lib()
    o = int(batch.off[i].item())
    data = batch.data.data_ptr() + o
    W = nbytes // 4
    bound = _header_bound(batch.data[o:o + 20].cpu().numpy().tobytes())
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    errs = torch.zeros(256, dtype=torch.uint8, device="cuda")
    cap = cap if cap is not None else max(1 << 20, 4 * nbytes)
    # id tables sized by the header bound first; ids at/above it (rc 2): once more with
    # tables for every id below 2W + 64 (the header bound still names BoundTooSmall)
    for min_table in (0, 2 * W + 64):
        if min_table and bound >= min_table:
            break
        ws_bytes = int(L.skg_large_workspace_bytes(W, min(max(bound, min_table), 2 * W + 64)))
        ws = _ws.get(ws_bytes)
        for _ in range(3):
            text = (pool or _large_text).get(cap)   # grow-only (a fresh ~GB allocation per call stalls)
            need = ctypes.c_uint64(0)
            rc = fn(data, nbytes, *args, text.data_ptr(), cap, ctypes.byref(need), status.data_ptr(),
                    errs.data_ptr(), ws.data_ptr(), ws_bytes, _stream(), min_table)
            if rc == 3:
                cap = int(need.value) + 16
                continue
            break
        if rc != 2:
            break
    _check(rc if rc < 0 else 0, getattr(fn, "__name__", "large call"))
    if rc != 0:
        return rc, None, errs
    return rc, ((stage or _pinned).to_bytes(text[: int(need.value)], view) if fetch else text[: int(need.value)]), errs


def _disasm_large(batch: DeviceBatch, i: int, nbytes: int, opts: int, spec, ext, view=False):
    """skg_disasm_large on module i -> text bytes | exception | None (= use the batch path);
    view=True: the text as a numpy view of the pinned staging buffer."""
    L = lib()
    th = tables_handle(spec, ext)

    def disasm_large(*a):
        return L.skg_disasm_large(th, a[0], a[1], *a[2:])
    rc, text, errs = _large_call(disasm_large, batch, i, nbytes, opts, view=view)
    if rc == 2:
        return None
    if rc == 0:
        return text
    return decode_errors(errs.cpu().numpy())[0]


def _disasm_validate_large(batch: DeviceBatch, i: int, nbytes: int, opts: int, spec, ext, view=False):
    """Module i through skg_disasm_large then skg_validate_large, the disassembly's text
    copied to the host on a side stream while the validation kernels run ->
    (text | exception | None, diagnostics text | exception | None); None = use the batch
    path.  view=True: the text as a numpy view of the pinned staging buffer."""
    torch = _torch()
    L = lib()
    th = tables_handle(spec, ext)

    def disasm_large(*a):
        return L.skg_disasm_large(th, a[0], a[1], *a[2:])
    rc, dtext, errs = _large_call(disasm_large, batch, i, nbytes, opts, fetch=False)
    if rc == 2:
        return None, _validate_large(batch, i, nbytes, spec)
    if rc != 0:
        return decode_errors(errs.cpu().numpy())[0], _validate_large(batch, i, nbytes, spec)
    n = int(dtext.numel())
    if n < (16 << 20):       # small text: the plain copy
        return _pinned.to_bytes(dtext, view), _validate_large(batch, i, nbytes, spec, pool=_large_vtext)
    stage = _pinned
    if stage.buf is None or stage.buf.numel() < n:
        stage.buf = torch.empty(n + (n >> 3), dtype=torch.uint8).pin_memory()
    side = _side_stream()
    ready = torch.cuda.Event()
    ready.record(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        side.wait_event(ready)
        # SM stores into the mapped pinned buffer: a copy-engine D2H would hold up the
        # validation's own small device->host reads queued behind it (config 3: 51.8 ms
        # per step with the copy engine; 8 CTAs 40.7 ms, 4: 49, 16: 44.8, 64: 51.2 -- more
        # CTAs take SMs from the validation kernels)
        _check(L.skg_copy_to_host(ctypes.c_void_p(stage.buf.data_ptr()), ctypes.c_void_p(dtext.data_ptr()), n,
                                  int(os.environ.get("SKG_D2H_CTAS", "8")), ctypes.c_void_p(side.cuda_stream)),
               "copy_to_host")
        copied = torch.cuda.Event()
        copied.record(side)
    # the validation writes its own arena (_large_vtext) and host staging (small: .cpu())
    diags = _validate_large(batch, i, nbytes, spec, pool=_large_vtext, stage=_pinned_v)
    copied.synchronize()
    torch.cuda.current_stream().wait_event(copied)   # the arena is reused by the next call
    host = stage.buf[:n].numpy()
    return (host if view else host.tobytes()), diags


_side_streams = {}


def _side_stream():
    """one side stream per device (result copies that overlap kernels)"""
    torch = _torch()
    dev = _device()
    st = _side_streams.get(dev)
    if st is None:
        st = _side_streams[dev] = torch.cuda.Stream()
    return st


def _validate_large(batch: DeviceBatch, i: int, nbytes: int, spec, pool=None, stage=None):
    """skg_validate_large on module i of a device batch -> text bytes | exception | None (= not handled)."""
    L = lib()
    th = tables_handle(spec, None)

    def validate_large(*a):
        return L.skg_validate_large(th, *a)
    rc, text, errs = _large_call(validate_large, batch, i, nbytes, cap=1 << 20, pool=pool, stage=stage)
    if rc == 2:
        return None
    if rc == 0:
        return text
    exc = decode_errors(errs.cpu().numpy())[0]
    if rc == 1:
        return exc
    code = _DECODE_CODES.get(rc - 10, "CorruptStream")   # the decode error is the only diagnostic
    return f"error {code} module {exc}\n".encode()


def fetch_texts(res: TextResult, n: int):
    """Host copies: list of (text bytes | exception) per module."""
    span = res.span.cpu().numpy()
    status = res.status.cpu().numpy()
    text = _pinned.to_bytes(res.text)
    errs = decode_errors(res.errors.cpu().numpy()) if res.errors.numel() else {}
    out = []
    for m in range(n):
        if status[m] != ST_OK:
            out.append(errs.get(m) or make_exception(int(status[m]), "error record dropped"))
        else:
            o = int(span[2 * m])
            out.append(text[o:o + int(span[2 * m + 1])])
    return out


LARGE_DECODE_WORDS = 1 << 16   # modules this size and up take the tiled boundary pass


def run_decode(data: bytes):
    """Single-module boundary pass -> (header tuple, words array, [(start, wc)]) or raises."""
    torch = _torch()
    L = lib()
    n = len(data)
    W = n // 4
    dev = torch.device("cuda")
    pad = bytes(data) + b"\x00" * (-n % 16 + 16)
    d = torch.frombuffer(bytearray(pad), dtype=torch.uint8).to(dev)
    if W >= LARGE_DECODE_WORDS:
        return _run_decode_large(d, n)
    meta = torch.tensor([0, n, 0], dtype=torch.int64, device=dev)   # off, len, base
    header = torch.zeros(5, dtype=torch.int32, device=dev)
    inst_off = torch.zeros(max(W, 1), dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    words = torch.zeros(max(W, 1), dtype=torch.int32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    errs = torch.zeros(256, dtype=torch.uint8, device=dev)
    ws = _ws.get(1 << 20)
    p = meta.data_ptr()
    _check(L.skg_decode(d.data_ptr(), p, p + 8, 1, header.data_ptr(), inst_off.data_ptr(), p + 16,
                        cnt.data_ptr(), words.data_ptr(), p + 16, status.data_ptr(), errs.data_ptr(), 1,
                        ws.data_ptr(), 1 << 20, _stream()), "decode")
    st = int(status.item())
    if st != ST_OK:
        raise decode_errors(errs.cpu().numpy())[0]
    h = header.cpu().numpy().view(np.uint32)
    k = int(cnt.item())
    return tuple(int(x) for x in h), words.cpu().numpy().view(np.uint32)[:W], \
        inst_off.cpu().numpy().view(np.uint32)[:k]


def _run_decode_large(d, n: int):
    """skg_decode_large: one large module already on the device (tiled boundary pass)."""
    torch = _torch()
    L = lib()
    W = n // 4
    dev = d.device
    header = torch.zeros(5, dtype=torch.int32, device=dev)
    inst_off = torch.zeros(max(W, 1), dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    words = torch.zeros(max(W, 1), dtype=torch.int32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    errs = torch.zeros(256, dtype=torch.uint8, device=dev)
    ws_bytes = int(L.skg_decode_large_workspace_bytes(W))
    ws = _ws.get(ws_bytes)
    from . import grammar as _grammar
    max_op = max((i.opcode for i in _grammar.load_pinned().instructions), default=0)
    _check(L.skg_decode_large(d.data_ptr(), n, max_op, header.data_ptr(), inst_off.data_ptr(), cnt.data_ptr(),
                              words.data_ptr(), status.data_ptr(), errs.data_ptr(), ws.data_ptr(), ws_bytes,
                              _stream()), "decode_large")
    if int(status.item()) != ST_OK:
        raise decode_errors(errs.cpu().numpy())[0]
    k = int(cnt.item())
    return tuple(int(x) for x in header.cpu().numpy().view(np.uint32)), \
        _pinned.to_u32(words, W), _pinned.to_u32(inst_off, k)


# -- standalone codec / tokenizer kernels (skg_codec.cuh) -------------------------------
def _dev(arr, dtype):
    """host numpy array -> device tensor (at least one element)"""
    torch = _torch()
    a = np.ascontiguousarray(arr, dtype=dtype)
    if a.size == 0:
        a = np.zeros(1, dtype=dtype)
    elif not a.flags.writeable:
        a = a.copy()
    return torch.from_numpy(a).to("cuda")


def run_tokenize(raws):
    """list[bytes] (one logical line each) -> per line (kind, [(text bytes, column, is_string)],
    err_col): kind 0 blank, 1 instruction, 2 with result, 3 unterminated string."""
    torch = _torch()
    n = len(raws)
    if n == 0:
        return []
    lens = np.array([len(r) for r in raws], dtype=np.int64)
    offs = np.zeros(n, dtype=np.int64)
    offs[1:] = np.cumsum(lens)[:-1]
    total = int(lens.sum())
    text = _dev(np.frombuffer(b"".join(raws) + b"\0", dtype=np.uint8), np.uint8)
    d_off, d_len = _dev(offs, np.int64), _dev(lens, np.int64)
    cap = max(total, 1)
    tok_off = torch.zeros(cap, dtype=torch.int64, device="cuda")
    tok_len = torch.zeros(cap, dtype=torch.int32, device="cuda")
    tok_col = torch.zeros(cap, dtype=torch.int32, device="cuda")
    tok_fl = torch.zeros(cap, dtype=torch.uint8, device="cuda")
    esc = torch.zeros(cap + 1, dtype=torch.uint8, device="cuda")
    kind = torch.zeros(n, dtype=torch.int32, device="cuda")
    ntok = torch.zeros(n, dtype=torch.int32, device="cuda")
    err = torch.zeros(n, dtype=torch.int32, device="cuda")
    _check(lib().skg_tokenize(text.data_ptr(), d_off.data_ptr(), d_len.data_ptr(), n, tok_off.data_ptr(),
                              tok_len.data_ptr(), tok_col.data_ptr(), tok_fl.data_ptr(), esc.data_ptr(),
                              kind.data_ptr(), ntok.data_ptr(), err.data_ptr(), _stream()), "tokenize")
    h_text, h_esc = text.cpu().numpy().tobytes(), esc.cpu().numpy().tobytes()
    h_off, h_len = tok_off.cpu().numpy(), tok_len.cpu().numpy()
    h_col, h_fl = tok_col.cpu().numpy(), tok_fl.cpu().numpy()
    h_kind, h_nt, h_err = kind.cpu().numpy(), ntok.cpu().numpy(), err.cpu().numpy()
    out = []
    for li in range(n):
        toks = []
        for k in range(int(offs[li]), int(offs[li]) + int(h_nt[li])):
            src = h_esc if h_fl[k] & 1 else h_text
            o = int(h_off[k])
            toks.append((src[o:o + int(h_len[k])], int(h_col[k]), bool(h_fl[k] & 1)))
        out.append((int(h_kind[li]), toks, int(h_err[li])))
    return out


ENC_MESSAGES = {1: "header bound is 0; recompute the bound before serializing"}


def run_encode_modules(headers, opcodes, op_counts, operands, inst_counts):
    """Batch encode_module: headers int64[n, 5] (major, minor, generator & mask, bound,
    schema & mask), per instruction opcode / operand count, operand words uint32 (masked),
    instructions per module.  -> (words uint32 arena, word offset per module (n + 1),
    err uint64 per module: all ones = ok, else (k << 8) | code)."""
    torch = _torch()
    headers = np.ascontiguousarray(headers, dtype=np.int64).reshape(-1, 5)
    n = len(headers)
    if n == 0:
        return np.zeros(0, np.uint32), np.zeros(1, np.int64), np.zeros(0, np.uint64)
    inst_counts = np.asarray(inst_counts, dtype=np.int64)
    inst_base = np.zeros(n + 1, dtype=np.int64)
    inst_base[1:] = np.cumsum(inst_counts)
    op_counts = np.asarray(op_counts, dtype=np.int64)
    n_inst = int(inst_base[-1])
    op_off = np.zeros(n_inst + 1, dtype=np.int64)
    op_off[1:] = np.cumsum(op_counts)
    n_ops = int(op_off[-1])
    mod_words = 5 * np.arange(n + 1, dtype=np.int64) + inst_base + op_off[inst_base]
    total = int(mod_words[-1])
    out = torch.zeros(max(total, 1), dtype=torch.int32, device="cuda")
    err = torch.zeros(n, dtype=torch.int64, device="cuda")
    d_hdr, d_ib = _dev(headers.reshape(-1), np.int64), _dev(inst_base, np.int64)
    d_opc, d_oo = _dev(opcodes, np.int64), _dev(op_off, np.int64)
    d_ops = _dev(np.asarray(operands, dtype=np.uint32).view(np.int32), np.int32)
    _check(lib().skg_encode_modules(d_hdr.data_ptr(), n, d_ib.data_ptr(), d_opc.data_ptr(), n_inst,
                                    d_oo.data_ptr(), d_ops.data_ptr(), n_ops, out.data_ptr(), err.data_ptr(),
                                    _stream()), "encode_modules")
    return (_pinned.to_u32(out, total) if total else np.zeros(0, np.uint32)), mod_words, \
        err.cpu().numpy().view(np.uint64)


def run_pack_strings(raws):
    """list[bytes] -> (words uint32 arena, word offsets (n + 1), has-NUL flags)."""
    torch = _torch()
    n = len(raws)
    lens = np.array([len(r) for r in raws], dtype=np.int64)
    offs = np.zeros(n, dtype=np.int64)
    if n > 1:
        offs[1:] = np.cumsum(lens)[:-1]
    wo = np.zeros(n + 1, dtype=np.int64)
    wo[1:] = np.cumsum(lens // 4 + 1)
    total = int(wo[-1])
    data = _dev(np.frombuffer(b"".join(raws) + b"\0", dtype=np.uint8), np.uint8)
    out = torch.zeros(max(total, 1), dtype=torch.int32, device="cuda")
    bad = torch.zeros(max(n, 1), dtype=torch.int32, device="cuda")
    d_off, d_len, d_wo = _dev(offs, np.int64), _dev(lens, np.int64), _dev(wo, np.int64)
    _check(lib().skg_pack_strings(data.data_ptr(), d_off.data_ptr(), d_len.data_ptr(), d_wo.data_ptr(), n, total,
                                  out.data_ptr(), bad.data_ptr(), _stream()), "pack_strings")
    return out.cpu().numpy().view(np.uint32)[:total], wo, bad.cpu().numpy()[:n]


def run_ctx_literals(widths, flags, vals):
    """Batch encode_context_dependent_literal -> (words uint32[n, 2], nwords, status)."""
    torch = _torch()
    n = len(widths)
    words = torch.zeros(2 * max(n, 1), dtype=torch.int32, device="cuda")
    nw = torch.zeros(max(n, 1), dtype=torch.int32, device="cuda")
    st = torch.zeros(max(n, 1), dtype=torch.int32, device="cuda")
    d_w, d_f = _dev(widths, np.int64), _dev(np.asarray(flags, dtype=np.uint32).view(np.int32), np.int32)
    d_v = _dev(np.asarray(vals, dtype=np.uint64).view(np.int64), np.int64)
    _check(lib().skg_ctx_literals(d_w.data_ptr(), d_f.data_ptr(), d_v.data_ptr(), n, words.data_ptr(),
                                  nw.data_ptr(), st.data_ptr(), _stream()), "ctx_literals")
    return words.cpu().numpy().view(np.uint32).reshape(-1, 2)[:n], nw.cpu().numpy()[:n], st.cpu().numpy()[:n]


__all__ = ["lib", "DeviceBatch", "run_disasm", "run_validate", "run_decode", "fetch_texts",
           "make_exception", "NativeUnavailable", "tables_handle", "struct"]


class DisasmPlan:
    """Preallocated device outputs for repeated launches over one DeviceBatch.

    ``launch()`` enqueues the workspace reset + ``skg_disasm`` on the current
    stream and returns immediately (no host synchronisation), which is what the
    benchmark times.  ``check()`` synchronises and verifies capacity/error counts.
    """

    def __init__(self, batch: DeviceBatch, opts: int, spec=None, ext=None, text_cap=None,
                 kind: str = "disasm", ws=None, bufs=None):
        """``bufs``: optional caller-owned device buffers (``text``, ``span``, ``status``,
        ``errs``; grow-only pools of a session) used instead of fresh allocations."""
        torch = _torch()
        bufs = bufs or {}
        self.kind = kind
        self.batch, self.opts = batch, opts
        self.th = tables_handle(spec, ext)
        n = batch.n
        self.ws_bytes = int(lib().skg_workspace_bytes(n, max(batch.max_words, 1)))
        if ws is not None and ws.numel() >= self.ws_bytes:   # shared by plans launched in order
            self.ws = ws
        else:
            self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device="cuda")
        self.cap = text_cap if text_cap is not None else 6 * batch.total_bytes + 4096
        self.ecap = max(16, min(n, 1 << 16))

        def buf(name, numel, dtype):
            b = bufs.get(name)
            if b is not None and b.numel() >= numel and b.dtype == dtype:
                return b[:numel]
            return torch.empty(numel, dtype=dtype, device="cuda")
        self.text = buf("text", self.cap, torch.uint8)
        self.span = buf("span", 2 * max(n, 1), torch.int64)
        self.status = buf("status", max(n, 1), torch.int32)
        self.errs = buf("errs", self.ecap * 256, torch.uint8)
        if kind == "pipeline":   # fused validation outputs (skg_disasm_validate)
            self.vcap = batch.total_bytes + 4096
            self.vtext = torch.empty(self.vcap, dtype=torch.uint8, device="cuda")
            self.vspan = torch.empty(2 * max(n, 1), dtype=torch.int64, device="cuda")
            self.vstatus = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
            self.verrs = torch.empty(self.ecap * 256, dtype=torch.uint8, device="cuda")

    def launch(self, stream=None):
        b = self.batch
        s = stream if stream is not None else _stream()
        if self.kind == "pipeline":
            rc = lib().skg_disasm_validate(self.th, b.data.data_ptr(), b.off.data_ptr(), b.len.data_ptr(), b.n,
                                           self.opts, b.max_words, self.text.data_ptr(), self.cap,
                                           self.span.data_ptr(), self.status.data_ptr(), self.errs.data_ptr(),
                                           self.ecap, self.vtext.data_ptr(), self.vcap, self.vspan.data_ptr(),
                                           self.vstatus.data_ptr(), self.verrs.data_ptr(), self.ecap,
                                           self.ws.data_ptr(), self.ws_bytes, s)
        elif self.kind == "disasm":
            rc = lib().skg_disasm(self.th, b.data.data_ptr(), b.off.data_ptr(), b.len.data_ptr(), b.n,
                                  self.opts, b.max_words, self.text.data_ptr(), self.cap,
                                  self.span.data_ptr(), self.status.data_ptr(), self.errs.data_ptr(),
                                  self.ecap, self.ws.data_ptr(), self.ws_bytes, s)
        else:
            rc = lib().skg_validate(self.th, b.data.data_ptr(), b.off.data_ptr(), b.len.data_ptr(), b.n,
                                    b.max_words, self.text.data_ptr(), self.cap, self.span.data_ptr(),
                                    self.status.data_ptr(), self.errs.data_ptr(), self.ecap,
                                    self.ws.data_ptr(), self.ws_bytes, s)
        _check(rc, self.kind)

    def check(self):
        nerr, over, used = last_counts(self.ws)
        info = {"errors": nerr, "overflow": over, "text_bytes": used}
        if self.kind == "pipeline":
            vnerr, vover, vused = last_counts(self.ws[VAL_COUNTERS:])
            info.update(verrors=vnerr, voverflow=vover, vtext_bytes=vused)
            info["overflow"] = over or vover
        return info

    def grow(self, need):
        torch = _torch()
        self.cap = need + 16
        self.text = torch.empty(self.cap, dtype=torch.uint8, device="cuda")

    def fit(self):
        """Run once and shrink/grow the text arena to the exact size needed."""
        self.launch()
        info = self.check()
        if info["overflow"] or info["text_bytes"] + 16 != self.cap:
            self.grow(info["text_bytes"])
            self.launch()
            info = self.check()
        return info


# -- assembler -----------------------------------------------------------------------
ST_OVERFLOW, ST_ASSEMBLY, ST_STRUCTURE, ST_SERIALIZATION = 8, 9, 10, 11


def _bind_asm(L):
    if getattr(L, "_asm_bound", False):
        return L
    P, U32, U64, I32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32
    L.skg_asm_slot_hint.argtypes = [U64]
    L.skg_asm_slot_hint.restype = U64
    L.skg_asm_workspace_bytes.argtypes = [U64, U32]
    L.skg_asm_workspace_bytes.restype = U64
    L.skg_asm.argtypes = [P, P, P, P, U32, U32, U64, P, U64, P, P, P, U64, P, U32]  # ..., stream, default_version
    L.skg_asm.restype = I32
    L._asm_bound = True
    return L


def pack_texts(texts):
    """list[str] -> (uint8 arena, int64 offsets, int64 lengths); module starts 16-byte aligned."""
    raws = [t.encode("utf-8", "surrogatepass") if isinstance(t, str) else bytes(t) for t in texts]
    lengths = np.array([len(r) for r in raws], dtype=np.int64)
    padded = (lengths + 15) // 16 * 16
    offsets = np.zeros(len(raws), dtype=np.int64)
    if len(raws) > 1:
        offsets[1:] = np.cumsum(padded)[:-1]
    buf = np.zeros(int(padded.sum()) + 16, dtype=np.uint8)
    for r, o in zip(raws, offsets):
        buf[o:o + len(r)] = np.frombuffer(r, dtype=np.uint8)
    return buf, offsets, lengths


class AsmPlan:
    """Device buffers for repeated skg_asm launches over one resident text batch."""

    def __init__(self, batch: DeviceBatch, spec=None, ext=None, out_cap=None, slot_bytes=None,
                 default_version=(1, 2), stride=1, ws=None, bufs=None):
        """``bufs``: optional caller-owned device buffers (``out``, ``span``, ``status``)."""
        torch = _torch()
        bufs = bufs or {}
        L = _bind_asm(lib())
        self.batch = batch
        self.stride = stride
        self.th = tables_handle(spec, ext)
        n = batch.n
        max_len = int(batch.max_words) * 4 + 16
        self.slot = int(slot_bytes or L.skg_asm_slot_hint(max_len))
        self.ws_bytes = int(L.skg_asm_workspace_bytes(self.slot, max(n, 1)))
        if ws is not None and ws.numel() >= self.ws_bytes:   # shared by plans launched in order
            self.ws = ws
        else:
            self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device="cuda")
        self.cap = int(out_cap or (batch.total_bytes + 64 * n + 4096))

        def buf(name, numel, dtype):
            b = bufs.get(name)
            if b is not None and b.numel() >= numel and b.dtype == dtype:
                return b[:numel]
            return torch.empty(numel, dtype=dtype, device="cuda")
        self.out = buf("out", self.cap, torch.uint8)
        self.span = buf("span", 2 * max(n, 1), torch.int64)
        self.status = buf("status", max(n, 1), torch.int32)
        maj, mnr = default_version
        self.dv = ((int(maj) & 0xFFFF) << 16) | (int(mnr) & 0xFFFF)

    def launch(self, stream=None):
        b = self.batch
        s = stream if stream is not None else _stream()
        rc = lib().skg_asm(self.th, b.data.data_ptr(), b.off.data_ptr(), b.len.data_ptr(), self.stride, b.n,
                           self.slot,
                           self.out.data_ptr(), self.cap, self.span.data_ptr(), self.status.data_ptr(),
                           self.ws.data_ptr(), self.ws_bytes, s, self.dv)
        _check(rc, "asm")

    def check(self):
        nerr, over, used = last_counts(self.ws)
        return {"overflow": over, "bytes": used}

    def grow(self, need):
        torch = _torch()
        self.cap = int(need) + 4096
        self.out = torch.empty(self.cap, dtype=torch.uint8, device="cuda")

    def fit(self):
        self.launch()
        info = self.check()
        if info["overflow"]:
            self.grow(info["bytes"])
            self.launch()
            info = self.check()
        return info


def asm_exception(status, msg: str):
    if status == ST_ASSEMBLY:
        lines = msg.split("\n")
        diags = []
        for ln in lines[1:]:
            a, b, rest = ln.split(":", 2)
            diags.append(_err.AsmDiagnostic(int(a), int(b), rest[1:]))
        exc = _err.AssemblyError(diags)
        return exc
    if status == ST_VALUE:
        return ValueError(msg)
    if status == ST_OVERFLOW:
        return OverflowError(msg)
    if status == ST_STRUCTURE:
        return _err.StructureError(msg)
    if status == ST_SERIALIZATION:
        return _err.SerializationError(msg)
    if status == ST_CODEC:
        return _err.CodecError(msg)
    return RuntimeError(f"libskgpu internal error: {msg}")


def run_asm(texts, spec=None, ext=None, default_version=(1, 2)):
    """list[str] -> list[bytes | exception instance]."""
    buf, off, ln = pack_texts(texts)
    n = len(texts)
    if n == 0:
        return []
    batch = DeviceBatch.from_host(buf, off, ln)
    batch.max_words = (int(ln.max()) + 3) // 4
    # per-warp slot for the largest text, capped by the workspace budget; modules
    # that need more report ST_INTERNAL and are rerun alone with larger slots below
    L = _bind_asm(lib())
    hint = int(L.skg_asm_slot_hint(int(batch.max_words) * 4 + 16))
    n_warps = int(L.skg_asm_workspace_bytes(1, n)) - int(L.skg_asm_workspace_bytes(0, n))   # slots
    per_warp_cap = max(1 << 20, WS_BUDGET // max(n_warps, 1))
    plan = AsmPlan(batch, spec, ext, slot_bytes=min(hint, per_warp_cap), default_version=default_version)
    plan.fit()
    status = plan.status[:n].cpu().numpy()
    span = plan.span[: 2 * n].cpu().numpy()
    out = _pinned.to_bytes(plan.out)
    res = []
    retry = []
    for m in range(n):
        o, k = int(span[2 * m]), int(span[2 * m + 1])
        data = out[o:o + k]
        st = int(status[m])
        if st == ST_OK:
            res.append(data)
        elif st == ST_INTERNAL:
            res.append(None)
            retry.append(m)
        else:
            res.append(asm_exception(st, data.decode("utf-8", "surrogatepass")))
    for m in retry:   # module larger than the default per-warp scratch: rerun alone, bigger slot
        slot = plan.slot
        for _ in range(6):
            slot *= 4
            b1, o1, l1 = pack_texts([texts[m]])
            single = DeviceBatch.from_host(b1, o1, l1)
            single.max_words = (int(l1.max()) + 3) // 4
            p1 = AsmPlan(single, spec, ext, slot_bytes=slot, default_version=default_version)
            p1.fit()
            st = int(p1.status[0].item())
            if st == ST_INTERNAL:
                continue
            o, k = (int(x) for x in p1.span[:2].cpu().numpy())
            data = p1.out[o:o + k].cpu().numpy().tobytes()
            res[m] = data if st == ST_OK else asm_exception(st, data.decode("utf-8", "surrogatepass"))
            break
        else:
            res[m] = RuntimeError("libskgpu internal error: module exceeds the assembler scratch")
    return res
