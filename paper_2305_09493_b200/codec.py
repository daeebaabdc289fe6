"""Binary codec on the GPU (reference ``spirvkit/codec.py``).

Types: ``ModuleHeader`` / ``RawInstruction`` (:23-41), ``TypedInt`` /
``TypedFloat`` (:44-58).  Decode: ``decode_module`` (:199-231) -- the
instruction-boundary walk, magic/endianness normalisation and every error
message come from the CUDA ``skg_decode`` kernel; Python only wraps the offsets
into the reference's objects.  Encode: ``encode_header`` (:61-79),
``encode_instruction`` (:92-101), ``encode_string_literal`` (:104-114),
``encode_context_dependent_literal`` (:132-168) and ``encode_module``
(:192-196) run the batch kernels of ``csrc/skg_codec.cuh``; ``encode_modules``
is the batch entry point (builder serialization of many modules at once,
SURVEY 8(f)1).  Python marshals arguments (ints masked / range-flagged, str ->
UTF-8) and raises the reference's exceptions from the per-item status codes.
"""

from __future__ import annotations

from dataclasses import dataclass

import struct

import numpy as np

from . import _native
from .errors import CodecError

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


# -- encode (csrc/skg_codec.cuh) --------------------------------------------------------
_I64_MIN, _I64_MAX = -(1 << 63), (1 << 63) - 1


def _i64(v) -> int:
    """an int field as int64 for the device range checks (out-of-int64 values are
    outside every range the kernels accept: the sentinel keeps them failing)"""
    v = int(v)
    return v if _I64_MIN <= v <= _I64_MAX else _I64_MIN


def _header_row(h):
    return [_i64(h.major_version), _i64(h.minor_version), int(h.generator_magic) & WORD_MASK,
            _i64(h.bound), int(h.schema) & WORD_MASK]


def _encode_error(code: int, header, insts, k: int) -> CodecError:
    if code == 1:
        return CodecError("header bound is 0; recompute the bound before serializing")
    if code == 2:
        return CodecError(f"header bound {header.bound} out of range")
    if code == 3:
        return CodecError("version bytes out of range")
    inst = insts[k - 1]
    if code == 4:
        return CodecError(f"instruction length {1 + len(inst.operands)} words overflows the 16-bit count")
    return CodecError(f"opcode {inst.opcode} out of range")


def encode_modules(modules):
    """Batch encode_module: [(ModuleHeader, [RawInstruction])] -> list[bytes | CodecError]
    (exception instances, not raised)."""
    modules = [(h, list(insts)) for h, insts in modules]
    if not modules:
        return []
    headers = np.array([_header_row(h) for h, _ in modules], dtype=np.int64).reshape(-1, 5)
    inst_counts = [len(insts) for _, insts in modules]
    flat = [i for _, insts in modules for i in insts]
    opcodes = np.array([_i64(i.opcode) for i in flat], dtype=np.int64)
    op_counts = np.array([len(i.operands) for i in flat], dtype=np.int64)
    ops = np.fromiter((int(w) & WORD_MASK for i in flat for w in i.operands), dtype=np.uint32,
                      count=int(op_counts.sum()))
    words, mod_words, err = _native.run_encode_modules(headers, opcodes, op_counts, ops, inst_counts)
    out = []
    for m, (h, insts) in enumerate(modules):
        e = int(err[m])
        if e != 0xFFFFFFFFFFFFFFFF:
            out.append(_encode_error(e & 0xFF, h, insts, e >> 8))
        else:
            out.append(words[int(mod_words[m]):int(mod_words[m + 1])].astype("<u4").tobytes())
    return out


def _raise_or(x):
    if isinstance(x, BaseException):
        raise x
    return x


def encode_module(header: ModuleHeader, instructions) -> bytes:
    """codec.py:192-196 on the GPU."""
    return _raise_or(encode_modules([(header, instructions)])[0])


def encode_header(header: ModuleHeader) -> list[int]:
    """codec.py:61-79 on the GPU (the five header words)."""
    data = encode_module(header, [])
    return list(struct.unpack("<5I", data))


def encode_instruction(inst) -> list[int]:
    """codec.py:92-101 on the GPU."""
    data = encode_module(ModuleHeader(0, 0, 0, 1, 0), [inst])
    return list(struct.unpack(f"<{len(data) // 4}I", data))[5:]


def encode_string_literals(texts):
    """Batch encode_string_literal -> list[list[int] | CodecError]."""
    raws = [t.encode("utf-8") for t in texts]
    if not raws:
        return []
    words, wo, bad = _native.run_pack_strings(raws)
    return [CodecError("string literal contains an embedded NUL byte") if bad[k]
            else words[int(wo[k]):int(wo[k + 1])].tolist() for k in range(len(raws))]


def encode_string_literal(text: str) -> list[int]:
    """codec.py:104-114 on the GPU."""
    return _raise_or(encode_string_literals([text])[0])


_LIT_SIGNED, _LIT_FLOAT, _LIT_NEG, _LIT_BIG, _LIT_NONE = 1, 2, 4, 8, 16


def encode_context_dependent_literals(items):
    """Batch encode_context_dependent_literal: [(value, bit_width, signed, floating)]
    -> list[list[int] | exception]."""
    widths, flags, vals, conv = [], [], [], []
    for value, bit_width, signed, floating in items:
        w = 0 if bit_width is None else _i64(bit_width)
        widths.append(w if w != _I64_MIN else 0)          # (out of int64: unsupported, as 0)
        f = (_LIT_SIGNED if signed else 0) | (_LIT_FLOAT if floating else 0) | \
            (_LIT_NONE if bit_width is None else 0)
        v, err, shown = 0, None, None
        try:                           # argument conversion; any failure surfaces only if
            if floating:               # the device accepts the width first (codec.py order)
                if not isinstance(value, (int, float)):
                    raise struct.error("required argument is not a float")
                try:
                    v = struct.unpack("<Q", struct.pack("<d", float(value)))[0]
                except OverflowError:
                    raise struct.error("required argument is not a float") from None
            else:
                iv = int(value)
                shown = iv
                mag = -iv if iv < 0 else iv
                if iv < 0:
                    f |= _LIT_NEG
                if mag >> 64:
                    f |= _LIT_BIG
                else:
                    v = mag
        except Exception as exc:  # noqa: BLE001 - re-raised below in the reference's order
            err = exc
        flags.append(f)
        vals.append(v)
        conv.append((err, shown))
    if not items:
        return []
    words, nw, st = _native.run_ctx_literals(np.array(widths, np.int64), np.array(flags, np.uint32),
                                             np.array(vals, np.uint64))
    out = []
    for k, (value, bit_width, signed, floating) in enumerate(items):
        s, (err, shown) = int(st[k]), conv[k]
        if s == 1:
            out.append(CodecError("context-dependent literal has an unresolved bit width"))
        elif s == 2:
            out.append(CodecError(f"unsupported literal width {bit_width}"))
        elif s == 3:
            out.append(CodecError(f"unsupported float width {bit_width}"))
        elif err is not None:
            out.append(err)
        elif s == 4:
            out.append(OverflowError("float too large to pack with e format"))
        elif s == 5:
            out.append(OverflowError("float too large to pack with f format"))
        elif s == 6:
            out.append(CodecError(f"value {shown} does not fit a signed {bit_width}-bit literal"))
        elif s == 7:
            out.append(CodecError(f"value {shown} does not fit an unsigned {bit_width}-bit literal"))
        else:
            out.append([int(x) for x in words[k, : int(nw[k])]])
    return out


def encode_context_dependent_literal(value, bit_width, *, signed: bool = False,
                                     floating: bool = False) -> list[int]:
    """codec.py:132-168 on the GPU."""
    return _raise_or(encode_context_dependent_literals([(value, bit_width, signed, floating)])[0])


def decode_header(words) -> ModuleHeader:
    """codec.py:82-89 (field extraction of five already-decoded words)."""
    return ModuleHeader(major_version=(words[1] >> 16) & 0xFF, minor_version=(words[1] >> 8) & 0xFF,
                        generator_magic=words[2], bound=words[3], schema=words[4])


def literal_word_count(bit_width: int) -> int:
    """codec.py:188-189."""
    return 2 if bit_width == 64 else 1


def serialize_modules(scopes):
    """Batch ModuleScope.serialize (builder.py:187-224) -> list[bytes | exception].

    The builder objects stay the caller's (host) structure: each scope's
    instruction stream in logical-layout order, its structure / reference checks
    (StructureError / SerializationError) and its header (bound recomputed) come
    from the builder as in the reference; the words of every module -- header
    and instruction encoding with the codec.py range checks -- are produced by
    ONE skg_encode_modules launch for the whole batch."""
    out, work = [None] * len(scopes), []
    for k, scope in enumerate(scopes):
        try:
            stream = scope.instruction_stream()
            scope._check_references(stream)
            work.append((k, scope.header(), [inst.raw() for inst in stream]))
        except Exception as exc:  # noqa: BLE001 - the builder's own errors, per module
            out[k] = exc
    for (k, _, _), res in zip(work, encode_modules([(h, insts) for _, h, insts in work])):
        out[k] = res
    return out
