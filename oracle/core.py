"""Oracle: binary codec + grammar slot walk (TEST INFRASTRUCTURE ONLY).

Restates ``spirvkit/codec.py`` (decode side) and ``spirvkit/ops.py:316-446``
(``decode_operands``).  Operands are returned as ``Operand`` tuples with the
reference's role vocabulary (``ops.py:321-322``).
"""

from __future__ import annotations

import struct
from typing import NamedTuple

from paper_2305_09493_b200.errors import (CorruptStreamError, NotSpirvError,
                                          TruncatedStreamError)

MAGIC = 0x07230203


class Operand(NamedTuple):
    kind: object          # OperandKindDef
    role: str
    value: object
    enumerant: object = None
    components: tuple = ()


def decode_module(data: bytes):
    """codec.py:199-231 -> ((major, minor, generator, bound, schema), [(opcode, operands)])."""
    n = len(data)
    if n % 4 or n < 20:
        raise TruncatedStreamError(f"{n} bytes is not a whole word stream of at least 5 words")
    count = n // 4
    words = struct.unpack(f"<{count}I", data)
    if words[0] != MAGIC:
        swapped = struct.unpack(f">{count}I", data)
        if swapped[0] != MAGIC:
            raise NotSpirvError(f"magic word 0x{words[0]:08X} is not SPIR-V")
        words = swapped
    header = ((words[1] >> 16) & 0xFF, (words[1] >> 8) & 0xFF, words[2], words[3], words[4])
    insts, pos = [], 5
    while pos < count:
        wc, op = words[pos] >> 16, words[pos] & 0xFFFF
        if wc == 0:
            raise CorruptStreamError(f"instruction at word {pos} has word count 0")
        if pos + wc > count:
            raise TruncatedStreamError(f"instruction at word {pos} runs past the end of the stream")
        insts.append((op, tuple(words[pos + 1:pos + wc])))
        pos += wc
    return header, insts


def decode_string(words, start=0):
    """codec.py:117-129: bytes up to the first NUL byte, strict UTF-8."""
    raw = bytearray()
    for i in range(start, len(words)):
        chunk = words[i].to_bytes(4, "little")
        cut = chunk.find(0)
        if cut >= 0:
            raw += chunk[:cut]
            return bytes(raw).decode("utf-8"), i + 1
        raw += chunk
    raise CorruptStreamError("string literal is not NUL-terminated")


def decode_ctx_literal(raw, width, signed=False, floating=False):
    """codec.py:171-185 (KeyError / ValueError escape exactly as there)."""
    if floating:
        if width == 64:
            return struct.unpack("<d", struct.pack("<2I", raw[0], raw[1]))[0]
        fmt = {16: "<e", 32: "<f", 64: "<d"}[width]        # KeyError(width)
        return struct.unpack(fmt, struct.pack("<I", raw[0])[: width // 8])[0]
    if width == 64:
        bits = raw[0] | (raw[1] << 32)
    else:
        # (1 << width) - 1 for width >= 32 keeps the whole word; avoid building
        # a 2**width integer for absurd widths (same value).
        bits = raw[0] & (((1 << width) - 1) if width < 32 else 0xFFFFFFFF)
    if signed:
        if width == 0:
            raise ValueError("negative shift count")
        if width <= 32 and bits >= (1 << (width - 1)):
            bits -= 1 << width
        elif width == 64 and bits >= (1 << 63):
            bits -= 1 << 64
    return bits


def literal_words(width):
    return 2 if width == 64 else 1


def bit_components(kind, mask):
    """ops.py:77-89: covering set-bit enumerants in file order, None if impossible."""
    if mask == 0:
        return []
    parts, covered = [], 0
    for e in kind.enumerants or ():
        v = e.value
        if v and (mask & v) == v and (covered & v) != v:
            parts.append(e)
            covered |= v
    return parts if covered == mask else None


class _Walk:
    """ops.py:358-446 decode state."""

    def __init__(self, spec, opdef, words, resolver):
        self.spec, self.opdef, self.words, self.pos = spec, opdef, words, 0
        self.resolver = resolver
        self.top = []

    def take(self):
        if self.pos >= len(self.words):
            raise CorruptStreamError(f"{self.opdef.name}: operand words exhausted mid-instruction")
        self.pos += 1
        return self.words[self.pos - 1]

    def one(self, kind_name, out):
        kind = self.spec.kind(kind_name)
        cat = kind.category
        if cat == "Id":
            role = {"IdResult": "result", "IdResultType": "result_type"}.get(kind.kind, "id")
            out.append(Operand(kind, role, self.take()))
        elif cat == "ValueEnum":
            word = self.take()
            enum = next((e for e in kind.enumerants or () if e.value == word), None)
            out.append(Operand(kind, "value_enum", word, enumerant=enum))
            for p in (enum.parameters if enum else ()):
                self.one(p.kind, out)
        elif cat == "BitEnum":
            mask = self.take()
            parts = bit_components(kind, mask)
            out.append(Operand(kind, "bit_enum", mask, components=tuple(parts or ())))
            for e in parts or ():
                for p in e.parameters:
                    self.one(p.kind, out)
        elif cat == "Composite":
            parts = []
            for b in kind.bases or ():
                self.one(b, parts)
            out.append(Operand(kind, "composite", None, components=tuple(parts)))
        else:
            self.literal(kind, out)

    def literal(self, kind, out):
        name, op = kind.kind, self.opdef.name
        if name == "LiteralString":
            text, self.pos = decode_string(self.words, self.pos)
            out.append(Operand(kind, "string", text))
            return
        if name == "LiteralContextDependentNumber":
            got = self.resolver(self.opdef, self.top) if self.resolver else None
            if got is None:
                raise CorruptStreamError(f"{op}: cannot resolve the width of a context-dependent literal")
            width, signed, floating = got
            raw = [self.take() for _ in range(literal_words(width))]
            out.append(Operand(kind, "ctx_number", decode_ctx_literal(raw, width, signed, floating)))
            return
        if name == "LiteralInteger" and op == "OpSwitch" and self.resolver:
            got = self.resolver(self.opdef, self.top)
            if got is not None:
                width, signed, _ = got
                raw = [self.take() for _ in range(literal_words(width))]
                out.append(Operand(kind, "literal", decode_ctx_literal(raw, width, signed)))
                return
        role = {"LiteralExtInstInteger": "ext_number",
                "LiteralSpecConstantOpInteger": "spec_opcode"}.get(name, "literal")
        out.append(Operand(kind, role, self.take()))


def decode_operands(spec, opdef, words, resolver=None):
    """ops.py:328-355."""
    w = _Walk(spec, opdef, list(words), resolver)
    out = w.top
    for slot in opdef.operands:
        if slot.quantifier == "*":
            while w.pos < len(w.words):
                w.one(slot.kind, out)
            break
        if slot.quantifier == "?" and w.pos >= len(w.words):
            continue
        w.one(slot.kind, out)
        if slot.kind == "LiteralSpecConstantOpInteger":
            while w.pos < len(w.words):
                w.one("IdRef", out)
    if w.pos < len(w.words):
        raise CorruptStreamError(f"{opdef.name}: {len(w.words) - w.pos} leftover operand word(s)")
    return out


def flat(operands):
    """validate.py:171-176."""
    for o in operands:
        if o.role == "composite":
            yield from flat(o.components)
        else:
            yield o


class TypeMaps:
    """The width maps behind the literal resolver.

    disasm.py:131-157 (prescan) and validate.py:179-204 build the same two
    maps: ``type_info`` from OpTypeInt (exactly 3 words) / OpTypeFloat (>= 2),
    ``value_type`` from every known instruction with result and result type
    (>= 2 words); later definitions overwrite earlier ones.
    """

    def __init__(self, spec, insts):
        self.type_info, self.value_type = {}, {}
        for opcode, words in insts:
            if not spec.has_instruction(opcode):
                continue
            d = spec.instruction(opcode)
            if d.name == "OpTypeInt" and len(words) == 3:
                self.type_info[words[0]] = (words[1], words[2] == 1, False)
            elif d.name == "OpTypeFloat" and len(words) >= 2:
                self.type_info[words[0]] = (words[1], False, True)
            if d.has_result and d.has_result_type and len(words) >= 2:
                self.value_type[words[1]] = words[0]

    def resolve(self, opdef, decoded):
        """disasm.py:69-79 / validate.py:194-202."""
        if opdef.name == "OpSwitch":
            if not decoded:
                return None
            return self.type_info.get(self.value_type.get(decoded[0].value, -1))
        for o in decoded:
            if o.role == "result_type":
                return self.type_info.get(o.value)
        return None
