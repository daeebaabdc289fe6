"""Oracle: binary -> text disassembly (TEST INFRASTRUCTURE ONLY).

Restates ``spirvkit/disasm.py`` (``Disassembler.to_text`` 117-127, prescan
131-157, friendly names 159-219, section tracking 253-267, rendering 269-377,
layout 284-318).  The friendly-name demotion is computed with the closed form
of SURVEY.md appendix A.3 (``refs_closed_form``); the reference's literal
restart-on-demotion fixpoint is kept as ``refs_fixpoint`` and the two are
cross-checked in the tests.
"""

from __future__ import annotations

import re

from paper_2305_09493_b200 import grammar as _grammar
from paper_2305_09493_b200.errors import CodecError

from .core import TypeMaps, decode_module, decode_operands, decode_string

ANSI = {"opcode": "\x1b[36m", "id": "\x1b[33m", "string": "\x1b[32m",
        "comment": "\x1b[90m", "reset": "\x1b[0m"}                       # disasm.py:18-24
SECTION_BY_NAME = {"OpCapability": 0, "OpExtension": 1, "OpExtInstImport": 2,
                   "OpMemoryModel": 3, "OpEntryPoint": 4, "OpExecutionMode": 5,
                   "OpExecutionModeId": 5}                                # disasm.py:26-34
SECTION_BY_CLASS = {"Debug": 6, "Annotation": 7, "Type-Declaration": 8,
                    "Constant-Creation": 8}                               # disasm.py:36-41
FUNCTION_SECTION = 9


class Options:
    def __init__(self, highlight=False, inline_names=True, no_indent=False, group=False,
                 no_header=False):
        self.highlight, self.inline_names = highlight, inline_names
        self.no_indent, self.group, self.no_header = no_indent, group, no_header


def sanitize(raw: str) -> str:
    """disasm.py:82-86."""
    text = re.sub(r"[^0-9A-Za-z_]", "_", raw)
    return "_" + text if not text or text[0].isdigit() else text


class Context:
    def __init__(self, maps: TypeMaps):
        self.maps = maps
        self.refs = {}
        self.import_sets = {}

    def ref(self, ident):
        return self.refs.get(ident) or f"%{ident}"


def _opdef(spec, opcode):
    return spec.instruction(opcode) if spec.has_instruction(opcode) else None


def definition_order(spec, insts):
    """disasm.py:208-219."""
    order, seen = [], set()
    for opcode, words in insts:
        d = _opdef(spec, opcode)
        if d is None or not d.has_result:
            continue
        i = 1 if d.has_result_type else 0
        if i < len(words) and words[i] not in seen:
            seen.add(words[i])
            order.append(words[i])
    return order


def referenced_ids(spec, insts, maps):
    """disasm.py:221-240 (CodecError instructions skipped, others escape)."""
    ids = set()

    def collect(ops):
        for o in ops:
            if o.role in ("result", "result_type", "id"):
                ids.add(o.value)
            elif o.role == "composite":
                collect(o.components)

    for opcode, words in insts:
        d = _opdef(spec, opcode)
        if d is None:
            continue
        try:
            collect(decode_operands(spec, d, words, maps.resolve))
        except CodecError:
            continue
    return ids


def unique_names(order, names):
    """disasm.py:173-185: sanitize, then base, base_0, base_1, ... in D order.

    The reference retries every serial from 0 for each duplicate (quadratic in
    the duplicates of one base).  The taken set only grows, so serials that
    were taken at a base's previous duplicate still are: restarting from the
    serial after the one that base took last gives the same names in linear
    time (needed for the config-3 module, ~10^7 named ids over a dozen bases).
    """
    out, taken, nxt = {}, set(), {}
    for ident in order:
        if ident not in names:
            continue
        base = sanitize(names[ident])
        cand = base
        if cand in taken:
            serial = nxt.get(base, 0)
            cand = f"{base}_{serial}"
            while cand in taken:
                serial += 1
                cand = f"{base}_{serial}"
            nxt[base] = serial + 1
        taken.add(cand)
        out[ident] = cand
    return out


def refs_fixpoint(order, uniq, all_ids):
    """disasm.py:187-206, literally (restart after every demotion)."""
    pinned = {i for i in all_ids if i not in uniq}
    while True:
        assigned, demoted = set(), None
        for ident in order:
            if ident in pinned:
                continue
            fresh = 1
            while fresh in pinned or fresh in assigned:
                fresh += 1
            if fresh != ident:
                demoted = ident
                break
            assigned.add(ident)
        if demoted is None:
            break
        pinned.add(demoted)
    return {i: f"%{uniq[i]}" for i in order if i in uniq and i not in pinned}


def refs_closed_form(order, uniq, all_ids):
    """c_j keeps its name iff [1, c_j) is covered by P0 and c_1..c_{j-1}."""
    p0 = {i for i in all_ids if i not in uniq}
    chain = [i for i in order if i not in p0]
    limit = len(p0) + len(chain)
    pos = [None] * (limit + 1)              # None = hole (+inf)
    for v in p0:
        if 1 <= v <= limit:
            pos[v] = -1
    for j, c in enumerate(chain):
        if 1 <= c <= limit:
            pos[c] = j
    out, run, prefix = {}, -1, [-1] * (limit + 1)   # prefix[v] = max(pos[1..v])
    for v in range(1, limit + 1):
        run = max(run, float("inf") if pos[v] is None else pos[v])
        prefix[v] = run
    for j, c in enumerate(chain):
        kept = 1 <= c <= limit and (c == 1 or prefix[c - 1] < j)
        if kept and c in uniq:
            out[c] = f"%{uniq[c]}"
    return out


def prescan(spec, insts, options, closed_form=True):
    """disasm.py:131-157 + _assign_refs 159-206."""
    maps = TypeMaps(spec, insts)
    ctx = Context(maps)
    names = {}
    for opcode, words in insts:
        d = _opdef(spec, opcode)
        name = d.name if d else None
        if name == "OpExtInstImport" and len(words) >= 2:
            try:
                ctx.import_sets[words[0]], _ = decode_string(words, 1)
            except CodecError:
                pass
        elif name == "OpName" and len(words) >= 2:
            try:
                text, _ = decode_string(words, 1)
            except CodecError:
                continue
            names.setdefault(words[0], text)
    if options.inline_names and names:
        order = definition_order(spec, insts)
        uniq = unique_names(order, names)
        all_ids = referenced_ids(spec, insts, maps)
        ctx.refs = (refs_closed_form if closed_form else refs_fixpoint)(order, uniq, all_ids)
    return ctx


def advance_section(d, section, in_function):
    """disasm.py:253-267."""
    if d is None:
        return section, in_function
    if d.name == "OpFunction":
        return FUNCTION_SECTION, True
    if in_function:
        return FUNCTION_SECTION, d.name != "OpFunctionEnd"
    if d.name in SECTION_BY_NAME:
        return SECTION_BY_NAME[d.name], False
    if d.class_attr in SECTION_BY_CLASS:
        return SECTION_BY_CLASS[d.class_attr], False
    if d.name in ("OpVariable", "OpUndef"):
        return 8, False
    return section, in_function


def operand_tokens(o, ctx, spec, ext, ext_known):
    """disasm.py:339-377."""
    r = o.role
    if r in ("id", "result_type"):
        return [(ctx.ref(o.value), "id")]
    if r == "value_enum":
        return [(o.enumerant.name if o.enumerant is not None else str(o.value), None)]
    if r == "bit_enum":
        if o.value == 0:
            zero = next((e.name for e in o.kind.enumerants or () if e.value == 0), "0")
            return [(zero, None)]
        if o.components:
            return [("|".join(e.name for e in o.components), None)]
        return [(f"0x{o.value:x}", None)]
    if r == "string":
        return [('"' + o.value.replace("\\", "\\\\").replace('"', '\\"') + '"', "string")]
    if r == "ctx_number":
        return [(repr(o.value) if isinstance(o.value, float) else str(o.value), None)]
    if r == "ext_number":
        if ext_known and ext is not None and ext.has_instruction(o.value):
            return [(ext.instruction(o.value).name, None)]
        return [(str(o.value), None)]
    if r == "spec_opcode":
        if spec.has_instruction(o.value):
            return [(spec.instruction(o.value).name[2:], None)]
        return [(str(o.value), None)]
    if r == "composite":
        toks = []
        for part in o.components:
            toks.extend(operand_tokens(part, ctx, spec, ext, ext_known))
        return toks
    return [(str(o.value), None)]


def render(d, decoded, ctx, spec, ext):
    """disasm.py:321-336 (format_operands)."""
    tokens, result_ref, ext_known = [(d.name, "opcode")], None, True
    if d.name == "OpExtInst":
        set_ids = [o.value for o in decoded if o.role == "id"]
        ext_known = bool(set_ids) and ctx.import_sets.get(set_ids[0]) == "OpenCL.std"
    for o in decoded:
        if o.role == "result":
            result_ref = ctx.ref(o.value)
            continue
        tokens.extend(operand_tokens(o, ctx, spec, ext, ext_known))
    return result_ref, tokens


def disassemble(data: bytes, options=None, spec=None, ext=None, strict=False,
                closed_form=True) -> str:
    """disasm.py:117-127 + 284-318."""
    options = options if options is not None else Options()
    spec = spec if spec is not None else _grammar.load_pinned()
    ext = ext if ext is not None else _grammar.load_pinned_extended()
    header, insts = decode_module(data)
    ctx = prescan(spec, insts, options, closed_form)
    rows, section, in_fn = [], 0, False
    for opcode, words in insts:
        d = _opdef(spec, opcode)
        section, in_fn = advance_section(d, section, in_fn)
        if d is None:
            if strict:
                raise CodecError(f"unknown opcode {opcode}")
            toks = [(f"OpUnknown({opcode})", "opcode")] + [(f"!0x{w:08X}", None) for w in words]
            rows.append((None, toks, section))
            continue
        decoded = decode_operands(spec, d, words, ctx.maps.resolve)
        ref, toks = render(d, decoded, ctx, spec, ext)
        rows.append((ref, toks, section))

    def paint(text, color):
        if not options.highlight or color is None:
            return text
        return ANSI[color] + text + ANSI["reset"]

    width = 0 if options.no_indent else max((len(r) for r, _, _ in rows if r), default=0)
    out = []
    if not options.no_header:
        major, minor, gen, bound, schema = header
        for line in ("; SPIR-V", f"; Version: {major}.{minor}",
                     f"; Generator: {gen >> 16}; {gen & 0xFFFF}", f"; Bound: {bound}",
                     f"; Schema: {schema}"):
            out.append(paint(line, "comment"))
    prev = None
    for ref, toks, section in rows:
        if options.group and prev is not None and section != prev:
            out.append("")
        prev = section
        body = " ".join(paint(t, c) for t, c in toks)
        if ref is not None:
            pad = " " * (width - len(ref)) if width else ""
            out.append(f"{pad}{paint(ref, 'id')} = {body}")
        else:
            out.append((" " * (width + 3) if width else "") + body)
    return "\n".join(out) + "\n" if out else ""
