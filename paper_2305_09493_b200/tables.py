"""Flatten a grammar (+ OpenCL.std) into the device table blob.

The blob is one little-endian ``uint32`` array the CUDA kernels index
directly (layout mirrored in ``csrc/skg_tables.cuh``).  It encodes every
lookup the reference codec path performs through Python dictionaries:

* opcode -> instruction record, first entry in file order for aliased
  opcodes (reference ``grammar.py:97-106``), with result/result-type flags
  (``grammar.py:74-80``), the slot list, the disassembler section code
  (``disasm.py:26-43, 253-267``) and the instruction's capability
  requirement (``validate.py:248-251``);
* operand kinds resolved by *first* kind of that name (``grammar.py:105``),
  with category, Id role (``ops.py:379-382``) and literal flavour
  (``ops.py:411-446``);
* enumerants in file order with parameters, plus a sorted (value, first
  index) table per ValueEnum kind for the "first enumerant with this value"
  lookup (``ops.py:385-390``), the first zero-valued name per BitEnum
  (``disasm.py:373-376``), and the merged same-value capability
  requirement (``validate.py:270-279``);
* capability closure bitsets: declaring a capability makes every name
  reachable over dependency + alias edges effective (``grammar.py:289-334``),
  precomputed once instead of per call;
* requirement records = bitmask of alternatives + the exact Python tuple
  repr used in diagnostics (``validate.py:286-290``);
* OpenCL.std number -> name (first by number, ``grammar.py:140-143``).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from . import grammar as _grammar

BLOB_MAGIC = 0x54474B53  # "SKGT"
BLOB_VERSION = 1
HEADER_WORDS = 64

CAT = {"Id": 0, "BitEnum": 1, "ValueEnum": 2, "Literal": 3, "Composite": 4}
ID_ROLE = {"IdResult": 1, "IdResultType": 2}          # else 0 = plain id
LIT = {"LiteralString": 1, "LiteralContextDependentNumber": 2, "LiteralInteger": 3,
       "LiteralExtInstInteger": 4, "LiteralSpecConstantOpInteger": 5}   # else 0
QUANT = {"": 0, "?": 1, "*": 2}

# special instruction codes (by name; csrc/skg_tables.cuh SP_*)
SPECIAL = {"OpTypeInt": 1, "OpTypeFloat": 2, "OpExtInstImport": 3, "OpName": 4, "OpSwitch": 5,
           "OpExtInst": 6, "OpFunction": 7, "OpFunctionEnd": 8, "OpCapability": 9,
           "OpMemoryModel": 10, "OpEntryPoint": 11, "OpLabel": 12, "OpFunctionParameter": 13,
           "OpVariable": 14, "OpUndef": 15, "OpLine": 16, "OpNoLine": 17}
SECTION_BY_NAME = {"OpCapability": 0, "OpExtension": 1, "OpExtInstImport": 2,
                   "OpMemoryModel": 3, "OpEntryPoint": 4, "OpExecutionMode": 5,
                   "OpExecutionModeId": 5}
SECTION_BY_CLASS = {"Debug": 6, "Annotation": 7, "Type-Declaration": 8, "Constant-Creation": 8}
SECTION_KEEP = 255
WIDTH_REQS = [("OpTypeInt", 8, ("Int8",)), ("OpTypeInt", 16, ("Int16",)),
              ("OpTypeInt", 64, ("Int64",)), ("OpTypeFloat", 16, ("Float16", "Float16Buffer")),
              ("OpTypeFloat", 64, ("Float64",))]

NONE32 = 0xFFFFFFFF


@dataclass
class PackedTables:
    blob: np.ndarray          # uint32
    n_inst: int
    n_kind: int
    n_enum: int
    cap_words: int


class _Strings:
    def __init__(self):
        self.buf = bytearray()
        self.index = {}

    def add(self, s: str):
        raw = s.encode("utf-8")
        if raw not in self.index:
            self.index[raw] = len(self.buf)
            self.buf += raw
        return self.index[raw], len(raw)


def _section(inst) -> int:
    if inst.name in SECTION_BY_NAME:
        return SECTION_BY_NAME[inst.name]
    if inst.class_attr in SECTION_BY_CLASS:
        return SECTION_BY_CLASS[inst.class_attr]
    if inst.name in ("OpVariable", "OpUndef"):
        return 8
    return SECTION_KEEP


def pack(spec=None, ext=None) -> PackedTables:
    spec = spec if spec is not None else _grammar.load_pinned()
    ext = ext if ext is not None else _grammar.load_pinned_extended()
    strings = _Strings()

    # kinds: first occurrence per name is the one every slot refers to
    kinds = list(spec.operand_kinds)
    kind_index = {}
    for i, k in enumerate(kinds):
        kind_index.setdefault(k.kind, i)

    slots: list[int] = []

    def slot_list(slot_objs, top_level=False) -> int:
        off = len(slots)
        for s in slot_objs:
            word = kind_index[s.kind] | (QUANT[s.quantifier] << 16)
            if top_level and s.kind == "LiteralSpecConstantOpInteger":
                word |= 1 << 24
            slots.append(word)
        return off

    # capability names: Capability enumerants (first per name), then extras
    cap_names: list[str] = []
    cap_id = {}

    def cap_index(name):
        if name not in cap_id:
            cap_id[name] = len(cap_names)
            cap_names.append(name)
        return cap_id[name]

    cap_kind = spec.kind("Capability") if spec.has_kind("Capability") else None
    for e in (cap_kind.enumerants or ()) if cap_kind else ():
        cap_index(e.name)
    requirements: list[tuple] = []
    req_index = {}

    def req(names) -> int:
        names = tuple(names)
        if not names:
            return NONE32
        if names not in req_index:
            for n in names:
                cap_index(n)
            req_index[names] = len(requirements)
            requirements.append(names)
        return req_index[names]

    # kinds whose operands can carry a capability requirement (an enumerant with required
    # capabilities, directly, through an enumerant parameter or a composite part): the
    # validator's operand-requirement walk is skipped for instructions without any
    kind_by_name = {}
    for k in kinds:
        kind_by_name.setdefault(k.kind, k)
    req_memo = {}

    def kind_has_req(name, stack=()):
        if name in req_memo:
            return req_memo[name]
        if name in stack:
            return False
        k = kind_by_name.get(name)
        r = False
        if k is not None:
            for e in k.enumerants or ():
                if e.required_capabilities or any(kind_has_req(p.kind, stack + (name,)) for p in e.parameters):
                    r = True
            for b in k.bases or ():
                r = r or kind_has_req(b, stack + (name,))
        req_memo[name] = r
        return r

    # instructions
    insts = list(spec.instructions)
    inst_rec = []
    for inst in insts:
        name_off, name_len = strings.add(inst.name)
        slot_off = slot_list(inst.operands, top_level=True)
        flags = (1 if inst.has_result else 0) | (2 if inst.has_result_type else 0)
        flags |= SPECIAL.get(inst.name, 0) << 8
        flags |= _section(inst) << 16
        flags2 = 1 if any(kind_has_req(sl.kind) for sl in inst.operands) else 0
        inst_rec.append([name_off, name_len | (len(inst.operands) << 16), slot_off, flags,
                         req(inst.required_capabilities), inst.opcode, flags2, 0])
    max_opcode = max((i.opcode for i in insts), default=0)
    opidx = np.full(max_opcode + 2, 0xFFFF, dtype=np.uint16)
    for i, inst in enumerate(insts):
        if opidx[inst.opcode] == 0xFFFF:
            opidx[inst.opcode] = i

    # enumerants + kinds
    enum_rec = []
    vsort = []
    kind_rec = []
    for k in kinds:
        cat = CAT[k.category]
        sub = ID_ROLE.get(k.kind, 0) if cat == 0 else (LIT.get(k.kind, 0) if cat == 3 else 0)
        enums = list(k.enumerants or ())
        enum_off = len(enum_rec)
        zero = NONE32
        for j, e in enumerate(enums):
            if e.value == 0 and zero == NONE32:
                zero = enum_off + j
        bases = list(k.bases or ()) if cat == 4 else []
        base_off = len(slots)
        for b in bases:
            slots.append(kind_index[b])
        vs_off = len(vsort)
        if cat == 2:
            first = {}
            for j, e in enumerate(enums):
                first.setdefault(e.value, enum_off + j)
            for v in sorted(first):
                vsort.append((v, first[v]))
        n_vs = len(vsort) - vs_off
        for e in enums:
            e_off, e_len = strings.add(e.name)
            p_off = slot_list(e.parameters)
            merged = []
            if cat == 2:
                for other in enums:
                    if other.value == e.value:
                        merged.extend(other.required_capabilities)
                merged = list(dict.fromkeys(merged))
            capname = cap_id.get(e.name, NONE32) if (cap_kind is not None and k is cap_kind) else NONE32
            enum_rec.append([e.value & 0xFFFFFFFF, e_off, e_len | (len(e.parameters) << 16), p_off,
                             req(e.required_capabilities), req(merged), capname, 0])
        kind_rec.append([cat | (sub << 8) | (len(bases) << 16), enum_off, len(enums), zero,
                         base_off, vs_off, n_vs, 0])

    width_req = [req(names) for _, _, names in WIDTH_REQS]
    linkage = cap_id.get("Linkage", NONE32)

    # capability closure over names (dependency + alias edges)
    n_cap = len(cap_names)
    cap_words = max(1, (n_cap + 63) // 64)
    closure = np.zeros((max(n_cap, 1), cap_words), dtype=np.uint64)
    edges = _grammar.capability_edges(spec) if cap_kind is not None else {}
    for name, ci in cap_id.items():
        if name not in edges:
            continue          # not a Capability enumerant: never effective
        seen, stack = set(), [name]
        while stack:
            n = stack.pop()
            if n in seen or n not in edges:
                continue
            seen.add(n)
            stack.extend(edges[n])
        for n in seen:
            j = cap_id[n]
            closure[ci, j // 64] |= np.uint64(1 << (j % 64))

    req_words = []
    for names in requirements:
        r_off, r_len = strings.add(repr(tuple(names)))
        bits = [0] * cap_words
        for n in names:
            j = cap_id[n]
            bits[j // 64] |= 1 << (j % 64)
        rec = [r_off, r_len]
        for b in bits:
            rec += [b & 0xFFFFFFFF, b >> 32]
        req_words.append(rec)

    # OpenCL.std (ext) number -> name
    ext_insts = list(ext.instructions) if ext is not None else []
    ext_max = max((i.opcode for i in ext_insts), default=-1)
    ext_tab = np.full((ext_max + 1, 2), NONE32, dtype=np.uint32)
    for i in ext_insts:
        if ext_tab[i.opcode, 0] == NONE32:
            off, ln = strings.add(i.name)
            ext_tab[i.opcode] = (off, ln)
    ocl_off, ocl_len = strings.add("OpenCL.std")
    idref = kind_index.get("IdRef", NONE32)

    # assemble the blob
    sections = []
    header = [0] * HEADER_WORDS

    def put(arr_u32) -> int:
        off = HEADER_WORDS + sum(len(s) for s in sections)
        sections.append(np.asarray(arr_u32, dtype=np.uint32).ravel())
        return off

    header[0], header[1] = BLOB_MAGIC, BLOB_VERSION
    header[2], header[3] = len(insts), put(inst_rec if inst_rec else np.zeros((0, 8)))
    header[4] = max_opcode
    ox = np.zeros((len(opidx) + 1) // 2 * 2, dtype=np.uint16)
    ox[: len(opidx)] = opidx
    header[5] = put(ox.view(np.uint32))
    header[6], header[7] = len(kinds), put(kind_rec)
    header[8], header[9] = len(enum_rec), put(enum_rec if enum_rec else np.zeros((0, 8)))
    header[10], header[11] = len(slots), put(slots if slots else [0])
    header[14], header[15] = len(requirements), put(req_words if req_words else [0])
    header[16], header[17] = n_cap, cap_words
    header[18] = put(closure.view(np.uint32).ravel())
    header[19] = put(np.array(vsort, dtype=np.uint32).ravel() if vsort else [0])
    header[20] = len(vsort)
    header[21], header[22] = ext_max, put(ext_tab.ravel() if ext_max >= 0 else [0])
    header[23] = idref
    for j, r in enumerate(width_req):
        header[24 + j] = r
    header[29] = linkage
    header[30], header[31] = ocl_off, ocl_len
    header[32] = 2 + 2 * cap_words   # requirement record stride (u32)
    _asm_sections(spec, ext, insts, kinds, kind_index, header, put, strings)
    sbuf = bytes(strings.buf) + b"\x00" * (-len(strings.buf) % 4)
    header[12] = put(np.frombuffer(sbuf, dtype=np.uint32) if sbuf else [0])
    header[13] = len(strings.buf)
    header[33] = kind_index.get("Capability", NONE32)
    blob = np.concatenate([np.asarray(header, dtype=np.uint32)] + sections)
    return PackedTables(blob=blob, n_inst=len(insts), n_kind=len(kinds), n_enum=len(enum_rec),
                        cap_words=cap_words)


def describe(t: PackedTables) -> str:
    return (f"{t.n_inst} instructions, {t.n_kind} kinds, {t.n_enum} enumerants, "
            f"{t.blob.nbytes} bytes")


__all__ = ["pack", "PackedTables", "describe", "struct"]


# -- assembler sections (asm.py / builder.py / ops.Encoder lookups) ---------------
# Route codes: bucket index 0..10 (builder._SECTIONS order), or
ROUTE_SCOPE, ROUTE_VARIABLE, ROUTE_KEYERROR = 11, 12, 13
SECTIONS = ("capabilities", "extensions", "ext_imports", "memory_model", "entry_points",
            "execution_modes", "debug_sources", "debug_names", "debug_processed",
            "annotations", "globals")                                    # builder.py:39-43
_MODE_BUCKET = {"OpCapability": 0, "OpMemoryModel": 3, "OpEntryPoint": 4,
                "OpExecutionMode": 5, "OpExecutionModeId": 5}          # builder.py:45-51
_DEBUG_BUCKET = {"OpName": 7, "OpMemberName": 7, "OpModuleProcessed": 8}   # builder.py:53-61
TERMINATORS = frozenset({"OpBranch", "OpBranchConditional", "OpSwitch", "OpKill", "OpReturn",
                         "OpReturnValue", "OpUnreachable", "OpTerminateInvocation",
                         "OpIgnoreIntersectionKHR", "OpTerminateRayKHR",
                         "OpEmitMeshTasksEXT"})                       # builder.py:31-35
AF_TERMINATOR, AF_BLOCK_FORBIDDEN, AF_CTXNUM = 1, 2, 4


def fnv1a(raw: bytes) -> int:
    h = 2166136261
    for b in raw:
        h = ((h ^ b) * 16777619) & 0xFFFFFFFF
    return h


def _route(inst) -> int:
    """builder.ModuleScope._route (builder.py:157-183) as a code."""
    name, cls = inst.name, inst.class_attr
    if name == "OpExtInst":
        return ROUTE_SCOPE
    if name == "OpUndef":
        return 10
    if name in ("OpLine", "OpNoLine"):
        return 6
    if name == "OpVariable":
        return ROUTE_VARIABLE
    if cls == "Mode-Setting":
        return _MODE_BUCKET.get(name, ROUTE_KEYERROR)
    if cls == "Extension":
        return 1 if name == "OpExtension" else 2
    if cls == "Debug":
        return _DEBUG_BUCKET.get(name, 6)
    if cls == "Annotation":
        return 9
    if cls in ("Type-Declaration", "Constant-Creation"):
        return 10
    if cls == "@exclude" and name.startswith("OpType"):
        return 10
    return ROUTE_SCOPE


def _hash_table(items, cap_min):
    """Open addressing (linear probe): items = [(hash, payload words...)]."""
    width = 1 + len(items[0][1]) if items else 2
    cap = 64
    while cap < 2 * len(items) + 8 or cap < cap_min:
        cap <<= 1
    tab = np.zeros((cap, width), dtype=np.uint32)
    used = np.zeros(cap, dtype=bool)
    for h, payload in items:
        s = h & (cap - 1)
        while used[s]:
            s = (s + 1) & (cap - 1)
        used[s] = True
        tab[s, 0] = h
        tab[s, 1:] = payload
    return tab, cap


def _unicode_tables():
    """Python str predicates the assembler relies on, as code-point tables:
    str.isprintable (repr), str.isspace / int()/float() whitespace, decimal
    digits (int(), float(), re ``\\d``) and str.isdigit-only digits."""
    printable = []
    prev, start = False, 0
    for c in range(0x110000):
        p = chr(c).isprintable()
        if p != prev:
            if p:
                start = c
            else:
                printable.append((start, c))
            prev = p
    if prev:
        printable.append((start, 0x110000))
    space = [c for c in range(0x110000) if chr(c).isspace()]
    dec_starts = [c for c in range(0x110000) if chr(c).isdecimal() and int(chr(c)) == 0]
    for s0 in dec_starts:
        assert all(chr(s0 + j).isdecimal() and int(chr(s0 + j)) == j for j in range(10))
    assert sum(chr(c).isdecimal() for c in range(0x110000)) == 10 * len(dec_starts)
    digit_only = [c for c in range(0x110000) if chr(c).isdigit() and not chr(c).isdecimal()]
    return printable, space, dec_starts, digit_only


def _asm_sections(spec, ext, insts, kinds, kind_index, header, put, strings):
    ctx_kind = "LiteralContextDependentNumber"
    info = []
    for inst in insts:
        rslot = next((j for j, s in enumerate(inst.operands) if s.kind == "IdResult"), 0xFF)
        flags = AF_TERMINATOR if inst.name in TERMINATORS else 0
        cls = inst.class_attr
        if cls in ("Mode-Setting", "Annotation", "Type-Declaration", "Constant-Creation") or \
                inst.name in ("OpExtension", "OpExtInstImport", "OpFunction",
                              "OpFunctionParameter", "OpFunctionEnd"):
            flags |= AF_BLOCK_FORBIDDEN
        if any(s.kind == ctx_kind for s in inst.operands):
            flags |= AF_CTXNUM
        c_off, c_len = strings.add(cls or "unclassified")
        info.append([min(rslot, 0xFF) | (_route(inst) << 8) | (flags << 16), c_off, c_len, 0])
    header[34] = put(info if info else [0])
    # opname -> instruction index (exact names, grammar.py:108-112)
    items = [(fnv1a(i.name.encode()), [j]) for j, i in enumerate(insts)]
    tab, cap = _hash_table(items, 1024)
    header[35], header[36] = put(tab), cap
    # (kind, enumerant name) -> first enumerant index by name (grammar.py:56-63)
    items, eoff = [], 0
    for ki, k in enumerate(kinds):
        seen = set()
        for j, e in enumerate(k.enumerants or ()):
            if e.name not in seen and kind_index.get(k.kind) == ki:
                seen.add(e.name)
                items.append(((fnv1a(e.name.encode()) ^ (ki * 0x9E3779B1)) & 0xFFFFFFFF,
                              [eoff + j, ki]))
        eoff += len(k.enumerants or ())
    tab, cap = _hash_table(items, 2048)
    header[37], header[38] = put(tab), cap
    # extended-instruction name -> number (last definition wins, grammar.py:139-141)
    by_name = {}
    for i in (ext.instructions if ext is not None else ()):
        by_name[i.name] = i.opcode
    items = []
    for nm, num in by_name.items():
        off, ln = strings.add(nm)
        items.append((fnv1a(nm.encode()), [num, off, ln]))
    tab, cap = _hash_table(items, 256)
    header[39], header[40] = put(tab), cap
    printable, space, dec_starts, digit_only = _unicode_tables_cached()
    header[41], header[42] = put(np.array(printable, dtype=np.uint32).ravel()), len(printable)
    header[43], header[44] = put(space), len(space)
    header[45], header[46] = put(dec_starts), len(dec_starts)
    header[47], header[48] = put(digit_only), len(digit_only)
    try:
        header[49] = spec.kind("StorageClass").enumerant("Function").value
    except Exception:  # noqa: BLE001 - custom grammar without StorageClass
        header[49] = NONE32
    knames = []
    for k in kinds:
        off, ln = strings.add(k.kind)
        knames += [off, ln]
    header[52] = put(knames if knames else [0])
    names = [i.name for i in insts]
    header[50] = names.index("OpLabel") if "OpLabel" in names else NONE32
    header[51] = names.index("OpFunctionEnd") if "OpFunctionEnd" in names else NONE32
    # the assembler's width scan tests the opname text (asm.py:215-230); with these it
    # compares instruction indices when the opname is in the grammar
    header[53] = names.index("OpTypeInt") if "OpTypeInt" in names else NONE32
    header[54] = names.index("OpTypeFloat") if "OpTypeFloat" in names else NONE32


_UNI = None


def _unicode_tables_cached():
    global _UNI
    if _UNI is None:
        _UNI = _unicode_tables()
    return _UNI
