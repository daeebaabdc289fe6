"""Oracle: text -> binary assembly (TEST INFRASTRUCTURE ONLY).

Restates ``spirvkit/asm.py`` (tokenizer 51-90, symbol table 93-120,
``Assembler.assemble`` 133-180, header scan 184-206, width scans 215-245,
emission 249-362) together with the parts of ``builder.py`` the assembler
relies on (id allocation 108-128, routing 157-183, scopes 245-334,
serialization 187-242) and the encode half of ``ops.py`` (``Encoder``
104-271) / ``codec.py`` (132-168, 61-114).

Exceptions are the package's classes (``paper_2305_09493_b200.errors``) plus
the builtins that escape the reference (ValueError, OverflowError, KeyError).
"""

from __future__ import annotations

import re
import struct

from paper_2305_09493_b200 import grammar as _grammar
from paper_2305_09493_b200.errors import (AsmDiagnostic, AssemblyError, CodecError,
                                          IdExhaustedError, NotFoundError, ScopeError,
                                          SerializationError, SpirvKitError, SsaError,
                                          StructureError)

MAGIC = 0x07230203
MASK = 0xFFFFFFFF
MAX_ID = MASK - 1
HEADER_RE = (("version", re.compile(r";\s*Version:\s*(\d+)\.(\d+)\s*$")),
             ("generator", re.compile(r";\s*Generator:\s*(\d+);\s*(\d+)\s*$")),
             ("schema", re.compile(r";\s*Schema:\s*(\d+)\s*$")))       # asm.py:25-29
INT_TOKEN = re.compile(r"[+-]?(0[xX][0-9a-fA-F]+|\d+)$")                   # asm.py:31
SECTIONS = ("capabilities", "extensions", "ext_imports", "memory_model", "entry_points",
            "execution_modes", "debug_sources", "debug_names", "debug_processed",
            "annotations", "globals")                                    # builder.py:39-43
MODE_BUCKET = {"OpCapability": "capabilities", "OpMemoryModel": "memory_model",
               "OpEntryPoint": "entry_points", "OpExecutionMode": "execution_modes",
               "OpExecutionModeId": "execution_modes"}
DEBUG_BUCKET = {"OpSourceContinued": "debug_sources", "OpSource": "debug_sources",
                "OpSourceExtension": "debug_sources", "OpString": "debug_sources",
                "OpName": "debug_names", "OpMemberName": "debug_names",
                "OpModuleProcessed": "debug_processed"}
OVERRIDES = {"OpExtInst": "block", "OpUndef": "globals_or_block", "OpLine": "block_or_debug",
             "OpNoLine": "block_or_debug"}
TERMINATORS = frozenset({"OpBranch", "OpBranchConditional", "OpSwitch", "OpKill", "OpReturn",
                         "OpReturnValue", "OpUnreachable", "OpTerminateInvocation",
                         "OpIgnoreIntersectionKHR", "OpTerminateRayKHR", "OpEmitMeshTasksEXT"})


class Id(int):
    """builder.Id: repr (and therefore str/format) is '%N' (builder.py:73-77)."""

    def __repr__(self):
        return f"%{int(self)}"


class Tok:
    __slots__ = ("text", "column", "is_string")

    def __init__(self, text, column, is_string=False):
        self.text, self.column, self.is_string = text, column, is_string


def tokenize(line: str, lineno: int):
    """asm.py:51-90 -> (result, opname, operands, lineno) or None."""
    toks, i, n = [], 0, len(line)
    while i < n:
        ch = line[i]
        if ch in " \t\r\n":
            i += 1
            continue
        if ch == ";":
            break
        start = i
        if ch == '"':
            i += 1
            buf = []
            while i < n and line[i] != '"':
                if line[i] == "\\" and i + 1 < n:
                    i += 1
                buf.append(line[i])
                i += 1
            if i >= n:
                raise AssemblyError([AsmDiagnostic(lineno, start + 1, "unterminated string literal")])
            i += 1
            toks.append(Tok("".join(buf), start + 1, True))
            continue
        while i < n and line[i] not in ' \t\r\n;"':
            i += 1
        toks.append(Tok(line[start:i], start + 1))
    if not toks:
        return None
    result = None
    if len(toks) >= 3 and toks[0].text.startswith("%") and toks[1].text == "=":
        result, toks = toks[0], toks[2:]
    return (result, toks[0], toks[1:], lineno)


# -- builder restatement ------------------------------------------------------------
class Inst:
    __slots__ = ("opdef", "words", "result", "result_type", "refs")

    def __init__(self, opdef, words, result, result_type, refs):
        self.opdef, self.words, self.result = opdef, words, result
        self.result_type, self.refs = result_type, refs


class Function:
    def __init__(self, module, inst):
        self.module, self.inst = module, inst
        self.params, self.blocks, self.ended = [], [], False


class Block:
    def __init__(self, label_inst):
        self.label, self.insts = label_inst, []

    def terminated(self):
        return bool(self.insts) and self.insts[-1].opdef.name in TERMINATORS


class Module:
    def __init__(self, spec, major, minor, schema):
        if not (major == 1 and 0 <= minor <= 6):
            raise ValueError(f"unsupported SPIR-V version {major}.{minor}")   # builder.py:90-91
        self.spec, self.major, self.minor = spec, major, minor
        self.generator = (32 << 16) & MASK
        self.schema = schema
        self.buckets = {s: [] for s in SECTIONS}
        self.functions, self.registry = [], {}
        self.counter, self.reserved, self.labels = 0, set(), set()
        self.fn_storage = spec.kind("StorageClass").enumerant("Function").value

    def new_id(self):                              # builder.py:108-116
        v = self.counter + 1
        while v in self.reserved:
            v += 1
        if v > MAX_ID:
            raise IdExhaustedError("module id space exhausted")
        self.counter = v
        return Id(v)

    def reserve_id(self, v):                       # builder.py:118-123
        if not 0 < v <= MAX_ID:
            raise ValueError(f"id {v} out of range")
        self.reserved.add(v)
        return Id(v)

    def register(self, inst):                      # builder.py:130-136
        if inst.result is None:
            return
        if inst.result in self.registry:
            raise SsaError(f"%{inst.result} is defined by more than one instruction")
        self.registry[inst.result] = inst

    def route(self, inst):                         # builder.py:157-183
        name, cls = inst.opdef.name, inst.opdef.class_attr
        ov = OVERRIDES.get(name)
        if ov == "block":
            raise ScopeError(f"{name} belongs in a block scope")
        if ov in ("globals_or_block", "block_or_debug"):
            return "globals" if ov == "globals_or_block" else "debug_sources"
        if name == "OpVariable":
            if inst.words[2] == self.fn_storage:
                raise ScopeError("OpVariable with Function storage belongs in a block scope")
            return "globals"
        if cls == "Mode-Setting":
            return MODE_BUCKET[name]
        if cls == "Extension":
            return "extensions" if name == "OpExtension" else "ext_imports"
        if cls == "Debug":
            return DEBUG_BUCKET.get(name, "debug_sources")
        if cls == "Annotation":
            return "annotations"
        if cls in ("Type-Declaration", "Constant-Creation"):
            return "globals"
        if cls == "@exclude" and name.startswith("OpType"):
            return "globals"
        if cls == "Function":
            raise ScopeError(f"{name} belongs in a function scope")
        raise ScopeError(f"{name} ({cls or 'unclassified'}) is not a module-level instruction")

    def add(self, inst):                           # builder.py:140-147
        bucket = self.route(inst)
        if bucket == "memory_model" and self.buckets["memory_model"]:
            raise StructureError("module already has a memory model")
        self.register(inst)
        self.buckets[bucket].append(inst)

    def begin_function(self, inst):                # builder.py:149-155
        if inst.opdef.name != "OpFunction":
            raise ScopeError(f"begin_function expects OpFunction, got {inst.opdef.name}")
        self.register(inst)
        f = Function(self, inst)
        self.functions.append(f)
        return f

    def fn_add(self, f, inst):                     # builder.py:255-268
        name = inst.opdef.name
        if name == "OpFunctionParameter":
            if f.blocks:
                raise StructureError("function parameters must precede all blocks")
            self.register(inst)
            f.params.append(inst)
            return
        if name == "OpFunctionEnd":
            if f.ended:
                raise StructureError("function already ended")
            f.ended = True
            return
        raise ScopeError(f"{name} cannot be added at function scope")

    def begin_block(self, f, label):               # builder.py:270-281
        if label in self.labels:
            raise SsaError(f"%{label} is already used as a block label")
        if f.ended:
            raise StructureError("cannot begin a block after OpFunctionEnd")
        d = self.spec.instruction("OpLabel")
        inst = Inst(d, (label,), label, None, ())
        self.register(inst)
        self.labels.add(int(label))
        b = Block(inst)
        f.blocks.append(b)
        return b

    def block_add(self, b, inst):                  # builder.py:315-334
        name, cls = inst.opdef.name, inst.opdef.class_attr
        if b.terminated():
            raise StructureError("block already has its terminator")
        if name == "OpLabel":
            raise ScopeError("open a new block with begin_block instead of adding OpLabel")
        if name == "OpVariable":
            if inst.words[2] != self.fn_storage:
                raise ScopeError("only Function-storage OpVariable belongs in a block")
            if any(i.opdef.name != "OpVariable" for i in b.insts):
                raise StructureError("Function-storage OpVariable must open the first block")
        elif cls in ("Mode-Setting", "Annotation", "Type-Declaration", "Constant-Creation") \
                or name in ("OpExtension", "OpExtInstImport", "OpFunction", "OpFunctionParameter",
                            "OpFunctionEnd"):
            raise ScopeError(f"{name} ({cls or 'unclassified'}) is not a block instruction")
        self.register(inst)
        b.insts.append(inst)

    def to_bytes(self):                            # builder.py:187-242 + codec.py:61-101
        for f in self.functions:
            fname = f"function %{f.inst.result}"
            if not f.ended:
                raise StructureError(f"{fname} has no OpFunctionEnd")
            for b in f.blocks:
                if not b.terminated():
                    raise StructureError(f"block %{b.label.result} in {fname} has no terminator")
        stream = [i for s in SECTIONS for i in self.buckets[s]]
        end = self.spec.instruction("OpFunctionEnd")
        for f in [f for f in self.functions if not f.blocks] + [f for f in self.functions if f.blocks]:
            stream.append(f.inst)
            stream.extend(f.params)
            for b in f.blocks:
                stream.append(b.label)
                stream.extend(b.insts)
            stream.append(Inst(end, (), None, None, ()))
        defined = set(self.registry)
        for inst in stream:
            for r in inst.refs:
                if r not in defined:
                    raise SerializationError(f"%{r} is referenced by {inst.opdef.name} but never defined")
        bound = max(self.counter, max(self.reserved, default=0)) + 1
        words = [MAGIC, (self.major << 16) | (self.minor << 8), self.generator & MASK, bound,
                 self.schema & MASK]
        for inst in stream:
            count = 1 + len(inst.words)
            if count > 0xFFFF:
                raise CodecError(f"instruction length {count} words overflows the 16-bit count")
            words.append((count << 16) | inst.opdef.opcode)
            words.extend(w & MASK for w in inst.words)
        return struct.pack(f"<{len(words)}I", *words)


# -- encoding -----------------------------------------------------------------------
def encode_string(text):                           # codec.py:104-114
    data = text.encode("utf-8")
    if 0 in data:
        raise CodecError("string literal contains an embedded NUL byte")
    data += b"\x00"
    data += b"\x00" * (-len(data) % 4)
    return list(struct.unpack(f"<{len(data) // 4}I", data))


def encode_typed(value, width, signed=False, floating=False):   # codec.py:132-168
    if width not in (8, 16, 32, 64):
        raise CodecError(f"unsupported literal width {width}")
    if floating:
        fmt = {16: "<e", 32: "<f", 64: "<d"}.get(width)
        if fmt is None:
            raise CodecError(f"unsupported float width {width}")
        raw = struct.pack(fmt, value)                            # OverflowError escapes
        if width == 64:
            return list(struct.unpack("<2I", raw))
        return [struct.unpack("<I", raw.ljust(4, b"\x00"))[0]]
    value = int(value)
    if signed:
        lim = 1 << (width - 1)
        if not -lim <= value < lim:
            raise CodecError(f"value {value} does not fit a signed {width}-bit literal")
    elif not 0 <= value < (1 << width):
        raise CodecError(f"value {value} does not fit an unsigned {width}-bit literal")
    bits = value & ((1 << width) - 1)
    if width == 64:
        return [bits & MASK, bits >> 32]
    if signed and value < 0:
        bits |= (MASK << width) & MASK
    return [bits]


def bit_components(kind, mask):                    # ops.py:77-89
    if mask == 0:
        return []
    parts, covered = [], 0
    for e in kind.enumerants or ():
        if e.value and (mask & e.value) == e.value and (covered & e.value) != e.value:
            parts.append(e)
            covered |= e.value
    return parts if covered == mask else None


class _Typed:
    def __init__(self, value, width, signed=False, floating=False):
        self.value, self.width, self.signed, self.floating = value, width, signed, floating


class Encoder:
    """ops.Encoder.encode with the assembler's coerce (asm.py:286-332, ops.py:120-271)."""

    def __init__(self, spec, ext, symbols, opdef, literal_info):
        self.spec, self.ext, self.symbols, self.opdef = spec, ext, symbols, opdef
        self.info = literal_info
        self.words, self.refs = [], []
        self.result = self.result_type = None
        self.items, self.pos = [], 0

    def take(self, what):
        if self.pos >= len(self.items):
            raise ValueError(f"missing operand: expected {what}")
        self.pos += 1
        return self.items[self.pos - 1]

    def coerce(self, kind, raw):
        if not isinstance(raw, Tok):
            return raw
        if raw.is_string:
            if kind.kind != "LiteralString":
                raise ValueError(f"string literal given for a {kind.kind} operand")
            return raw.text
        text = raw.text
        if kind.category == "Composite":
            return raw
        if kind.category == "Id":
            return self.symbols.resolve(text)
        if kind.category in ("ValueEnum", "BitEnum"):
            return int(text, 0) if INT_TOKEN.match(text) else text
        if kind.kind == "LiteralContextDependentNumber":
            if self.info is None:
                raise ValueError("cannot resolve the literal width (unknown governing type)")
            width, signed, floating = self.info
            if floating:
                return _Typed(float(text), width, floating=True)
            return _Typed(int(text, 0), width, signed)
        if kind.kind == "LiteralInteger" and self.opdef.name == "OpSwitch" and self.info:
            width, signed, _ = self.info
            return _Typed(int(text, 0), width, signed)
        if kind.kind in ("LiteralExtInstInteger", "LiteralSpecConstantOpInteger"):
            return int(text, 0) if INT_TOKEN.match(text) else text
        value = int(text, 0)
        if value < 0:
            raise ValueError(f"{kind.kind} cannot be negative")
        return value

    def encode(self, inputs):
        self.items = list(inputs)
        d = self.opdef
        stopped = False
        for slot in d.operands:
            if slot.quantifier == "*":
                while self.pos < len(self.items):
                    self.one(slot.kind)
                break
            if slot.quantifier == "?":
                if self.pos >= len(self.items) or self.items[self.pos] is None:
                    if self.pos < len(self.items):
                        self.pos += 1
                    stopped = True
                    continue
                if stopped:
                    raise ValueError(f"{d.name}: optional operand {slot.kind} given after an omitted one")
            self.one(slot.kind)
            if slot.kind == "LiteralSpecConstantOpInteger":
                while self.pos < len(self.items):
                    self.value(self.spec.kind("IdRef"), self.take("id"))
        if self.pos < len(self.items):
            raise ValueError(f"{d.name}: {len(self.items) - self.pos} unexpected extra operand(s)")
        return Inst(d, tuple(self.words), self.result, self.result_type, tuple(self.refs))

    def one(self, kind_name):
        v = self.take(f"{self.opdef.name} operand of kind {kind_name}")
        self.value(self.spec.kind(kind_name), v)

    def param(self, kind_name):
        v = self.take(f"{self.opdef.name} enumerant parameter of kind {kind_name}")
        self.value(self.spec.kind(kind_name), v)

    def value(self, kind, value):
        value = self.coerce(kind, value)
        cat, name = kind.category, self.opdef.name
        if cat == "Id":
            if isinstance(value, bool) or not isinstance(value, int):
                raise ValueError(f"{name} ({kind.kind}) expects an id, got {value!r}")
            if not 0 < value <= MASK:
                raise ValueError(f"{name} ({kind.kind}): id {value} out of range")
            self.words.append(value)
            if kind.kind == "IdResult":
                self.result = value
            else:
                self.refs.append(value)
                if kind.kind == "IdResultType":
                    self.result_type = value
            return
        if cat == "ValueEnum":
            e = kind.enumerant(value if isinstance(value, str) else int(value))
            self.words.append(e.value)
            for p in e.parameters:
                self.param(p.kind)
            return
        if cat == "BitEnum":
            if isinstance(value, int) and not isinstance(value, bool):
                mask, parts = value, bit_components(kind, value) or []
            else:
                mask, parts = 0, []
                names = [x.strip() for x in value.split("|") if x.strip()] if isinstance(value, str) \
                    else [str(x) for x in value]
                for nm in names:
                    e = kind.enumerant(nm)
                    if e.value and (mask & e.value) != e.value:
                        parts.append(e)
                    mask |= e.value
                parts.sort(key=lambda e: (kind.enumerants or ()).index(e))
            if not 0 <= mask <= MASK:
                raise ValueError(f"{name}: {kind.kind} mask {mask:#x} out of range")
            self.words.append(mask)
            for e in parts:
                for p in e.parameters:
                    self.param(p.kind)
            return
        if cat == "Composite":
            bases = kind.bases or ()
            self.value(self.spec.kind(bases[0]), value)
            for b in bases[1:]:
                self.param(b)
            return
        kn = kind.kind
        if kn == "LiteralString":
            if not isinstance(value, str):
                raise ValueError(f"{name}: literal string expected, got {value!r}")
            self.words.extend(encode_string(value))
            return
        if kn == "LiteralContextDependentNumber":
            if not isinstance(value, _Typed):
                raise ValueError(f"{name}: context-dependent literal needs a TypedInt or TypedFloat")
            self.words.extend(encode_typed(value.value, value.width, value.signed, value.floating))
            return
        if kn == "LiteralInteger" and isinstance(value, _Typed):
            self.words.extend(encode_typed(value.value, value.width, value.signed))
            return
        if kn == "LiteralExtInstInteger" and isinstance(value, str):
            self.words.append(self.ext.instruction(value).opcode)
            return
        if kn == "LiteralSpecConstantOpInteger" and isinstance(value, str):
            self.words.append(self.spec.instruction(value if value.startswith("Op") else "Op" + value).opcode)
            return
        if isinstance(value, bool) or not isinstance(value, int):
            raise ValueError(f"{name}: {kn} expects an integer, got {value!r}")
        if not 0 <= value <= MASK:
            raise ValueError(f"{name}: {kn} value {value} out of range")
        self.words.append(value)


class Symbols:                                     # asm.py:93-120
    def __init__(self, module):
        self.module, self.by_name = module, {}

    def resolve(self, name):
        if not name.startswith("%") or len(name) == 1:
            raise ValueError(f"expected an id like %name, got {name!r}")
        if name in self.by_name:
            return self.by_name[name]
        body = name[1:]
        ident = self.module.reserve_id(int(body)) if body.isdigit() else self.module.new_id()
        self.by_name[name] = ident
        return ident


def create_module(text, spec):                     # asm.py:184-206
    version, gen, schema = (1, 2), None, 0
    for raw in text.splitlines():
        s = raw.strip()
        if s and not s.startswith(";"):
            break
        for key, pat in HEADER_RE:
            mt = pat.match(s)
            if not mt:
                continue
            if key == "version":
                version = (int(mt.group(1)), int(mt.group(2)))
            elif key == "generator":
                gen = (int(mt.group(1)) << 16) | int(mt.group(2))
            else:
                schema = int(mt.group(1))
    m = Module(spec, version[0], version[1], schema)
    if gen is not None:
        m.generator = gen
    return m


def assemble(text: str, spec=None, ext=None) -> bytes:
    """asm.py:133-180."""
    spec = spec if spec is not None else _grammar.load_pinned()
    ext = ext if ext is not None else _grammar.load_pinned_extended()
    diags, lines = [], []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        try:
            p = tokenize(raw, lineno)
        except AssemblyError as exc:
            diags.extend(exc.diagnostics)
            continue
        if p is not None:
            lines.append(p)
    module = create_module(text, spec)
    syms = Symbols(module)
    for result, _, operands, _ in lines:
        toks = ([result] if result is not None else []) + \
               [t for t in operands if not t.is_string and t.text.startswith("%")]
        for t in toks:
            if t.text[1:].isdigit():
                module.reserve_id(int(t.text[1:]))
    for result, _, _, ln in lines:
        if result is not None and not result.text[1:].isdigit():
            try:
                syms.resolve(result.text)
            except (ValueError, SpirvKitError) as exc:
                diags.append(AsmDiagnostic(ln, result.column, str(exc)))
    widths, vtypes = {}, {}
    for result, op, operands, _ in lines:
        if result is None or not operands:
            continue
        try:
            if op.text == "OpTypeInt":
                widths[result.text] = (int(operands[0].text, 0), int(operands[1].text, 0) == 1, False)
            elif op.text == "OpTypeFloat":
                widths[result.text] = (int(operands[0].text, 0), False, True)
        except (ValueError, IndexError):
            pass
    for result, op, operands, _ in lines:
        if result is None or not operands:
            continue
        try:
            d = spec.instruction(op.text)
        except NotFoundError:
            continue
        if d.has_result_type and operands[0].text.startswith("%"):
            vtypes[result.text] = operands[0].text
    fn = blk = None
    for p in lines:
        try:
            fn, blk = _emit(p, spec, ext, module, syms, widths, vtypes, fn, blk)
        except (SpirvKitError, ValueError, KeyError) as exc:
            diags.append(AsmDiagnostic(p[3], p[1].column, str(exc)))
    if diags:
        raise AssemblyError(diags)
    return module.to_bytes()


def _literal_info(d, operands, widths, vtypes):    # asm.py:351-362
    if d.name == "OpSwitch":
        if not operands:
            return None
        return widths.get(vtypes.get(operands[0].text, ""))
    if not any(s.kind == "LiteralContextDependentNumber" for s in d.operands):
        return None
    if d.has_result_type and operands:
        return widths.get(operands[0].text)
    return None


def _emit(p, spec, ext, module, syms, widths, vtypes, fn, blk):   # asm.py:249-284
    result, op, operands, _ = p
    name = op.text
    d = spec.instruction(name)
    if name == "OpLabel":
        if fn is None:
            raise ScopeError("OpLabel outside a function")
        if result is None:
            raise ValueError("OpLabel needs a result name")
        return fn, module.begin_block(fn, syms.resolve(result.text))
    inputs = list(operands)
    if d.has_result:
        if result is None:
            raise ValueError(f"{d.name} needs a result name")
        idx = next((i for i, s in enumerate(d.operands) if s.kind == "IdResult"), None)
        if idx is None:
            raise ValueError(f"{d.name} has no result slot")
        inputs.insert(idx, result)
    elif result is not None:
        raise ValueError(f"{d.name} does not produce a result")
    inst = Encoder(spec, ext, syms, d, _literal_info(d, operands, widths, vtypes)).encode(inputs)
    if name == "OpFunction":
        if fn is not None and not fn.ended:
            raise ScopeError("OpFunction before the previous OpFunctionEnd")
        return module.begin_function(inst), None
    if name in ("OpFunctionParameter", "OpFunctionEnd"):
        if fn is None:
            raise ScopeError(f"{name} outside a function")
        module.fn_add(fn, inst)
        return (None, None) if name == "OpFunctionEnd" else (fn, blk)
    try:
        module.add(inst)
        return fn, blk
    except ScopeError:
        pass
    if blk is None:
        raise ScopeError(f"{name} must appear inside a block")
    module.block_add(blk, inst)
    return fn, blk
