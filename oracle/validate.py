"""Oracle: structural + capability validation (TEST INFRASTRUCTURE ONLY).

Restates ``spirvkit/validate.py:73-296``.  Returns a list of
``(severity, code, location, message)`` tuples (``location`` None for
module-level findings), ordered as ``validate_module`` orders them.
Non-codec exceptions raised by the operand walk (UnicodeDecodeError,
KeyError, ValueError) escape, as they do from the reference.
"""

from __future__ import annotations

from paper_2305_09493_b200 import grammar as _grammar
from paper_2305_09493_b200.errors import (CodecError, CorruptStreamError, NotSpirvError,
                                          TruncatedStreamError)

from .core import TypeMaps, decode_module, decode_operands, flat

WIDTH_CAPS = {("OpTypeInt", 8): ("Int8",), ("OpTypeInt", 16): ("Int16",),
              ("OpTypeInt", 64): ("Int64",), ("OpTypeFloat", 16): ("Float16", "Float16Buffer"),
              ("OpTypeFloat", 64): ("Float64",)}                     # validate.py:36-42


def _opdef(spec, opcode):
    return spec.instruction(opcode) if spec.has_instruction(opcode) else None


def declared_capabilities(spec, insts):
    """validate.py:101-112."""
    out = set()
    cap = spec.kind("Capability") if spec.has_kind("Capability") else None
    for opcode, words in insts:
        d = _opdef(spec, opcode)
        if d is not None and d.name == "OpCapability" and words and cap is not None:
            hit = next((e for e in cap.enumerants or () if e.value == words[0]), None)
            if hit is not None:
                out.add(hit.name)
    return out


def module_shape(spec, insts):
    """validate.py:115-136."""
    names = [(_opdef(spec, op).name if _opdef(spec, op) else None) for op, _ in insts]
    out = []
    if "OpFunction" not in names:
        out.append(("error", "MissingFunction", None, "module declares no function"))
    if "OpCapability" not in names:
        out.append(("error", "MissingCapability", None, "module declares no capability"))
    k = names.count("OpMemoryModel")
    if k == 0:
        out.append(("error", "MissingMemoryModel", None, "module has no memory model"))
    elif k > 1:
        out.append(("error", "MultipleMemoryModels", None,
                    f"module has {k} memory model instructions"))
    if "OpEntryPoint" not in names:
        eff = _grammar.transitive_capabilities(spec, declared_capabilities(spec, insts))
        sev = "warning" if "Linkage" in eff else "error"
        out.append((sev, "MissingEntryPoint", None, "module declares no entry point"))
    return out


def _unsatisfied(req, eff):
    if not req or any(c in eff for c in req):
        return ()
    return tuple(req)


def _operand_reqs(o):
    """validate.py:270-283."""
    if o.role == "value_enum" and o.enumerant is not None:
        merged = []
        for other in o.kind.enumerants or ():
            if other.value == o.enumerant.value:
                merged.extend(other.required_capabilities)
        req = tuple(dict.fromkeys(merged))
        return [req] if req else []
    if o.role == "bit_enum":
        return [e.required_capabilities for e in o.components if e.required_capabilities]
    return []


def validate(data: bytes, spec=None):
    """validate.py:73-94."""
    spec = spec if spec is not None else _grammar.load_pinned()
    try:
        header, insts = decode_module(bytes(data))
    except NotSpirvError as exc:
        return [("error", "NotSpirv", None, str(exc))]
    except TruncatedStreamError as exc:
        return [("error", "TruncatedStream", None, str(exc))]
    except CorruptStreamError as exc:
        return [("error", "CorruptStream", None, str(exc))]
    bound = header[3]
    maps = TypeMaps(spec, insts)
    diags = module_shape(spec, insts)
    located = []
    # _check_ids (validate.py:139-168)
    defined = {}
    for i, (opcode, words) in enumerate(insts):
        d = _opdef(spec, opcode)
        if d is None or not d.has_result:
            continue
        ri = 1 if d.has_result_type else 0
        if ri >= len(words):
            continue
        r = words[ri]
        if r in defined:
            located.append(("error", "DuplicateResultId", i, f"%{r} already defined at instruction {defined[r]}"))
        else:
            defined[r] = i
    decoded_all = []
    for i, (opcode, words) in enumerate(insts):
        d = _opdef(spec, opcode)
        if d is None:
            decoded_all.append(None)
            continue
        try:
            dec = decode_operands(spec, d, words, maps.resolve)
        except CodecError as exc:
            decoded_all.append(exc)
            continue
        decoded_all.append(dec)
        for o in flat(dec):
            if o.role in ("result", "result_type", "id") and o.value >= bound:
                located.append(("error", "BoundTooSmall", i,
                                f"%{o.value} is not below the header bound {bound}"))
    # _check_operand_layout (validate.py:207-220)
    for i, (opcode, words) in enumerate(insts):
        if _opdef(spec, opcode) is None:
            located.append(("warning", "UnknownOpcode", i, f"opcode {opcode} is not in the loaded grammar"))
        elif isinstance(decoded_all[i], CodecError):
            located.append(("error", "OperandMismatch", i, str(decoded_all[i])))
    # _closure_diagnostics (validate.py:237-267)
    eff = _grammar.transitive_capabilities(spec, declared_capabilities(spec, insts))
    for i, (opcode, words) in enumerate(insts):
        d = _opdef(spec, opcode)
        if d is None or d.name == "OpCapability":
            continue
        miss = _unsatisfied(d.required_capabilities, eff)
        if miss:
            located.append(("error", "MissingCapability", i, f"{d.name} requires one of {miss}"))
        dec = decoded_all[i]
        if isinstance(dec, CodecError):
            continue
        for o in flat(dec):
            for req in _operand_reqs(o):
                miss = _unsatisfied(req, eff)
                if miss:
                    located.append(("error", "MissingCapability", i,
                                    f"{d.name} operand requires one of {miss}"))
        req = ()
        if d.name in ("OpTypeInt", "OpTypeFloat") and len(words) >= 2:
            req = WIDTH_CAPS.get((d.name, words[1]), ())
        miss = _unsatisfied(req, eff)
        if miss:
            located.append(("error", "MissingCapability", i,
                            f"{d.name} with this width requires one of {miss}"))
    located.sort(key=lambda t: -1 if t[2] is None else t[2])
    return diags + located


def diagnostics_text(diags):
    """validate.py:52-54, 299-301."""
    return "\n".join(f"{s} {c} {'module' if loc is None else loc} {m}" for s, c, loc, m in diags)
