"""Golden vectors for the fine-grained boundary functions,
recorded by running the REFERENCE (build container only, /root/reference):

* ``tokenize_line`` (asm.py:51-90) on every line of the assembler goldens'
  texts plus hand-made edge cases (escapes, trailing backslash, unterminated
  strings, non-ASCII columns, comments, odd whitespace, "%r =" shapes);
* ``encode_header`` / ``encode_instruction`` / ``encode_module`` /
  ``encode_string_literal`` / ``encode_context_dependent_literal``
  (codec.py:61-196) on seeded random and edge inputs, errors included;
* ``format_instruction`` (disasm.py:380-389) with RenderContexts (refs,
  type_info, value_type, import_sets; with and without the ext grammar);
* ``capability_dependency_graph`` (grammar.py:289-315) for both pinned grammars.

Output: tests/golden/boundary.json.gz.
"""

from __future__ import annotations

import gzip
import json
import random
import struct
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, str(ROOT))

import spirvkit as sk  # noqa: E402  (the reference)
from spirvkit.disasm import RenderContext  # noqa: E402

sys.path.insert(0, str(ROOT / "tests"))
from golden_io import asm_texts  # noqa: E402

OUT = ROOT / "tests" / "golden" / "boundary.json.gz"


def enc_val(v):
    """JSON-safe value: floats by repr (nan / inf / -0.0), big ints as strings."""
    if isinstance(v, bool):
        return {"b": v}
    if isinstance(v, float):
        return {"f": repr(v)}
    if isinstance(v, int):
        return {"i": str(v)}
    if v is None:
        return None
    return {"s": v}


def outcome(fn):
    try:
        return {"ok": fn()}
    except Exception as exc:  # noqa: BLE001 - every class is recorded
        rec = {"exc": [type(exc).__name__, str(exc)]}
        if isinstance(exc, sk.AssemblyError):
            rec["diags"] = [[d.line, d.column, d.message] for d in exc.diagnostics]
        return rec


def tok(t):
    return None if t is None else [t.text, t.column, t.is_string]


def tokenize_cases():
    lines = []
    for rec in asm_texts():
        lines += rec["text"].splitlines()[:60]
    lines = list(dict.fromkeys(lines))[:4000]
    lines += [
        "", "   ", "\t", "; comment only", "  ; indented comment", "OpNop", "OpNop ; trailing",
        '%a = OpString "x"', '%a = OpString "with \\"quote\\" and \\\\ back"', 'OpName %x "a;b"',
        'OpString "unterminated', 'OpString "trailing backslash\\', 'OpString "\\', '"',
        '"" "" ""', 'a"b"c', "a;b", "%x = = y", "%x =", "x = y", '"%x" = OpFoo', '%x "=" OpFoo',
        "%é = OpTypeVoid", '  %ü = OpString "ünï €" %ü', "éé \"€", "\t%a\t=\tOpNop\t%b",
        "%a = OpNop\r", "x\x0by", "x\x0cy", "OpDecorate %x LinkageAttributes \"n\" Export",
        '%s = OpString "tab\there"', "%1 = OpTypeInt 32 0", "  " * 40 + "%v = OpIAdd %t %a %b",
        '"\\x" "\\"" "\\\\\\\\"', "\U0001d11e \"\U0001d11e\" \U0001d11e", '%a = OpString "\\\U0001d11e"',
    ]
    out = []
    for k, ln in enumerate(lines):
        lineno = 1 + (k % 97)
        r = outcome(lambda: sk.tokenize_line(ln, lineno))
        if "ok" in r:
            ti = r["ok"]
            r = {"ok": None if ti is None else {"result": tok(ti.result), "opname": tok(ti.opname),
                                                "operands": [tok(t) for t in ti.operands], "line": ti.line}}
        out.append({"line": ln, "lineno": lineno, "out": r})
    return out


def codec_cases(rng):
    headers = [(1, 2, 32 << 16, 6, 0), (1, 0, 0, 1, 0), (1, 6, 0, 1, 0), (1, 2, 0, 0, 0), (1, 2, 0, 2 ** 32, 0),
               (1, 2, 0, -1, 0), (256, 0, 0, 5, 0), (1, -1, 0, 5, 0), (1, 2, -1, 5, -7), (1, 2, 2 ** 40 + 3, 5, 2 ** 33),
               (255, 255, 2 ** 32 - 1, 2 ** 32 - 1, 2 ** 32 - 1), (1, 2, 0, 2 ** 70, 0), (2 ** 70, 0, 0, 5, 0)]
    for _ in range(40):
        headers.append((rng.randrange(0, 300), rng.randrange(-2, 300), rng.randrange(-2 ** 33, 2 ** 33),
                        rng.choice([0, 1, rng.randrange(1, 2 ** 32), 2 ** 32, rng.randrange(2 ** 32, 2 ** 40)]),
                        rng.randrange(0, 2 ** 34)))
    hdr = [{"h": [str(x) for x in h], "out": outcome(lambda: sk.encode_header(sk.ModuleHeader(*h)))}
           for h in headers]
    insts = [(17, (6,)), (0, ()), (1, tuple(range(0xFFFE))), (1, tuple(range(0xFFFF))), (0x10000, ()), (-1, (1,)),
             (0xFFFF, (2 ** 32 + 5, -1, 2 ** 64 - 1, -(2 ** 40))), (5, (0,) * 3), (2 ** 70, ())]
    for _ in range(60):
        insts.append((rng.randrange(0, 0x10000), tuple(rng.randrange(-2 ** 33, 2 ** 34)
                                                         for _ in range(rng.randrange(0, 9)))))
    def ops_rec(w):   # long operand runs are range(n): stored by length
        return {"range": len(w)} if len(w) > 1000 and list(w) == list(range(len(w))) else [str(x) for x in w]
    ins = []
    for o, w in insts:
        r = outcome(lambda: sk.encode_instruction(sk.RawInstruction(o, w)))
        if "ok" in r and len(r["ok"]) > 1000:
            r = {"ok_sha": __import__("hashlib").sha256(struct.pack(f"<{len(r['ok'])}I", *r["ok"])).hexdigest()}
        ins.append({"op": str(o), "ops": ops_rec(w), "out": r})
    mods = []
    for k in range(40):
        h = sk.ModuleHeader(1, rng.randrange(0, 7), rng.randrange(0, 2 ** 32), rng.randrange(1, 2 ** 32), 0)
        if k % 9 == 3:
            h = sk.ModuleHeader(1, 2, 0, 0, 0)
        body = [sk.RawInstruction(rng.randrange(0, 0x10000), tuple(rng.randrange(0, 2 ** 32)
                                                                   for _ in range(rng.randrange(0, 8))))
                for _ in range(rng.randrange(0, 30))]
        if k % 7 == 5 and body:
            body[len(body) // 2] = sk.RawInstruction(0x12345, (1,))
        if k % 11 == 4 and body:
            body[-1] = sk.RawInstruction(3, tuple(range(0x10000)))
        r = outcome(lambda: sk.encode_module(h, body).hex())
        mods.append({"h": [h.major_version, h.minor_version, h.generator_magic, h.bound, h.schema],
                     "insts": [[i.opcode, ops_rec(i.operands)] for i in body], "out": r})
    strs = ["", "a", "ab", "abc", "abcd", "abcde", "ünïcödé", "x" * 100, "OpenCL.std", "a\x00b", "\x00",
            "q\"uote\\back", "\U0001d11e" * 7, "white  space"]
    strs += ["".join(chr(rng.choice([0x41, 0x7A, 0xE9, 0x20AC, 0x1D11E, 0x30])) for _ in range(rng.randrange(0, 40)))
             for _ in range(30)]
    st = [{"s": s, "out": outcome(lambda: sk.encode_string_literal(s))} for s in strs]
    lits = []
    vals_i = [0, 1, -1, 42, 127, 128, -128, -129, 255, 256, 32767, 32768, -32768, -32769, 65535, 65536,
              2 ** 31 - 1, 2 ** 31, -(2 ** 31), -(2 ** 31) - 1, 2 ** 32 - 1, 2 ** 32, 2 ** 63 - 1, 2 ** 63,
              -(2 ** 63), -(2 ** 63) - 1, 2 ** 64 - 1, 2 ** 64, -(2 ** 64), 10 ** 30, 1.7, -2.5, True]
    vals_f = [0.0, -0.0, 1.0, -1.5, 3.4028234663852886e38, 3.4028235677973366e38, 3.402823669209385e38, 1e39,
              65504.0, 65519.99, 65520.0, 1e-8, 5e-324, float("inf"), float("-inf"), float("nan"), 1, 2 ** 1100,
              True, 0.1, 1e300]
    widths = [8, 16, 32, 64, None, 0, 12, 128, -8]
    for w in widths:
        for v in vals_i:
            for signed in (False, True):
                lits.append((v, w, signed, False))
        for v in vals_f:
            lits.append((v, w, False, True))
    for _ in range(200):
        w = rng.choice([8, 16, 32, 64])
        if rng.random() < 0.5:
            lits.append((rng.randrange(-2 ** 65, 2 ** 65) >> rng.randrange(0, 66), w, rng.random() < 0.5, False))
        else:
            lits.append((struct.unpack("<d", struct.pack("<Q", rng.getrandbits(64)))[0], w, False, True))
    lit = [{"v": enc_val(v), "w": w, "signed": s, "floating": f,
            "out": outcome(lambda: sk.encode_context_dependent_literal(v, w, signed=s, floating=f))}
           for v, w, s, f in lits]
    return {"encode_header": hdr, "encode_instruction": ins, "encode_module": mods, "encode_string": st,
            "encode_ctx": lit}


def format_cases(rng):
    g16, ext = sk.load_pinned(), sk.load_pinned_extended()
    op = lambda n: g16.instruction(n).opcode  # noqa: E731
    w = lambda s: list(struct.unpack(f"<{(len(s) + 4) // 4}I", s + b"\0" * (4 - len(s) % 4)))  # noqa: E731
    insts = [(op("OpCapability"), (6,)), (0, ()), (op("OpFunction"), (1, 2, 3, 3)), (op("OpCapability"), (6, 7)),
             (op("OpIAdd"), (3, 10, 11, 12)), (op("OpConstant"), (3, 10, 0xFFFFFFFF)),
             (op("OpConstant"), (4, 11, 0, 0x3FF00000)), (op("OpConstant"), (5, 12, 0x3F800000)),
             (op("OpConstant"), (9, 12, 5)), (op("OpSwitch"), (20, 21, 7, 22, 0xFFFFFFFF, 23)),
             (op("OpSwitch"), (24, 21, 1, 0, 22)), (op("OpExtInst"), (3, 30, 31, 23, 10)),
             (op("OpExtInst"), (3, 30, 32, 23, 10)), (op("OpName"), (10, *w(b"nm"))), (op("OpLoad"), (3, 40, 41)),
             (op("OpStore"), (41, 40, 2, 4)), (op("OpDecorate"), (10, 44)), (op("OpSpecConstantOp"), (3, 50, 128, 10, 11))]
    ctxs = [None, RenderContext(),
            RenderContext(refs={10: "%sum", 3: "%int", 40: "%v", 41: "%ptr", 12: "", 1: "x", 2: "%%"}),
            RenderContext(type_info={3: (32, False, False), 4: (64, False, True), 5: (32, True, True),
                                     9: (16, True, False), 6: (64, True, False)},
                          value_type={20: 3, 24: 6}),
            RenderContext(refs={30: "%ocl", 31: "%set2", 23: "%f"}, type_info={3: (32, True, False)},
                          import_sets={31: "OpenCL.std", 32: "GLSL.std.450"}),
            RenderContext(type_info={3: (8, True, False), 9: (128, False, False)}, value_type={20: 99}),
            RenderContext(refs={k: f"%n{k}_é" for k in range(60)}, type_info={3: (64, True, False)},
                          value_type={20: 3, 24: 3}, import_sets={31: "OpenCL.std"})]
    out = []
    for o, ops in insts:
        for ci, c in enumerate(ctxs):
            for e in (None, ext):
                r = outcome(lambda: sk.format_instruction(g16, sk.RawInstruction(o, ops), c, e))
                rc = None if c is None else {"refs": {str(k): v for k, v in c.refs.items()},
                                             "type_info": {str(k): list(v) for k, v in c.type_info.items()},
                                             "value_type": {str(k): v for k, v in c.value_type.items()},
                                             "import_sets": {str(k): v for k, v in c.import_sets.items()}}
                out.append({"op": o, "ops": list(ops), "ctx": rc, "ext": e is not None, "out": r})
    return out


def dependency_cases():
    out = {}
    for v in ("unified1", "1.2"):
        rep = sk.capability_dependency_graph(sk.load_pinned(v))
        out[v] = {"nodes": list(rep.nodes), "edges": {k: list(x) for k, x in rep.edges.items()},
                  "cycles": [list(c) for c in rep.cycles]}
    return out


def main():
    rng = random.Random(20261017)
    rec = {"tokenize": tokenize_cases(), **codec_cases(rng), "format_instruction": format_cases(rng),
           "dependency": dependency_cases()}
    with gzip.open(OUT, "wt", encoding="utf-8") as fh:
        json.dump(rec, fh)
    print({k: len(v) for k, v in rec.items()})


if __name__ == "__main__":
    main()
