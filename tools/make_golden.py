"""Generate golden vectors by running the REFERENCE implementation.

Runs in the build container only (needs /root/reference).  Imports the
reference ``spirvkit`` from /root/reference/pkg/src and records, for a corpus
of binary modules and assembly texts, exactly what the reference returns or
raises:

* ``decode``:   header + (opcode, operand count) per instruction, or exception
* ``disasm``:   text for several option sets (+ strict), or exception
* ``validate``: ``diagnostics_text`` output (+ per-diagnostic tuples), or exception
* ``asm``:      words (hex) for assembly texts, or exception

Corpus: the reference test-suite corpus (``pkg/tests/corpus.py``: crafted +
seeded random builder modules), the paper-family synthetic modules
(``synth/families.py``), hand-made edge cases (bad magic, truncation, word
count 0, leftover/exhausted operands, UTF-8 errors, odd literal widths,
OpSwitch widths, name collisions, A.8 goldens ...), and seeded mutations of
valid modules.  Output: ``tests/golden/modules.jsonl.gz``,
``tests/golden/asm.jsonl.gz``.
"""

from __future__ import annotations

import base64
import gzip
import json
import random
import struct
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
OUT = ROOT / "tests" / "golden"

sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REF_TESTS))
sys.path.insert(1, str(ROOT))

import spirvkit as sk  # noqa: E402  (the reference)
import corpus  # noqa: E402  (the reference's own test corpus)

from synth.families import FAMILIES, build_module  # noqa: E402

MAGIC = 0x07230203
OPTION_SETS = {
    "default": {},
    "no_header": {"no_header": True},
    "numeric": {"inline_names": False},
    "highlight": {"highlight": True},
    "group_noindent": {"group": True, "no_indent": True},
    "all": {"highlight": True, "group": True, "no_header": True},
}


def words_to_bytes(words, big=False):
    return struct.pack(("<" if not big else ">") + f"{len(words)}I", *[w & 0xFFFFFFFF for w in words])


def inst(opcode, *ops):
    return [((len(ops) + 1) << 16) | opcode, *ops]


def string_words(raw: bytes):
    raw = raw + b"\x00"
    raw += b"\x00" * (-len(raw) % 4)
    return list(struct.unpack(f"<{len(raw) // 4}I", raw))


def module(insts, bound=64, minor=2, gen=0, schema=0):
    words = [MAGIC, (1 << 16) | (minor << 8), gen, bound, schema]
    for i in insts:
        words += i
    return words_to_bytes(words)


def outcome(fn):
    try:
        return {"ok": fn()}
    except Exception as exc:  # noqa: BLE001 - we record every class
        return {"exc": [type(exc).__name__, str(exc), repr(exc.args[0]) if exc.args else None]}


def edge_cases():
    spec = sk.load_pinned()
    op = lambda n: spec.instruction(n).opcode  # noqa: E731
    cap = lambda n: spec.kind("Capability").enumerant(n).value  # noqa: E731
    cases = {}
    cases["empty_header_only"] = module([], bound=1)
    cases["truncated_19"] = b"\x00" * 19
    cases["truncated_odd"] = b"\x03\x02\x23\x07" * 5 + b"\x00"
    cases["bad_magic"] = words_to_bytes([0xDEADBEEF, 0, 0, 1, 0])
    cases["elf"] = b"\x7fELF" + b"\x00" * 20
    cases["zero_wc"] = words_to_bytes([MAGIC, 0x00010200, 0, 1, 0, 0x00000011])
    cases["past_end"] = words_to_bytes([MAGIC, 0x00010200, 0, 1, 0, 0x00050011])
    base = [MAGIC, 0x00010200, 0x00200007, 9, 0] + inst(op("OpCapability"), cap("Kernel")) + inst(0)
    cases["big_endian"] = words_to_bytes(base, big=True)
    cases["little_endian"] = words_to_bytes(base)
    cases["unknown_opcode"] = module([inst(0xFFF0, 1, 2)], bound=5)
    cases["leftover"] = module([inst(op("OpCapability"), 6, 6)])
    cases["exhausted"] = module([inst(op("OpCapability"))])
    cases["no_nul"] = module([inst(op("OpTypeVoid"), 1), inst(op("OpName"), 1, 0x41414141)])
    cases["string_no_nul_opstring"] = module([inst(op("OpString"), 1, 0x41414141)])
    # A.8 goldens
    cases["a8_names"] = module([
        inst(op("OpTypeVoid"), 1), inst(op("OpTypeBool"), 2), inst(op("OpTypeInt"), 3, 32, 0),
        inst(op("OpName"), 1, *string_words(b"x_0")), inst(op("OpName"), 2, *string_words(b"x")),
        inst(op("OpName"), 3, *string_words(b"x")),
        inst(op("OpName"), 1, *string_words(b"ignored second name"))], bound=4)
    cases["a8_validate"] = module([
        inst(op("OpCapability"), cap("Kernel")), inst(op("OpTypeInt"), 5, 64, 0),
        inst(op("OpTypeInt"), 5, 64, 0), inst(0xFFF0), inst(op("OpCapability"))], bound=3)
    # UTF-8 errors in names / imports / plain strings
    bad = [b"\xff", b"\x80abc", b"ab\xc3", b"\xe2\x82", b"\xe0\x80\x80", b"\xed\xa0\x80",
           b"\xf0\x90\x80", b"\xf4\x90\x80\x80", b"\xf0\x28\x8c\x28", b"a\xe2\x28\xa1",
           b"\xc0\xaf", b"\xf8\x88\x80\x80\x80", b"ok\xe2\x82\xac\xf0\x9f", b"\xe1\x80",
           b"\xe1\x80\x41", b"\xf1\x80\x80\x41"]
    for k, raw in enumerate(bad):
        cases[f"utf8_name_{k}"] = module([inst(op("OpTypeVoid"), 1),
                                          inst(op("OpName"), 1, *string_words(raw))])
        cases[f"utf8_string_{k}"] = module([inst(op("OpString"), 1, *string_words(raw))])
        cases[f"utf8_import_{k}"] = module([inst(op("OpExtInstImport"), 1, *string_words(raw))])
    cases["utf8_ok_multibyte"] = module([
        inst(op("OpTypeVoid"), 1), inst(op("OpName"), 1, *string_words("ünï€𝄞 x".encode())),
        inst(op("OpString"), 2, *string_words('q"\\\n\t€'.encode()))], bound=3)
    # odd literal widths
    for width, signed in [(8, 0), (8, 1), (16, 1), (16, 0), (0, 0), (0, 1), (1, 1), (7, 1),
                          (33, 1), (63, 1), (64, 1), (64, 0), (128, 0), (31, 1)]:
        cases[f"int_width_{width}_{signed}"] = module([
            inst(op("OpTypeInt"), 1, width, signed),
            inst(op("OpConstant"), 1, 2, 0xFFFFFFF7, 0x80000001),
            inst(op("OpConstant"), 1, 3, 0x7F)], bound=4)
    for width in (8, 16, 32, 64, 128, 0):
        vals = [0x7FC00001, 0xFFFF3C00, 0x00000001, 0x80000000, 0x7F800000, 0xFF800000, 0x3DCCCCCD,
                0x00007BFF, 0x00008001, 0x0000FC00, 0x0000FE01]
        cases[f"float_width_{width}"] = module(
            [inst(op("OpTypeFloat"), 1, width)]
            + [inst(op("OpConstant"), 1, 2 + k, v, v ^ 0x12345678) for k, v in enumerate(vals)], bound=20)
    # OpSwitch with resolved widths
    for width, signed in [(32, 1), (64, 1), (64, 0), (16, 1), (8, 0)]:
        n = 2 if width == 64 else 1
        lits = [0xFFFFFFFF] * n
        cases[f"switch_{width}_{signed}"] = module([
            inst(op("OpTypeInt"), 1, width, signed),
            inst(op("OpConstant"), 1, 2, *([5] * n)),
            inst(op("OpSwitch"), 2, 3, *lits, 4, *([7] * n), 5)], bound=6)
    cases["switch_unresolved"] = module([inst(op("OpSwitch"), 9, 3, 0xFFFFFFFF, 4)], bound=10)
    # ext inst rendering
    cases["extinst_other_set"] = module([
        inst(op("OpExtInstImport"), 1, *string_words(b"GLSL.std.450")),
        inst(op("OpTypeFloat"), 2, 32), inst(op("OpExtInst"), 2, 3, 1, 23, 3),
        inst(op("OpExtInstImport"), 4, *string_words(b"OpenCL.std")),
        inst(op("OpExtInst"), 2, 5, 4, 23, 3), inst(op("OpExtInst"), 2, 6, 4, 999, 3)], bound=7)
    cases["spec_constant_op"] = module([
        inst(op("OpTypeInt"), 1, 32, 0), inst(op("OpSpecConstantOp"), 1, 2, op("OpIAdd"), 3, 4),
        inst(op("OpSpecConstantOp"), 1, 5, 0xFFF0, 3)], bound=6)
    # bit enums: zero, full cover, partial cover, params
    fc = spec.kind("FunctionControl")
    cases["bitenum"] = module([
        inst(op("OpTypeVoid"), 1), inst(op("OpTypeFunction"), 2, 1),
        inst(op("OpFunction"), 1, 3, 0, 2), inst(op("OpFunctionEnd")),
        inst(op("OpFunction"), 1, 4, 3, 2), inst(op("OpFunctionEnd")),
        inst(op("OpFunction"), 1, 5, 0x80000000, 2), inst(op("OpFunctionEnd")),
        inst(op("OpLoad"), 1, 6, 7, 0x3, 16), inst(op("OpLoad"), 1, 8, 7, 0),
        inst(op("OpLoad"), 1, 9, 7, 0x1000),
        inst(op("OpDecorate"), 1, 11, 4), inst(op("OpDecorate"), 1, 999999)], bound=10)
    del fc
    # enumerant with '*' parameter (exactly one decoded) and unknown enum values
    bank = spec.kind("Decoration").enumerant("BankBitsINTEL").value
    cases["enum_params"] = module([
        inst(op("OpTypeInt"), 1, 32, 0), inst(op("OpDecorate"), 1, bank, 1, 2),
        inst(op("OpDecorate"), 1, bank, 1), inst(op("OpDecorate"), 1, bank),
        inst(op("OpExecutionMode"), 2, 17, 1, 2, 3), inst(op("OpExecutionMode"), 2, 17, 1)], bound=3)
    # ids: zero, huge, undefined named, duplicates, demotion patterns
    cases["ids_weird"] = module([
        inst(op("OpTypeVoid"), 0), inst(op("OpTypeBool"), 0xFFFFFFF0), inst(op("OpTypeInt"), 7, 32, 0),
        inst(op("OpName"), 0, *string_words(b"zero")), inst(op("OpName"), 0xFFFFFFF0, *string_words(b"huge")),
        inst(op("OpName"), 7, *string_words(b"seven")), inst(op("OpName"), 99, *string_words(b"ghost")),
        inst(op("OpConstant"), 7, 3, 5), inst(op("OpName"), 3, *string_words(b"three"))], bound=8)
    cases["names_demotion"] = module([
        inst(op("OpTypeBool"), 2), inst(op("OpTypeVoid"), 1),
        inst(op("OpName"), 1, *string_words(b"first")), inst(op("OpName"), 2, *string_words(b"second"))], bound=3)
    cases["names_collide"] = module(
        [inst(op("OpTypeInt"), k, 32, 0) for k in range(1, 13)]
        + [inst(op("OpName"), k, *string_words(n)) for k, n in
           zip(range(1, 13), [b"x", b"x_0", b"x", b"x_1", b"x_0", b"x", b"x_0_0", b"", b"1", b"_1", b"a-b", b"a_b"])],
        bound=13)
    cases["names_serial_10"] = module(
        [inst(op("OpTypeInt"), k, 32, 0) for k in range(1, 16)]
        + [inst(op("OpName"), k, *string_words(b"v")) for k in range(1, 14)]
        + [inst(op("OpName"), 14, *string_words(b"v_10")), inst(op("OpName"), 15, *string_words(b"v_1"))],
        bound=16)
    return cases


def mutations(seeds, rng):
    out = {}
    for name, data in seeds:
        words = list(struct.unpack(f"<{len(data) // 4}I", data))
        for k in range(4):
            w = list(words)
            kind = rng.randrange(6)
            pos = rng.randrange(5, len(w))
            if kind == 0:
                w[pos] = rng.getrandbits(32)
            elif kind == 1:
                w[pos] = (w[pos] & 0xFFFF) | (rng.randrange(0, 8) << 16)
            elif kind == 2:
                w[pos] = (w[pos] & 0xFFFF0000) | rng.randrange(0, 400)
            elif kind == 3:
                w = w[: rng.randrange(5, len(w))]
            elif kind == 4:
                w[pos] ^= 1 << rng.randrange(32)
            else:
                w[3] = rng.randrange(0, 40)
            out[f"mut_{name}_{k}"] = words_to_bytes(w)
    return out


def corpus_modules():
    mods = {}
    for name, data in corpus.corpus_binaries(random_count=30).items():
        mods[f"ref_{name}"] = data
    for fam in FAMILIES:
        for s in range(6):
            mods[f"synth_{fam}_{s}"] = build_module(fam, s)
    return mods


def run_module(data):
    rec = {"data": base64.b64encode(data).decode()}

    def dec():
        h, insts = sk.decode_module(data)
        return [[h.major_version, h.minor_version, h.generator_magic, h.bound, h.schema],
                [[i.opcode, len(i.operands)] for i in insts]]

    rec["decode"] = outcome(dec)
    rec["disasm"] = {k: outcome(lambda o=o: sk.disassemble_module(data, sk.DisassemblerOptions(**o)))
                     for k, o in OPTION_SETS.items()}
    rec["disasm_strict"] = outcome(lambda: sk.disassemble_module(data, strict=True))
    rec["validate"] = outcome(lambda: [[d.severity, d.code, d.location, d.message]
                                       for d in sk.validate_module(data)])
    return rec


def asm_cases(mods):
    texts = {}
    for name, data in list(mods.items()):
        if not name.startswith(("ref_", "synth_")):
            continue
        for k in ("default", "numeric", "group_noindent"):
            try:
                texts[f"{name}:{k}"] = sk.disassemble_module(
                    data, sk.DisassemblerOptions(**OPTION_SETS[k]))
            except Exception:  # noqa: BLE001
                pass
    base = texts.get("ref_minimal_kernel:default", "")
    crafted = {
        "unterminated": 'OpCapability Kernel\nOpName %x "abc\n',
        "bad_opname": "OpCapability Kernel\nOpFrobnicate %1\n",
        "bad_version": "; Version: 2.0\nOpCapability Kernel\n",
        "id_zero": "OpCapability Kernel\n%0 = OpTypeVoid\n",
        "unicode_digit": "%² = OpTypeVoid\n",
        "leading_zero": "%1 = OpTypeInt 032 0\n",
        "float_overflow": "%1 = OpTypeFloat 32\n%2 = OpConstant %1 1e39\n",
        "half_overflow": "%1 = OpTypeFloat 16\n%2 = OpConstant %1 65520\n",
        "no_terminator": base.replace("OpReturn\n", ""),
        "undefined_ref": "OpCapability Kernel\n%2 = OpTypeFunction %3\n",
        "outside_block": "OpCapability Kernel\nOpNop\n",
        "label_outside": "%1 = OpLabel\n",
        "crlf": base.replace("\n", "\r\n"),
        "vt_split": base.replace("\n", "\x0b"),
        "empty": "",
        "comments_only": "; hi\n\n; there\n",
        "negative_literal": "%1 = OpTypeInt -32 0\n",
        "ext_by_number": ('OpCapability Kernel\n%1 = OpExtInstImport "OpenCL.std"\n'
                          "%2 = OpTypeFloat 32\n%3 = OpConstant %2 1.5\n"),
        "mask_names": "%1 = OpTypeVoid\n%2 = OpTypeFunction %1\n%3 = OpFunction %1 Inline|Pure %2\nOpFunctionEnd\n",
        "extra_operand": "OpCapability Kernel Shader\n",
        "missing_operand": "OpMemoryModel Physical64\n",
    }
    texts.update({f"crafted:{k}": v for k, v in crafted.items()})
    texts.update(asm_mutations(texts))
    recs = []
    for name, text in texts.items():
        res = outcome(lambda t=text: sk.assemble_module(t).hex())
        recs.append({"name": name, "text": text, "asm": res})
    return recs


JUNK = ["foo", "%", "007", "1e999", "-5", "0x", '"str"', "Inline|Bogus", "99999999999999999999",
        "-0x1F", "+7", "1_000", "0b101", "0o17", "%undefined_name", "%0", "%4294967295", "1.5",
        "-1", "nan", "inf", "2.5e-300", "0x1p3", "%٣", "None", "Const|Pure", "|Inline|", "4294967296"]


def asm_mutations(texts):
    rng = random.Random(99)
    out = {}
    bases = [(k, v) for k, v in texts.items() if k.endswith(":default")][:25]
    for name, text in bases:
        lines = text.split("\n")
        body = [i for i, ln in enumerate(lines) if ln.strip() and not ln.startswith(";")]
        for k in range(6):
            ls = list(lines)
            i = rng.choice(body)
            toks = ls[i].split(" ")
            kind = rng.randrange(7)
            if kind == 0 and len(toks) > 1:
                j = rng.randrange(1, len(toks))
                toks[j] = rng.choice(JUNK)
            elif kind == 1 and len(toks) > 2:
                del toks[rng.randrange(1, len(toks))]
            elif kind == 2:
                toks.append(rng.choice(JUNK))
            elif kind == 3:
                ls.insert(i, ls[rng.choice(body)])
            elif kind == 4:
                del ls[i]
                toks = None
            elif kind == 5:
                ls[i], ls[body[-1]] = ls[body[-1]], ls[i]
                toks = None
            else:
                ls.insert(i, rng.choice(["OpNop", "OpFunctionEnd", "%x = OpLabel", "OpReturn",
                                         "%q = OpTypeInt 12 1", "OpMemoryModel Logical GLSL450",
                                         '%s = OpString "a\\"b"', "OpCapability Bogus"]))
                toks = None
            if toks is not None:
                ls[i] = " ".join(toks)
            out[f"mut:{name}:{k}"] = "\n".join(ls)
    return out


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    rng = random.Random(20261017)
    mods = corpus_modules()
    seeds = [(n, d) for n, d in mods.items() if n.startswith("ref_")][:20]
    seeds += [(n, d) for n, d in mods.items() if n.startswith("synth_")][:10]
    mods.update(edge_cases())
    mods.update(mutations(seeds, rng))
    with gzip.open(OUT / "modules.jsonl.gz", "wt", encoding="utf-8") as fh:
        for name, data in mods.items():
            rec = run_module(data)
            rec["name"] = name
            fh.write(json.dumps(rec) + "\n")
    recs = asm_cases(mods)
    with gzip.open(OUT / "asm.jsonl.gz", "wt", encoding="utf-8") as fh:
        for rec in recs:
            fh.write(json.dumps(rec) + "\n")
    print(len(mods), "modules;", len(recs), "asm texts")


if __name__ == "__main__":
    main()
