"""CUDA assembler vs. the reference's golden vectors and the CPU oracle (needs a B200)."""

import random

import pytest

from golden_io import asm_texts, outcome, same

pytestmark = pytest.mark.gpu

ASM = asm_texts()


@pytest.fixture(scope="module")
def sk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2305_09493_b200 as sk
    return sk


def _outcome(r):
    if isinstance(r, BaseException):
        return {"exc": [type(r).__name__, str(r)]}
    return {"ok": r.hex()}


def test_asm_golden_batch(sk):
    got = sk.assemble_batch([r["text"] for r in ASM])
    bad = [(r["name"], _outcome(g), r["asm"]) for r, g in zip(ASM, got) if not same(_outcome(g), r["asm"])]
    assert not bad, bad[:5]


@pytest.mark.parametrize("rec", ASM[:30], ids=[r["name"] for r in ASM[:30]])
def test_assemble_module_single(sk, rec):
    got = outcome(lambda: sk.assemble_module(rec["text"]).hex())
    assert same(got, rec["asm"])


def test_asm_diagnostics_objects(sk):
    """AssemblyError carries AsmDiagnostic objects equal to the oracle's."""
    from oracle import asm as oasm
    texts = [r["text"] for r in ASM if "exc" in r["asm"] and r["asm"]["exc"][0] == "AssemblyError"]
    got = sk.assemble_batch(texts)
    for t, g in zip(texts, got):
        try:
            oasm.assemble(t)
        except Exception as exc:  # noqa: BLE001
            assert [(d.line, d.column, d.message) for d in g.diagnostics] == \
                [(d.line, d.column, d.message) for d in exc.diagnostics]


def _family_texts(n_per=6, numeric=False):
    from oracle import disasm as odis
    from synth.families import FAMILIES, build_module
    mods, texts = [], []
    for f in FAMILIES:
        for s in range(n_per):
            m = build_module(f, s)
            mods.append(m)
            texts.append(odis.disassemble(m, odis.Options(inline_names=not numeric)))
    return mods, texts


def test_roundtrip_families(sk):
    for numeric in (False, True):
        mods, texts = _family_texts(numeric=numeric)
        got = sk.assemble_batch(texts)
        bad = [i for i, (m, g) in enumerate(zip(mods, got)) if g != m]
        assert not bad, (numeric, bad[:5], got[bad[0]] if bad else None)


def _mutate(text, rng):
    lines = text.split("\n")
    k = rng.randrange(9)
    i = rng.randrange(len(lines))
    if k == 0:
        del lines[i]
    elif k == 1:
        j = rng.randrange(len(lines))
        lines[i], lines[j] = lines[j], lines[i]
    elif k == 2:
        lines.insert(i, rng.choice(["OpNop", "%zz = OpUndef %1", "OpReturn", "%q = OpLabel",
                                    "OpFunctionEnd", "OpCapability Shader", "OpName %zz \"a\\\"b\""]))
    elif k == 3:
        toks = lines[i].split(" ")
        toks[rng.randrange(len(toks))] = rng.choice(["0x1F", "-1", "1e5", "%", "%0", "\"s\"", "Foo|Bar",
                                                    "None|Inline", "4294967296", "0b101", "1_0", "٣",
                                                    "+7", "%٣", "nan", "-inf", "1.5"])
        lines[i] = " ".join(toks)
    elif k == 4:
        lines[i] = lines[i] + rng.choice([" extra", " 1", " %1", " ;comment", " \"unterminated"])
    elif k == 5:
        lines[i] = lines[i].replace("%", "%x", 1)
    elif k == 6:
        lines[i] = lines[i][: rng.randrange(len(lines[i]) + 1)]
    elif k == 7:
        lines.insert(i, rng.choice(["; Version: 1.5", "; Version: 2.0", "; Generator: 7; 9", "; Schema: 3",
                                    "; Version: 1.٣"]))
    else:
        lines[i] = lines[i].replace(" ", "\t", 1)
    return "\n".join(lines)


def test_asm_mutations_vs_oracle(sk):
    from oracle import asm as oasm
    rng = random.Random(1234)
    _, base = _family_texts(n_per=3)
    base += [r["text"] for r in ASM if "ok" in r["asm"]]
    texts = []
    for _ in range(1500):
        t = rng.choice(base)
        for _ in range(rng.randrange(1, 4)):
            t = _mutate(t, rng)
        texts.append(t)
    got = sk.assemble_batch(texts)
    bad = []
    for t, g in zip(texts, got):
        want = outcome(lambda: oasm.assemble(t).hex())
        if not same(_outcome(g), want):
            bad.append((t[:300], _outcome(g), want))
    assert not bad, (len(bad), bad[:3])


EDGE = [
    "",
    "\n\n",
    "OpCapability Kernel",
    "; Version: 1.0\nOpCapability Kernel\nOpMemoryModel Logical OpenCL\n",
    "%1 = OpTypeFloat 32\n%2 = OpConstant %1 1.5\n%3 = OpConstant %1 -0.0\n%4 = OpConstant %1 1e39\n",
    "%1 = OpTypeFloat 16\n%2 = OpConstant %1 65504\n%3 = OpConstant %1 65520\n",
    "%1 = OpTypeFloat 64\n%2 = OpConstant %1 0.1\n%3 = OpConstant %1 nan\n%4 = OpConstant %1 -inf\n",
    "%1 = OpTypeInt 64 1\n%2 = OpConstant %1 -9223372036854775808\n%3 = OpConstant %1 9223372036854775808\n",
    "%1 = OpTypeInt 8 1\n%2 = OpConstant %1 -128\n%3 = OpConstant %1 -1\n%4 = OpConstant %1 0x7f\n",
    "%1 = OpTypeInt 7 0\n%2 = OpConstant %1 1\n",
    "%1 = OpTypeFloat 8\n%2 = OpConstant %1 1\n",
    "%1 = OpTypeInt 32 0\n%2 = OpConstant %1 4294967296\n%3 = OpConstant %1 0x" + "f" * 40 + "\n",
    "OpCapability 17\nOpCapability 0x11\nOpCapability 99999\nOpCapability -1\n",
    "OpMemoryModel Physical64 OpenCL\nOpMemoryModel Logical GLSL450\n",
    "%1 = OpTypeVoid\n%2 = OpTypeFunction %1\n%3 = OpFunction %1 Inline|DontInline %2\n%4 = OpLabel\nOpReturn\nOpFunctionEnd\n",
    "%3 = OpFunction %1 Inline| Const |  %2\n",
    "%3 = OpFunction %1 0x3 %2\n%5 = OpFunction %1 0x100 %2\n",
    "%1 = OpTypeInt 32 0\n%2 = OpVariable %1 Function\n",
    "OpName %x \"\\x\\\"y\\\\\"\nOpName %y \"café 😀\"\nOpName %z \"a\x00b\"\n",
    "OpName %x \"\ud800\"\nOpName %y \"a\udc80\udc81b\"\n",
    "OpExtInstImport \"OpenCL.std\"\n%1 = OpExtInstImport \"OpenCL.std\"\n%2 = OpExtInst %3 %1 fabs %4\n",
    "%1 = OpSpecConstantOp %2 IAdd %3 %4\n%5 = OpSpecConstantOp %2 OpIAdd %3\n%6 = OpSpecConstantOp %2 Bogus\n",
    "%a = OpTypeInt 32 1\n%b = OpUndef %a\nOpSwitch %b %c -1 %d 5 %e\n",
    "%%% = OpNop\n%x = \n= = =\n%1 = OpTypeVoid extra\n",
    "﻿OpNop\r\nOpNop\x0bOpNop\x1cOpNop OpNop\x85OpNop\r",
    "OpCapability Kernel ; comment \"x\nOpCapability \"Kernel\"\n\"OpCapability\" Kernel\n",
    "OpDecorate %1 BuiltIn GlobalInvocationId\nOpDecorate %1 LinkageAttributes \"n\" Export\n",
    "OpLoad %1 %2 %3 Aligned 4\n%5 = OpLoad %1 %2 Aligned|Volatile 4\n%6 = OpLoad %1 %2 Aligned\n",
    "%²= OpNop\n",
    "%² = OpTypeVoid\n",
    "%0 = OpTypeVoid\n",
    "%4294967295 = OpTypeVoid\n",
    "%4294967294 = OpTypeVoid\n%a = OpTypeInt 32 0\n",
    "%05 = OpTypeVoid\n%5 = OpTypeBool\n",
    "; Version: 1.7\n",
    "; Version: 1." + "9" * 4301 + "\n",
    "  ; Generator: 99999; 4294967297\n; Schema: 4294967296\n; Version: ١.٣\nOpNop\n",
    "%1 = OpTypeInt 32 0\n%2 = OpConstant %1 " + "1" * 4400 + "\n",
    "%1 = OpTypeInt 32 0\n%2 = OpConstant %1 0x" + "1" * 4000 + "\n",
    "%f = OpFunction %v None %t\n%p = OpFunctionParameter %v\n%l = OpLabel\nOpReturn\nOpFunctionEnd\n"
    "%g = OpFunction %v None %t\nOpFunctionEnd\n%v = OpTypeVoid\n%t = OpTypeFunction %v\n",
    "%f = OpFunction %v None %t\n%l = OpLabel\n%p = OpFunctionParameter %v\nOpReturn\n",
    "%f = OpFunction %v None %t\n%l = OpLabel\n%x = OpVariable %p Function\nOpReturn\nOpFunctionEnd\n",
    "OpEntryPoint Kernel %f \"main\" %a %b\nOpExecutionMode %f LocalSize 1 2 3\nOpSource OpenCL_C 120\n",
    "OpLine %1 2 3\nOpNoLine\n%5 = OpUndef %1\nOpModuleProcessed \"x\"\nOpString \"s\"\n",
    # four-bytes-per-step scans: quotes / escapes / delimiters at every offset mod 4
    "".join(f"OpSourceExtension \"{'abcdefgh'[:k]}\\\"{'xyz'[:k % 4]}\\\\q\"\n" for k in range(9)),
    "".join(f"%{'s' * (k + 1)} = OpString \"{'s' * k}\"\nOpName %{'s' * (k + 1)} \"{'t' * (k + 2)}\";{'c' * k}\n"
            for k in range(9)),
    "".join(f"%{'a' * k}\t=\tOpTypeInt 32 0\n%{'b' * (k + 1)}\t=\tOpConstant\t%{'a' * k} {7 * k}\r\n"
            for k in range(1, 9)),
    "OpName %x \"abcdefghij\nOpName %y \"abcdefg\\\nOpName %z \"abc\"def\"\n",
]


def test_asm_edge_cases_vs_oracle(sk):
    from oracle import asm as oasm
    got = sk.assemble_batch(EDGE)
    bad = []
    for t, g in zip(EDGE, got):
        want = outcome(lambda: oasm.assemble(t).hex())
        if not same(_outcome(g), want):
            bad.append((t[:200], _outcome(g), want))
    assert not bad, bad


def test_roundtrip_session_pipelined(sk):
    """RoundTripSession: chunked 3-stream pipeline; text == oracle, binaries == inputs."""
    import numpy as np
    from oracle import disasm as odis
    from paper_2305_09493_b200.asm import RoundTripSession
    from synth.families import sample_batch
    b = sample_batch(3000, 300, 7)
    for chunks in (1, 5):
        sess = RoundTripSession(chunks=chunks)
        sess.stage(b.data, b.offsets, b.lengths)
        for _ in range(2):
            text, tspan, tst, binv, bspan, bst = sess.run_staged()
            assert (tst == 0).all() and (bst == 0).all()
            assert (bspan[:, 1] == b.lengths).all()
            for i in range(0, b.n, 37):
                m = b.module(i)
                assert binv[bspan[i, 0]:bspan[i, 0] + bspan[i, 1]].tobytes() == m
                t = text[tspan[i, 0]:tspan[i, 0] + tspan[i, 1]].tobytes().decode()
                if i % 111 == 0:
                    assert t == odis.disassemble(m)
        assert int(np.sum(tspan[:, 1])) <= len(text)


def test_asm_mixed_batch_with_large_text(sk, monkeypatch):
    """Small texts plus one large one: the per-warp slot is capped by the workspace
    budget and the large module is re-run alone with a larger slot."""
    from oracle import disasm as odis
    from paper_2305_09493_b200 import _native
    from synth.families import FAMILIES, build_module
    from synth.huge import build_huge
    monkeypatch.setattr(_native, "WS_BUDGET", 256 << 20)
    mods = [build_module(f, s) for f in FAMILIES for s in range(2)]
    mods.insert(3, build_huge(60, chain=150, seed=2))
    texts = [odis.disassemble(m) for m in mods]
    got = sk.assemble_batch(texts)
    for t, m, g in zip(texts, mods, got):
        if g != m:   # the huge module is not builder-canonical: compare with the oracle assembler
            from oracle import asm as oasm
            try:
                want = oasm.assemble(t)
            except Exception as exc:   # noqa: BLE001
                want = exc
            assert (type(g), str(g)) == (type(want), str(want)) if isinstance(want, Exception) else g == want


def test_roundtrip_session_fresh_batches_and_regrowth(sk, monkeypatch):
    """RoundTripSession.run on new batches with no sizing pass: different batches through
    one session; a text-arena bound too small (overflow: the chunk is re-run with grown
    arenas) and an assembler slot too small (internal status: re-run with slots for the
    real maximum) give the same results; host arenas that start too small grow
    mid-run keeping the chunks already copied."""
    from oracle import disasm as odis
    from paper_2305_09493_b200.asm import RoundTripSession
    from synth.families import sample_batch
    sess = RoundTripSession(chunks=4)
    for seed, factor in ((11, 6), (12, 6), (13, 1)):
        monkeypatch.setattr(RoundTripSession, "TEXT_FACTOR", factor)
        if seed == 12:   # host arenas grown chunk by chunk
            sess._buf.pop("h_text", None), sess._buf.pop("h_out", None)
            sess._ratio = (0.01, 0.01)
        b = sample_batch(2000 + 500 * (seed - 11), 200, seed)
        text, tspan, tst, binv, bspan, bst = sess.run(b.data, b.offsets, b.lengths)
        assert (tst == 0).all() and (bst == 0).all()
        assert (bspan[:, 1] == b.lengths).all()
        for i in range(0, b.n, 29):
            m = b.module(i)
            assert binv[bspan[i, 0]:bspan[i, 0] + bspan[i, 1]].tobytes() == m
            if i % 87 == 0:
                assert text[tspan[i, 0]:tspan[i, 0] + tspan[i, 1]].tobytes().decode() == odis.disassemble(m)


def test_composite_operand_string_literal(sk):
    """A string token where a composite operand (PairIdRefIdRef of OpPhi) starts is
    reported under the composite's kind; one in a later component under the
    component's kind (reference asm.py:293-295 via ops.py:160-164).  Found by the
    differential fuzz (tests/test_gpu_fuzz.py, seed 202)."""
    from oracle import asm as oasm
    from synth.families import build_module
    texts = []
    for fam in ("saxpy", "dft", "nbody"):
        lines = sk.disassemble_module(build_module(fam, 7)).split("\n")
        phi = next(i for i, ln in enumerate(lines) if " OpPhi " in ln)
        for col in (4, 5, 6):          # first pair: first / second component; second pair: first
            toks = lines[phi].split()
            toks[col] = '"s"'
            texts.append("\n".join(lines[:phi] + [" ".join(toks)] + lines[phi + 1:]))
    got = sk.assemble_batch(texts)
    for t, g in zip(texts, got):
        try:
            want = ("ok", oasm.assemble(t).hex())
        except Exception as exc:  # noqa: BLE001
            want = ("exc", type(exc).__name__, str(exc))
        have = ("ok", g.hex()) if isinstance(g, bytes) else ("exc", type(g).__name__, str(g))
        assert have == want
    assert "PairIdRefIdRef operand" in str(got[0]) and "IdRef operand" in str(got[1])
