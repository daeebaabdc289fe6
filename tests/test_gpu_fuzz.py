"""Seeded differential fuzzing of the CUDA path against the CPU oracle.

Binary mutants (the mutation kinds of tools/make_golden.py: random words, word
counts, opcodes, truncation, bit flips, header bounds) of the synthetic paper
families and of the reference-recorded golden modules go through
disassemble_batch (default, numeric, no_indent, and highlight+group+no_header
under strict), validate_batch and the fused disassemble_validate_batch, also
packed at unaligned offsets, some big-endian or not a whole number of words; text mutants (the kinds
of tests/test_gpu_asm.py) go through assemble_batch.  Every outcome -- text,
words, diagnostics, exception class and message -- must equal the oracle's.

Size: SKG_FUZZ_MODULES binary mutants (default 1200) and SKG_FUZZ_TEXTS text
mutants (default 400); the oracle runs in a process pool.
"""

import multiprocessing
import os
import random
import struct
from concurrent.futures import ProcessPoolExecutor

import pytest

pytestmark = pytest.mark.gpu

N_MOD = int(os.environ.get("SKG_FUZZ_MODULES", "1200"))
N_TXT = int(os.environ.get("SKG_FUZZ_TEXTS", "400"))
SEED = int(os.environ.get("SKG_FUZZ_SEED", "20261018"))


@pytest.fixture(scope="module")
def sk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2305_09493_b200 as pkg
    return pkg


def _outcome(fn):
    try:
        r = fn()
    except Exception as exc:  # noqa: BLE001
        return ("exc", type(exc).__name__, str(exc))
    if isinstance(r, list):
        r = [tuple(d) if not hasattr(d, "severity") else (d.severity, d.code, d.location, d.message) for d in r]
    return ("ok", r)


def _gpu(r):
    if isinstance(r, BaseException):
        return ("exc", type(r).__name__, str(r))
    if isinstance(r, list):
        return ("ok", [(d.severity, d.code, d.location, d.message) for d in r])
    return ("ok", r)


def _seed_module(rng):
    """a synthetic family module, or one of the reference-recorded golden modules (more
    instruction kinds: switches, ext-inst sets, debug strings, decorations ...)"""
    from golden_io import modules
    from synth.families import FAMILIES, build_module
    if rng.random() < 0.5:
        return build_module(rng.choice(FAMILIES), rng.randrange(1 << 20))
    gold = modules()
    return gold[rng.randrange(len(gold))]["bytes"]


def _mutants(n, seed):
    rng = random.Random(seed)
    out = []
    while len(out) < n:
        m = _seed_module(rng)
        if len(m) < 24 or len(m) % 4:
            continue
        w = list(struct.unpack(f"<{len(m) // 4}I", m))
        for _ in range(rng.randrange(1, 3)):
            kind = rng.randrange(6)
            pos = rng.randrange(5, len(w)) if len(w) > 5 else 0
            if kind == 0:
                w[pos] = rng.getrandbits(32)
            elif kind == 1:
                w[pos] = (w[pos] & 0xFFFF) | (rng.randrange(0, 8) << 16)
            elif kind == 2:
                w[pos] = (w[pos] & 0xFFFF0000) | rng.randrange(0, 400)
            elif kind == 3:
                w = w[: rng.randrange(5, len(w) + 1)]
            elif kind == 4:
                w[pos] ^= 1 << rng.randrange(32)
            else:
                w[3] = rng.randrange(0, 60)
        r = rng.random()
        if r < 0.1:      # big-endian stream (the decoder reads all words byte-swapped)
            out.append(struct.pack(f">{len(w)}I", *w))
        elif r < 0.15:   # not a whole number of words
            out.append(struct.pack(f"<{len(w)}I", *w) + bytes(rng.randrange(1, 4)))
        else:
            out.append(struct.pack(f"<{len(w)}I", *w))
    return out


ALL_OPTS = {"highlight": True, "group": True, "no_header": True}


def _oracle_binary(m):
    from oracle import disasm as odis, validate as oval
    from paper_2305_09493_b200.disasm import DisassemblerOptions
    return (_outcome(lambda: odis.disassemble(m)),
            _outcome(lambda: odis.disassemble(m, DisassemblerOptions(inline_names=False))),
            _outcome(lambda: oval.validate(m)),
            _outcome(lambda: odis.disassemble(m, DisassemblerOptions(**ALL_OPTS), strict=True)),
            _outcome(lambda: odis.disassemble(m, DisassemblerOptions(no_indent=True))))


def _oracle_text(t):
    from oracle import asm as oasm
    return _outcome(lambda: oasm.assemble(t).hex())


def _pool():
    # spawned workers: the parent holds a CUDA context
    return ProcessPoolExecutor(max_workers=min(32, os.cpu_count() or 4), mp_context=multiprocessing.get_context("spawn"))


def test_fuzz_binary_mutants(sk):
    mods = _mutants(N_MOD, SEED)
    with _pool() as ex:
        want = list(ex.map(_oracle_binary, mods, chunksize=16))
    got_d = sk.disassemble_batch(mods)
    got_n = sk.disassemble_batch(mods, sk.DisassemblerOptions(inline_names=False))
    got_v = sk.validate_batch(mods)
    fused = sk.disassemble_validate_batch(mods)
    got_a = sk.disassemble_batch(mods, sk.DisassemblerOptions(**ALL_OPTS), strict=True)
    # the same modules packed back to back with 0-3 gap bytes: unaligned module offsets
    import numpy as np
    from paper_2305_09493_b200 import _native
    rng = random.Random(SEED + 6)
    offs, buf = [], bytearray()
    for m in mods:
        buf += bytes(rng.randrange(4))
        offs.append(len(buf))
        buf += m
    packed = _native.DeviceBatch.from_host(np.frombuffer(bytes(buf + bytes(16)), dtype=np.uint8),
                                           np.array(offs, dtype=np.int64),
                                           np.array([len(m) for m in mods], dtype=np.int64))
    got_u = sk.disassemble_batch(packed)
    fused_u = sk.disassemble_validate_batch(packed)
    got_i = sk.disassemble_batch(mods, sk.DisassemblerOptions(no_indent=True))
    bad = []
    for k, (m, w) in enumerate(zip(mods, want)):
        if _gpu(got_d[k]) != w[0]:
            bad.append((k, "disasm"))
        if _gpu(got_n[k]) != w[1]:
            bad.append((k, "numeric"))
        if _gpu(got_v[k]) != w[2]:
            bad.append((k, "validate"))
        if _gpu(fused[k][0]) != w[0] or _gpu(fused[k][1]) != w[2]:
            bad.append((k, "fused"))
        if _gpu(got_a[k]) != w[3]:
            bad.append((k, "highlight+group+no_header strict"))
        if _gpu(got_i[k]) != w[4]:
            bad.append((k, "no_indent"))
        if _gpu(got_u[k]) != w[0] or _gpu(fused_u[k][0]) != w[0] or _gpu(fused_u[k][1]) != w[2]:
            bad.append((k, "unaligned offsets"))
    print(f"binary mutants: {len(mods)} modules x 9 outcomes, {len(bad)} mismatches")
    assert not bad, bad[:10]


def test_fuzz_text_mutants(sk):
    import importlib.util
    from pathlib import Path
    spec = importlib.util.spec_from_file_location("_asm_tests", Path(__file__).parent / "test_gpu_asm.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    rng = random.Random(SEED + 1)
    texts = []
    while len(texts) < N_TXT:
        t = sk.disassemble_batch([_seed_module(rng)], sk.DisassemblerOptions(inline_names=rng.random() < 0.7))[0]
        if not isinstance(t, str) or not t:
            continue
        for _ in range(rng.randrange(1, 4)):
            t = mod._mutate(t, rng)
        texts.append(t)
    with _pool() as ex:
        want = list(ex.map(_oracle_text, texts, chunksize=8))
    got = sk.assemble_batch(texts)
    bad = [k for k, (g, w) in enumerate(zip(got, want))
           if (_gpu(g.hex()) if isinstance(g, bytes) else _gpu(g)) != w]
    print(f"text mutants: {len(texts)} texts, {len(bad)} mismatches")
    assert not bad, bad[:10]


_WORDS = ["Inline", "DontInline", "Kernel", "Float64", "Aligned", "None", "Volatile|Aligned", "OpNop", "OpLabel",
          "CrossWorkgroup", "Function", "%", "%_", "%0", "%4294967295", "%name_0", "0x1p3", "1e400", "-0.0",
          "inf", "-nan", "0x7fffffff", "-2147483648", "4294967295", "18446744073709551616", "0o17", "0b1_0",
          "1__0", "00", "+1", "٣", "\"\"", "\"a\\\\b\"", "\"é\"", "=", ";", "OpExtInst", "sqrt", "exp", "12"]


def _mutate_more(t, rng):
    lines = t.split("\n")
    k = rng.randrange(6)
    i = rng.randrange(len(lines))
    if k == 0:                                   # CRLF / other separators on some lines
        sep = rng.choice(["\r\n", "\r", "\x0b", "\x0c", "\x1c", " ", "\x85"])
        return "".join(ln + (sep if rng.random() < 0.2 else "\n") for ln in lines)
    if k == 1:                                   # tabs / odd blanks as separators
        lines[i] = lines[i].replace(" ", rng.choice(["\t", "  ", " \t "]))
    elif k == 2:                                 # a token replaced by a grammar word / number form
        toks = lines[i].split(" ")
        toks[rng.randrange(len(toks))] = rng.choice(_WORDS)
        lines[i] = " ".join(toks)
    elif k == 3:                                 # a line duplicated
        lines.insert(i, lines[i])
    elif k == 4:                                 # trailing comment / blanks
        lines[i] = lines[i] + rng.choice([" ; x", "\t", "   ", ";\"", " ;;"])
    else:                                        # two tokens swapped
        toks = lines[i].split(" ")
        if len(toks) > 1:
            a, b = rng.randrange(len(toks)), rng.randrange(len(toks))
            toks[a], toks[b] = toks[b], toks[a]
            lines[i] = " ".join(toks)
    return "\n".join(lines)


def test_fuzz_text_mutants_more(sk):
    """text mutants with line separators other than LF, blanks, grammar words and number
    forms in random operand positions, duplicated lines and swapped tokens"""
    rng = random.Random(SEED + 2)
    texts = []
    while len(texts) < N_TXT:
        t = sk.disassemble_batch([_seed_module(rng)], sk.DisassemblerOptions(inline_names=rng.random() < 0.7))[0]
        if not isinstance(t, str) or not t:
            continue
        for _ in range(rng.randrange(1, 4)):
            t = _mutate_more(t, rng)
        texts.append(t)
    with _pool() as ex:
        want = list(ex.map(_oracle_text, texts, chunksize=8))
    got = sk.assemble_batch(texts)
    bad = [k for k, (g, w) in enumerate(zip(got, want))
           if (_gpu(g.hex()) if isinstance(g, bytes) else _gpu(g)) != w]
    print(f"text mutants (separators, words, numbers): {len(texts)} texts, {len(bad)} mismatches")
    assert not bad, bad[:10]


def test_fuzz_grid_wide_single_modules(sk):
    """binary mutants of mid-size modules (synth/huge.py) as single-module calls: the
    grid-wide kernels (skg_disasm_large / skg_validate_large) against the oracle"""
    from synth.huge import build_huge
    rng = random.Random(SEED + 3)
    n = max(8, N_TXT // 20)
    mods = []
    while len(mods) < n:
        m = build_huge(rng.randrange(4, 12), chain=rng.randrange(150, 250), seed=rng.randrange(1 << 20),
                       string_kib=(1,))
        w = list(struct.unpack(f"<{len(m) // 4}I", m))
        for _ in range(rng.randrange(0, 3)):
            if len(w) <= 5:      # truncated to the header by an earlier mutation
                break
            pos = rng.randrange(5, len(w))
            kind = rng.randrange(4)
            if kind == 0:
                w[pos] = rng.getrandbits(32)
            elif kind == 1:
                w[pos] = (w[pos] & 0xFFFF) | (rng.randrange(0, 8) << 16)
            elif kind == 2:
                w = w[: rng.randrange(5, len(w) + 1)]
            else:
                w[pos] ^= 1 << rng.randrange(32)
        mods.append(struct.pack(f"<{len(w)}I", *w))
    with _pool() as ex:
        want = list(ex.map(_oracle_binary, mods))
    bad = []
    for k, m in enumerate(mods):
        if _gpu(sk.disassemble_batch([m])[0]) != want[k][0]:
            bad.append((k, "disasm"))
        if _gpu(sk.validate_batch([m])[0]) != want[k][2]:
            bad.append((k, "validate"))
        t, v = sk.disassemble_validate_batch([m])[0]
        if _gpu(t) != want[k][0] or _gpu(v) != want[k][2]:
            bad.append((k, "fused"))
    from paper_2305_09493_b200 import _native
    big = sum(len(m) // 4 >= _native.SINGLE_LARGE_WORDS for m in mods)
    print(f"grid-wide single modules: {len(mods)} modules ({big} of {_native.SINGLE_LARGE_WORDS}+ words) "
          f"x 3 outcomes, {len(bad)} mismatches")
    assert 2 * big >= len(mods)     # most calls take the grid-wide kernels (truncations make some small)
    assert not bad, bad[:10]


_SPECS = {}


def _spec_named(which):
    """the pinned 1.2 grammar, or the custom GrammarSpec of tests/golden/grammars.json.gz
    (an opcode removed, one renamed, a capability dependency and a mask enumerant added)"""
    if which not in _SPECS:
        import gzip
        import json
        from pathlib import Path
        from paper_2305_09493_b200 import grammar
        if which == "1.2":
            _SPECS[which] = grammar.load_pinned("1.2")
        else:
            with gzip.open(Path(__file__).parent / "golden" / "grammars.json.gz", "rt", encoding="utf-8") as fh:
                _SPECS[which] = grammar.load_core_grammar(json.load(fh)["custom_grammar"])
    return _SPECS[which]


def _oracle_binary_spec(arg):
    which, m = arg
    from oracle import disasm as odis, validate as oval
    spec = _spec_named(which)
    return (_outcome(lambda: odis.disassemble(m, spec=spec)), _outcome(lambda: oval.validate(m, spec=spec)))


def _oracle_text_spec(arg):
    which, t = arg
    from oracle import asm as oasm
    return _outcome(lambda: oasm.assemble(t, spec=_spec_named(which)).hex())


@pytest.mark.parametrize("which", ["1.2", "custom"])
def test_fuzz_other_grammars(sk, which):
    """the same binary and text mutants under the pinned SPIR-V 1.2 grammar (empty
    instruction classes, fewer opcodes / enumerants) and a custom GrammarSpec:
    disassembly, validation, assembly"""
    spec = _spec_named(which)
    mods = _mutants(max(100, N_MOD // 4), SEED + 4)
    with _pool() as ex:
        want = list(ex.map(_oracle_binary_spec, [(which, m) for m in mods], chunksize=16))
    got_d = sk.disassemble_batch(mods, spec=spec)
    got_v = sk.validate_batch(mods, spec=spec)
    bad = [(k, "disasm") for k in range(len(mods)) if _gpu(got_d[k]) != want[k][0]]
    bad += [(k, "validate") for k in range(len(mods)) if _gpu(got_v[k]) != want[k][1]]
    rng = random.Random(SEED + 5)
    texts = []
    while len(texts) < max(50, N_TXT // 4):
        t = sk.disassemble_batch([_seed_module(rng)], spec=spec)[0]
        if not isinstance(t, str) or not t:
            continue
        t = _mutate_more(t, rng) if rng.random() < 0.5 else t
        texts.append(t)
    with _pool() as ex:
        want_t = list(ex.map(_oracle_text_spec, [(which, t) for t in texts], chunksize=8))
    got_t = sk.assemble_batch(texts, spec=spec)
    bad += [(k, "asm") for k, (g, w) in enumerate(zip(got_t, want_t))
            if (_gpu(g.hex()) if isinstance(g, bytes) else _gpu(g)) != w]
    print(f"{which} grammar: {len(mods)} binary mutants x 2, {len(texts)} texts, {len(bad)} mismatches")
    assert not bad, bad[:10]


def mod_text_mutate(t, rng):
    """tests/test_gpu_asm.py's text mutations"""
    import importlib.util
    from pathlib import Path
    global _ASM_TESTS
    if "_ASM_TESTS" not in globals():
        spec = importlib.util.spec_from_file_location("_asm_tests", Path(__file__).parent / "test_gpu_asm.py")
        _ASM_TESTS = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(_ASM_TESTS)
    return _ASM_TESTS._mutate(t, rng)


def _grammar_module(rng, spec):
    """a module of random instructions drawn from the whole grammar, operands built from
    each instruction's slot list (ids below a small bound, enumerants with their
    parameters, literals, strings, context-dependent numbers), then mutated or not"""
    insts = [d for d in spec.instructions if d.opcode < 0xFFFF]
    words = []
    for _ in range(rng.randrange(1, 12)):
        d = rng.choice(insts)
        ops = []

        def value(kind_name, depth=0):
            k = spec.kind(kind_name)
            if k.category == "Id":
                ops.append(rng.randrange(1, 40))
            elif k.category in ("ValueEnum", "BitEnum") and k.enumerants:
                if k.category == "BitEnum" and rng.random() < 0.5:
                    es = [e for e in k.enumerants if e.value and rng.random() < 0.2]
                    ops.append(sum({e.value for e in es}))
                    for e in es:
                        for p in e.parameters if depth < 2 else ():
                            value(getattr(p, "kind", p), depth + 1)
                else:
                    e = rng.choice(k.enumerants)
                    ops.append(e.value)
                    for p in e.parameters if depth < 2 else ():
                        value(getattr(p, "kind", p), depth + 1)
            elif k.category == "Composite":
                for b in k.bases or ():
                    value(b, depth + 1)
            elif k.kind == "LiteralString":
                s = "".join(rng.choice(["a", "b", "_", " ", "\u00e9", "\\", '"']) for _ in range(rng.randrange(0, 9))).encode()
                s += b"\0"
                s += b"\0" * (-len(s) % 4)
                ops.extend(struct.unpack(f"<{len(s) // 4}I", s))
            else:
                ops.append(rng.choice([0, 1, 7, 0xFFFFFFFF, 0x80000000, rng.getrandbits(32)]))
                if k.kind == "LiteralContextDependentNumber" and rng.random() < 0.3:
                    ops.append(rng.getrandbits(32))

        for slot in d.operands:
            q = getattr(slot, "quantifier", "")
            reps = 1 if q not in ("?", "*") else (rng.randrange(0, 3) if q == "*" else rng.randrange(2))
            for _ in range(reps):
                value(slot.kind)
        words += [((1 + len(ops)) << 16) | d.opcode, *ops]
    w = [0x07230203, 0x00010200, 0, rng.choice([40, 20, 1 << 20]), 0] + words
    return struct.pack(f"<{len(w)}I", *[x & 0xFFFFFFFF for x in w])


def test_fuzz_grammar_random_instructions(sk):
    """random instructions of every kind the grammar has (not only the ones the paper
    families and the corpus use): disassembly (default, numeric, highlight+group
    strict), validation; then their disassembly re-assembled"""
    spec = sk.load_pinned()
    rng = random.Random(SEED + 7)
    mods = [_grammar_module(rng, spec) for _ in range(max(200, N_MOD // 2))]
    with _pool() as ex:
        want = list(ex.map(_oracle_binary, mods, chunksize=16))
    got_d = sk.disassemble_batch(mods)
    got_n = sk.disassemble_batch(mods, sk.DisassemblerOptions(inline_names=False))
    got_v = sk.validate_batch(mods)
    got_a = sk.disassemble_batch(mods, sk.DisassemblerOptions(**ALL_OPTS), strict=True)
    bad = []
    for k, w in enumerate(want):
        for name, g, i in (("disasm", got_d, 0), ("numeric", got_n, 1), ("validate", got_v, 2), ("strict", got_a, 3)):
            if _gpu(g[k]) != w[i]:
                bad.append((k, name))
    texts = [g for g in got_d if isinstance(g, str) and g]
    with _pool() as ex:
        want_t = list(ex.map(_oracle_text, texts, chunksize=8))
    got_t = sk.assemble_batch(texts)
    bad += [(k, "asm") for k, (g, w) in enumerate(zip(got_t, want_t))
            if (_gpu(g.hex()) if isinstance(g, bytes) else _gpu(g)) != w]
    # the same texts mutated (assembler error paths over every opcode)
    mut = [_mutate_more(t, rng) if rng.random() < 0.5 else mod_text_mutate(t, rng) for t in texts]
    with _pool() as ex:
        want_m = list(ex.map(_oracle_text, mut, chunksize=8))
    got_m = sk.assemble_batch(mut)
    bad += [(k, "asm mutated") for k, (g, w) in enumerate(zip(got_m, want_m))
            if (_gpu(g.hex()) if isinstance(g, bytes) else _gpu(g)) != w]
    ok = sum(1 for w in want if w[0][0] == "ok")
    print(f"grammar-random modules: {len(mods)} ({ok} disassemble) x 4 outcomes + {len(texts)} texts "
          f"+ {len(mut)} mutated texts, {len(bad)} mismatches")
    assert not bad, bad[:10]
