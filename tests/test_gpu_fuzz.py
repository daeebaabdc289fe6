"""Seeded differential fuzzing of the CUDA path against the CPU oracle.

Binary mutants (the mutation kinds of tools/make_golden.py: random words, word
counts, opcodes, truncation, bit flips, header bounds) of the synthetic paper
families and of the reference-recorded golden modules go through
disassemble_batch (default, numeric, no_indent, and highlight+group+no_header
under strict), validate_batch and the fused disassemble_validate_batch; text mutants (the kinds
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
    print(f"binary mutants: {len(mods)} modules x 6 outcomes, {len(bad)} mismatches")
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
