"""CUDA path vs. the reference's golden vectors and the CPU oracle (needs a B200)."""

import random
import struct

import numpy as np
import pytest

from golden_io import OPTION_SETS, modules, outcome, same

pytestmark = pytest.mark.gpu

CASES = modules()


@pytest.fixture(scope="module")
def sk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2305_09493_b200 as sk
    return sk


def _as_outcome(r):
    if isinstance(r, BaseException):
        return {"exc": [type(r).__name__, str(r)]}
    return {"ok": r}


def test_disasm_golden_batch_all_options(sk):
    datas = [r["bytes"] for r in CASES]
    for key, opts in OPTION_SETS.items():
        got = sk.disassemble_batch(datas, sk.DisassemblerOptions(**opts))
        bad = [r["name"] for r, g in zip(CASES, got) if not same(_as_outcome(g), r["disasm"][key])]
        assert not bad, f"{key}: {bad[:10]}"
    got = sk.disassemble_batch(datas, strict=True)
    bad = [r["name"] for r, g in zip(CASES, got) if not same(_as_outcome(g), r["disasm_strict"])]
    assert not bad, bad[:10]


def test_golden_grid_wide_single_module_path(sk, monkeypatch):
    """Every reference-recorded golden module, one call per module, through the
    grid-wide kernels (skg_disasm_large / skg_validate_large) that single-module
    calls of _native.SINGLE_LARGE_WORDS words and up take (forced here for all):
    all six option sets, strict, and validation."""
    from paper_2305_09493_b200 import _native
    monkeypatch.setattr(_native, "SINGLE_LARGE_WORDS", 1)
    bad = []
    for r in CASES:
        m = r["bytes"]
        for key, opts in OPTION_SETS.items():
            if not same(_as_outcome(sk.disassemble_batch([m], sk.DisassemblerOptions(**opts))[0]), r["disasm"][key]):
                bad.append((r["name"], key))
        if not same(_as_outcome(sk.disassemble_batch([m], strict=True)[0]), r["disasm_strict"]):
            bad.append((r["name"], "strict"))
        o = _as_outcome(sk.validate_batch([m])[0])
        if "ok" in o:
            o = {"ok": [[d.severity, d.code, d.location, d.message] for d in o["ok"]]}
        if not same(o, r["validate"]):
            bad.append((r["name"], "validate"))
    assert not bad, bad[:10]


@pytest.mark.parametrize("rec", CASES[:40], ids=[r["name"] for r in CASES[:40]])
def test_disassemble_module_single(sk, rec):
    got = outcome(lambda: sk.disassemble_module(rec["bytes"]))
    assert same(got, rec["disasm"]["default"])


def test_validate_golden_batch(sk):
    datas = [r["bytes"] for r in CASES]
    got = sk.validate_batch(datas)
    bad = []
    for r, g in zip(CASES, got):
        o = _as_outcome(g)
        if "ok" in o:
            o = {"ok": [[d.severity, d.code, d.location, d.message] for d in o["ok"]]}
        if not same(o, r["validate"]):
            bad.append(r["name"])
    assert not bad, bad[:10]


@pytest.mark.parametrize("rec", CASES[::7], ids=[r["name"] for r in CASES[::7]])
def test_decode_module_golden(sk, rec):
    def run():
        h, insts = sk.decode_module(rec["bytes"])
        return [[h.major_version, h.minor_version, h.generator_magic, h.bound, h.schema],
                [[i.opcode, len(i.operands)] for i in insts]]
    assert same(outcome(run), rec["decode"])


def test_synthetic_families_vs_oracle(sk):
    from oracle import disasm as odis, validate as oval
    from synth.families import FAMILIES, build_module
    mods = [build_module(f, s) for f in FAMILIES for s in range(40)]
    got = sk.disassemble_batch(mods)
    assert all(g == odis.disassemble(m) for m, g in zip(mods, got))
    opts = sk.DisassemblerOptions(highlight=True, group=True)
    got = sk.disassemble_batch(mods, opts)
    oo = odis.Options(highlight=True, group=True)
    assert all(g == odis.disassemble(m, oo) for m, g in zip(mods, got))
    vd = sk.validate_batch(mods)
    for m, d in zip(mods, vd):
        assert [(x.severity, x.code, x.location, x.message) for x in d] == \
            [tuple(x) for x in oval.validate(m)]


def _const_module(width, values):
    """One OpTypeFloat/OpTypeInt + one OpConstant per value (raw words)."""
    words = [0x07230203, 0x00010200, 0, len(values) + 2, 0]
    words += [(3 << 16) | 22, 1, width]                       # OpTypeFloat %1 width
    for k, v in enumerate(values):
        if width == 64:
            words += [(5 << 16) | 43, 1, k + 2, v & 0xFFFFFFFF, v >> 32]
        else:
            words += [(4 << 16) | 43, 1, k + 2, v]
    return struct.pack(f"<{len(words)}I", *words)


def _expected_floats(width, values):
    fmt = {16: "<e", 32: "<f", 64: "<d"}[width]
    out = []
    for v in values:
        raw = struct.pack("<Q" if width == 64 else "<I", v)
        out.append(repr(struct.unpack(fmt, raw[: width // 8])[0]))
    return out


@pytest.mark.parametrize("width", [16, 32, 64])
def test_float_repr_matches_cpython(sk, width):
    rng = random.Random(width)
    if width == 16:
        values = list(range(65536))
    elif width == 32:
        values = [rng.getrandbits(32) for _ in range(200000)]
        values += [0x00000001, 0x007FFFFF, 0x00800000, 0x7F7FFFFF, 0x3DCCCCCD, 0x80000000]
    else:
        values = [rng.getrandbits(64) for _ in range(200000)]
        values += [struct.unpack("<Q", struct.pack("<d", x))[0] for x in
                   (1e16, 9999999999999998.0, 1e-05, 0.0001, 5e-324, 1.7976931348623157e308, 0.1)]
    chunks = [values[i:i + 4000] for i in range(0, len(values), 4000)]
    mods = [_const_module(width, c) for c in chunks]
    texts = sk.disassemble_batch(mods, sk.DisassemblerOptions(no_header=True, inline_names=False,
                                                              no_indent=True))
    for c, t in zip(chunks, texts):
        assert not isinstance(t, BaseException), t
        lines = t.splitlines()[1:]
        got = [ln.split(" ")[-1] for ln in lines]
        want = _expected_floats(width, c)
        bad = [(hex(v), w, g) for v, w, g in zip(c, want, got) if w != g]
        assert not bad, bad[:5]


def test_batch_with_mixed_errors_and_sizes(sk):
    """A large shuffled batch: results must not depend on batch position."""
    from oracle import disasm as odis
    rng = random.Random(5)
    pool = [r["bytes"] for r in CASES]
    mods = [rng.choice(pool) for _ in range(3000)]
    got = sk.disassemble_batch(mods)
    cache = {}
    for m, g in zip(mods, got):
        if m not in cache:
            cache[m] = outcome(lambda: odis.disassemble(m))
        assert same(_as_outcome(g), cache[m])


def test_sharded_disasm_world1_gpu(sk):
    """run_sharded + the GPU DisasmSession step (gloo group of one, real kernel)."""
    import socket
    import numpy as np
    import torch.distributed as dist
    from oracle import disasm as odis
    from paper_2305_09493_b200.shard import disasm_shard_fn, run_sharded
    from synth.families import sample_batch
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        b = sample_batch(300, 100, 9)
        m0, m1, arena, spans, status, base, totals = run_sharded(disasm_shard_fn(), b.data, b.offsets,
                                                                 b.lengths)
        assert (m0, m1, base, totals) == (0, b.n, 0, [len(arena)])
        assert (status == 0).all()
        for i in range(0, b.n, 7):
            got = np.asarray(arena)[spans[i, 0]:spans[i, 0] + spans[i, 1]].tobytes().decode()
            assert got == odis.disassemble(b.module(i))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("path", ["grid-wide", "one-warp"])
def test_huge_single_module_vs_oracle(sk, monkeypatch, path):
    """Config-3 shape (one large module, dense OpName, long OpString, ids > 2^16)
    at a size the oracle finishes in seconds: disassembly (default options and
    numeric refs) and validation identical, on the grid-wide path a single-module
    call takes at this size (_native.SINGLE_LARGE_WORDS) and on the one-warp batch
    path it takes inside a batch."""
    from oracle import disasm as odis, validate as oval
    from paper_2305_09493_b200 import _native
    from synth.huge import build_huge
    if path == "one-warp":
        monkeypatch.setattr(_native, "SINGLE_LARGE_WORDS", 1 << 40)
    m = build_huge(400, chain=200, seed=3)          # ~740k words, ids up to ~81k
    assert len(m) // 4 > 500_000
    got = sk.disassemble_batch([m])[0]
    assert got == odis.disassemble(m)
    opts = sk.DisassemblerOptions(inline_names=False)
    assert sk.disassemble_batch([m], opts)[0] == odis.disassemble(m, opts)
    d = sk.validate_batch([m])[0]
    want_v = [tuple(x) for x in oval.validate(m)]
    assert [(x.severity, x.code, x.location, x.message) for x in d] == want_v
    # the fused entry point (grid-wide: text copy overlapped with the validation kernels)
    t, v = sk.disassemble_validate_batch([m])[0]
    assert t == got
    assert [(x.severity, x.code, x.location, x.message) for x in v] == want_v


def test_single_module_routing_sizes(sk):
    """Single-module calls on either side of _native.SINGLE_LARGE_WORDS (one-warp
    batch kernel below, grid-wide kernels from it): every option set, the fused
    disassemble+validate entry point and the decode errors equal the oracle's."""
    import struct
    from oracle import disasm as odis, validate as oval
    from paper_2305_09493_b200 import _native
    from synth.huge import build_huge
    mods = [build_huge(k, chain=c, string_kib=s) for k, c, s in ((1, 20, ()), (4, 50, ()), (8, 200, (1,)))]
    sizes = [len(m) // 4 for m in mods]
    assert min(sizes) < _native.SINGLE_LARGE_WORDS <= max(sizes)
    mods.append(mods[2][:-6])                                        # truncated mid-instruction
    mods.append(mods[2][:20] + struct.pack("<I", 0x00000011) + mods[2][24:])   # word count 0
    option_sets = [sk.DisassemblerOptions(), sk.DisassemblerOptions(inline_names=False),
                   sk.DisassemblerOptions(highlight=True, group=True),
                   sk.DisassemblerOptions(no_indent=True, no_header=True)]
    for m in mods:
        for o in option_sets:
            try:
                want = odis.disassemble(m, o)
            except Exception as exc:  # noqa: BLE001
                want = (type(exc).__name__, str(exc))
            got = sk.disassemble_batch([m], o)[0]
            got = (type(got).__name__, str(got)) if isinstance(got, BaseException) else got
            assert got == want, (len(m), o)
        want_v = [tuple(x) for x in oval.validate(m)]
        got_v = sk.validate_batch([m])[0]
        assert [(x.severity, x.code, x.location, x.message) for x in got_v] == want_v
        _, v = sk.disassemble_validate_batch([m])[0]
        assert [(x.severity, x.code, x.location, x.message) for x in v] == want_v


def test_format_instruction_known_answers(sk):
    """reference tests/test_disasm.py:23-41 known answers through the GPU path."""
    from paper_2305_09493_b200 import CorruptStreamError, NotFoundError, RawInstruction, load_pinned
    spec = load_pinned()
    assert sk.format_instruction(spec, RawInstruction(17, (6,))) == "OpCapability Kernel"
    assert sk.format_instruction(spec, RawInstruction(0, ())) == "OpNop"
    assert sk.format_instruction(spec, RawInstruction(54, (1, 2, 3, 3))) == "%2 = OpFunction %1 Inline|DontInline %3"
    with pytest.raises(CorruptStreamError):
        sk.format_instruction(spec, RawInstruction(17, (6, 7)))
    with pytest.raises(NotFoundError):
        sk.format_instruction(spec, RawInstruction(65520, ()))


def test_mixed_batch_with_large_module(sk, monkeypatch):
    """A batch mixing small modules with one large one (separate launch when the
    shared per-warp slot would exceed the workspace budget)."""
    from oracle import disasm as odis
    from paper_2305_09493_b200 import _native
    from synth.families import FAMILIES, build_module
    from synth.huge import build_huge
    monkeypatch.setattr(_native, "WS_BUDGET", 64 << 20)
    mods = [build_module(f, s) for f in FAMILIES for s in range(3)]
    big = build_huge(40, chain=100, seed=5)
    mods.insert(4, big)
    got = sk.disassemble_batch(mods)
    for m, g in zip(mods, got):
        assert g == odis.disassemble(m)
    val = sk.validate_batch(mods)
    assert all(isinstance(v, list) for v in val)


def test_decode_large_module_tiled(sk):
    """decode_module on large modules takes the tiled boundary pass (skg_decode_large):
    same instructions as the oracle, LE and BE, and the exact first error."""
    import struct
    from oracle import core
    from synth.huge import build_huge
    m = build_huge(300, chain=200, seed=4)          # ~560k words, long OpStrings
    assert len(m) // 4 >= 1 << 16
    from dataclasses import astuple
    h, insts = sk.decode_module(m)
    oh, oinsts = core.decode_module(m)
    assert astuple(h) == tuple(oh)
    assert [(i.opcode, tuple(i.operands)) for i in insts] == [(op, tuple(o)) for op, o in oinsts]
    words = list(struct.unpack(f"<{len(m) // 4}I", m))
    be = struct.pack(f">{len(words)}I", *words)
    h2, insts2 = sk.decode_module(be)
    assert astuple(h2) == astuple(h) and insts2 == insts
    # errors: word count 0 deep inside, and an overrun at the end
    starts = []
    p = 5
    while p < len(words):
        starts.append(p)
        p += words[p] >> 16
    bad = list(words)
    bad[starts[len(starts) * 2 // 3]] &= 0xFFFF
    over = list(words)
    over[starts[-1]] = (5 << 16) | (over[starts[-1]] & 0xFFFF)
    for data in (struct.pack(f"<{len(bad)}I", *bad), struct.pack(f"<{len(over)}I", *over)):
        with pytest.raises(Exception) as e1:
            sk.decode_module(data)
        with pytest.raises(Exception) as e2:
            core.decode_module(data)
        assert (type(e1.value).__name__, str(e1.value)) == (type(e2.value).__name__, str(e2.value))


def test_decode_large_random_word_counts(sk):
    """the tiled boundary pass under corrupted word counts anywhere in the stream (the
    true chain re-enters tiles at arbitrary offsets, merges late or hits an error):
    instructions or the exact first error, as the oracle."""
    import random
    import struct
    from oracle import core
    from synth.huge import build_huge
    m = build_huge(120, chain=150, seed=9, string_kib=(1, 24))
    words = list(struct.unpack(f"<{len(m) // 4}I", m))
    assert len(words) >= 1 << 16
    starts, p = [], 5
    while p < len(words):
        starts.append(p)
        p += words[p] >> 16
    rng = random.Random(5)
    for _ in range(10):
        w = list(words)
        for _ in range(rng.choice((1, 3))):
            at = rng.choice(starts)
            w[at] = (rng.choice((0, 1, 2, 3, 7, 4096, 5000)) << 16) | (w[at] & 0xFFFF)
        data = struct.pack(f"<{len(w)}I", *w)
        try:
            want = core.decode_module(data)
        except Exception as exc:   # noqa: BLE001
            want = exc
        try:
            got = sk.decode_module(data)
        except Exception as exc:   # noqa: BLE001
            got = exc
        if isinstance(want, Exception):
            assert (type(got).__name__, str(got)) == (type(want).__name__, str(want))
        else:
            from dataclasses import astuple
            h, insts = got
            assert astuple(h) == tuple(want[0])
            assert [(i.opcode, tuple(i.operands)) for i in insts] == [(op, tuple(o)) for op, o in want[1]]


def test_validate_large_module_grid_wide(sk, monkeypatch):
    """validate on one large module runs grid-wide (skg_validate_large): same diagnostics
    as the batch path / oracle, including decode errors and instruction diagnostics."""
    import struct
    from oracle import validate as oval
    from paper_2305_09493_b200 import _native
    from synth.huge import build_huge
    monkeypatch.setattr(_native, "LARGE_MODULE_WORDS", 1 << 14)
    m = build_huge(60, chain=100, seed=6)
    words = list(struct.unpack(f"<{len(m) // 4}I", m))
    cases = [m]
    # an unknown opcode (warning), a bound violation and a duplicate result id
    w2 = list(words)
    p = 5
    starts = []
    while p < len(w2):
        starts.append(p)
        p += w2[p] >> 16
    k = starts[len(starts) // 2]
    w2[k] = (w2[k] & 0xFFFF0000) | 0x7FF0
    w2[3] = 50
    cases.append(struct.pack(f"<{len(w2)}I", *w2))
    w3 = list(words)
    w3[starts[-5]] = 0
    cases.append(struct.pack(f"<{len(w3)}I", *w3))           # word count 0: decode error
    cases.append(struct.pack(f">{len(words)}I", *words))     # big-endian
    got = sk.validate_batch(cases)
    for c, g in zip(cases, got):
        want = [tuple(x) for x in oval.validate(c)]
        assert [(x.severity, x.code, x.location, x.message) for x in g] == want


def test_disasm_large_module_grid_wide(sk, monkeypatch):
    """disassembly of one large module runs grid-wide (skg_disasm_large): text
    identical to the oracle under every option set, and the same exceptions."""
    import struct
    from oracle import disasm as odis
    from paper_2305_09493_b200 import _native
    from synth.families import FAMILIES, build_module
    from synth.huge import build_huge
    monkeypatch.setattr(_native, "LARGE_MODULE_WORDS", 1 << 12)
    mods = [build_huge(12, chain=120, seed=7), build_huge(3, chain=400, seed=8)]
    mods += [build_module(f, s) for f in FAMILIES for s in range(2)]   # small ones: batch path
    opts = [sk.DisassemblerOptions(), sk.DisassemblerOptions(inline_names=False),
            sk.DisassemblerOptions(highlight=True, group=True), sk.DisassemblerOptions(no_indent=True, no_header=True)]
    for o in opts:
        got = sk.disassemble_batch(mods, o)
        for m, g in zip(mods, got):
            assert g == odis.disassemble(m, o)
    # exceptions: an unknown opcode under strict, invalid UTF-8 in an OpName
    words = list(struct.unpack(f"<{len(mods[0]) // 4}I", mods[0]))
    p, starts = 5, []
    while p < len(words):
        starts.append(p)
        p += words[p] >> 16
    w1 = list(words)
    k = starts[len(starts) // 2]
    w1[k] = (w1[k] & 0xFFFF0000) | 0x7FF0
    name_at = next(s for s in starts if words[s] & 0xFFFF == 5)
    w2 = list(words)
    w2[name_at + 2] = 0x00FFFE61
    bad = [struct.pack(f"<{len(w)}I", *w) for w in (w1, w2)]
    for strict in (False, True):
        got = sk.disassemble_batch(bad, None, strict=strict)
        for m, g in zip(bad, got):
            try:
                want = odis.disassemble(m, strict=strict)
            except Exception as exc:   # noqa: BLE001
                want = exc
            if isinstance(want, Exception):
                assert (type(g).__name__, str(g)) == (type(want).__name__, str(want))
            else:
                assert g == want


def test_disasm_large_module_many_name_families(sk, monkeypatch):
    """grid-wide name de-duplication with many parent / child / grandchild name
    groups (x, x_0, x_1, x_0_0 ...) over several 1024-ident chunks, so the ordered
    pass's group-state cache sees collisions and evictions: text == oracle."""
    from oracle import disasm as odis
    from paper_2305_09493_b200 import _native
    import synth.huge as huge
    monkeypatch.setattr(_native, "LARGE_MODULE_WORDS", 1 << 12)
    vocab = [f"p{i}" for i in range(700)] + [f"p{i}_0" for i in range(0, 700, 2)]
    vocab += [f"p{i}_1" for i in range(0, 700, 3)] + [f"p{i}_0_0" for i in range(0, 100, 4)]
    vocab += ["x", "x_0", "x_1", "x_0_0", "x_2"]
    monkeypatch.setattr(huge, "VOCAB", tuple(vocab))
    for seed in (3, 4):
        m = huge.build_huge(8, chain=200, seed=seed)
        got = sk.disassemble_batch([m])[0]
        assert got == odis.disassemble(m)


def test_large_paths_edge_cases(sk, monkeypatch):
    """The whole-GPU single-module paths on degenerate inputs: header only, a
    truncated stream, a foreign magic, big-endian, and an empty-string OpName."""
    import struct
    from oracle import core
    from oracle import disasm as odis, validate as oval
    from paper_2305_09493_b200 import _native
    monkeypatch.setattr(_native, "LARGE_MODULE_WORDS", 1)
    monkeypatch.setattr(_native, "LARGE_DECODE_WORDS", 1)
    hdr = [0x07230203, 0x00010200, 0, 10, 0]
    cases = [struct.pack("<5I", *hdr),
             struct.pack("<5I", *hdr) + b"\x01\x02",
             struct.pack("<5I", 0x12345678, *hdr[1:]),
             struct.pack(">5I", *hdr) + struct.pack(">2I", (2 << 16) | 17, 6),
             struct.pack("<5I", *hdr) + struct.pack("<3I", (3 << 16) | 5, 1, 0)]

    def outcome(f, m):
        try:
            r = f(m)
        except Exception as exc:   # noqa: BLE001
            return ("exc", type(exc).__name__, str(exc))
        return ("ok", r)

    for m in cases:
        got = sk.disassemble_batch([m])[0]
        want = outcome(odis.disassemble, m)
        assert (("exc", type(got).__name__, str(got)) if isinstance(got, BaseException) else ("ok", got)) == want
        gv = sk.validate_batch([m])[0]
        wv = [tuple(x) for x in oval.validate(m)]
        assert [(x.severity, x.code, x.location, x.message) for x in gv] == wv
        gd = outcome(lambda x: [(i.opcode, tuple(i.operands)) for i in sk.decode_module(x)[1]], m)
        wd = outcome(lambda x: [(op, tuple(o)) for op, o in core.decode_module(x)[1]], m)
        assert gd == wd


def test_small_module_with_large_bound(sk):
    """A small module whose header bound exceeds the hash capacity its per-warp slot is
    sized for (bound up to 2W + 64 still takes the direct id tables) falls back to the
    hash tables instead of failing (regression: "module exceeds the per-warp scratch
    slot" for format_instruction contexts)."""
    import struct as st
    from oracle import disasm as odis, validate as oval
    done = 0
    for rec in CASES:
        data = rec["bytes"]
        if "ok" not in rec["disasm"]["default"] or len(data) < 24 or len(data) > 400:
            continue
        w = list(st.unpack(f"<{len(data) // 4}I", data))
        if w[0] != 0x07230203:
            continue
        for bound in (2 * len(w) + 40, 2 * len(w) + 64):
            w[3] = bound
            m = st.pack(f"<{len(w)}I", *w)
            assert sk.disassemble_batch([m])[0] == odis.disassemble(m)
            d = sk.validate_batch([m])[0]
            assert [(x.severity, x.code, x.location, x.message) for x in d] == [tuple(x) for x in oval.validate(m)]
        done += 1
        if done >= 25:
            break
    assert done >= 10


def test_fused_disasm_validate_goldens(sk):
    """the fused decode -> validate -> disassemble pass gives, for every
    golden module and every option set, exactly the reference's text (or exception) AND
    its diagnostics (or exception) -- both goldens from one kernel."""
    datas = [r["bytes"] for r in CASES]
    for key, opts in OPTION_SETS.items():
        got = sk.disassemble_validate_batch(datas, sk.DisassemblerOptions(**opts))
        bad = []
        for r, (t, d) in zip(CASES, got):
            if not same(_as_outcome(t), r["disasm"][key]):
                bad.append((r["name"], "disasm"))
            o = _as_outcome(d)
            if "ok" in o:
                o = {"ok": [[x.severity, x.code, x.location, x.message] for x in o["ok"]]}
            if not same(o, r["validate"]):
                bad.append((r["name"], "validate"))
        assert not bad, (key, bad[:10])
    got = sk.disassemble_validate_batch(datas, strict=True)
    bad = [r["name"] for r, (t, _) in zip(CASES, got) if not same(_as_outcome(t), r["disasm_strict"])]
    assert not bad, bad[:10]


def test_fused_matches_separate_on_families(sk):
    """the fused pass on a shuffled synthetic batch equals the two separate kernels"""
    from synth.families import sample_batch
    b = sample_batch(3000, 300, 77)
    mods = [b.module(i) for i in range(b.n)]
    fused = sk.disassemble_validate_batch(mods)
    texts = sk.disassemble_batch(mods)
    diags = sk.validate_batch(mods)
    assert [t for t, _ in fused] == texts
    assert [d for _, d in fused] == diags


def test_large_module_ids_above_header_bound_stay_grid_wide(sk, monkeypatch):
    """A large module whose ids reach its header bound is redone grid-wide with id tables
    widened to 2W + 64 (BoundTooSmall still names the header bound) instead of the
    one-warp batch path (which this test disables)."""
    import struct
    from oracle import disasm as odis, validate as oval
    from paper_2305_09493_b200 import _native
    from synth.huge import build_huge
    monkeypatch.setattr(_native, "LARGE_MODULE_WORDS", 1 << 14)

    def no_warp_path(*a, **k):
        raise AssertionError("the one-warp batch path was used")
    monkeypatch.setattr(_native, "run_disasm", no_warp_path)
    monkeypatch.setattr(_native, "run_validate", no_warp_path)
    m = build_huge(40, chain=100, seed=9)
    w = list(struct.unpack(f"<{len(m) // 4}I", m))
    for bound in (100, w[3] - 1):
        w[3] = bound
        mm = struct.pack(f"<{len(w)}I", *w)
        d = sk.validate_batch([mm])[0]
        assert [(x.severity, x.code, x.location, x.message) for x in d] == [tuple(x) for x in oval.validate(mm)]
        for o in (sk.DisassemblerOptions(), sk.DisassemblerOptions(inline_names=False)):
            assert sk.disassemble_batch([mm], o)[0] == odis.disassemble(mm, o)


def test_f32_repr_exhaustive_on_device(sk):
    """All 2^32 float32 bit patterns (SURVEY.md 7 hard part 2): the disassembler's repr of
    the widened value reads back exactly through the assembler's independent float()
    parser and is the shortest such text (skg_selftest_repr_f32); plus an exact
    comparison with CPython repr on 300k random patterns through the disasm kernel."""
    import ctypes
    import random
    import struct as st
    import torch
    from paper_2305_09493_b200 import _native
    L = _native.lib()
    th = _native.tables_handle(None, None)
    fails = torch.zeros(1, dtype=torch.int64, device="cuda")
    first = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    step = 1 << 28
    for start in range(0, 1 << 32, step):
        assert L.skg_selftest_repr_f32(th, start, step, fails.data_ptr(), first.data_ptr(),
                                       ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
    torch.cuda.synchronize()
    assert int(fails.item()) == 0, hex(int(first.item()) & 0xFFFFFFFF)
    rng = random.Random(5)
    vals = [rng.getrandbits(32) for _ in range(300_000)]
    vals = [v for v in vals if (v >> 23) & 0xFF != 0xFF]
    want = [repr(st.unpack("<f", st.pack("<I", v))[0]) for v in vals]
    # one OpConstant per value under a 32-bit float type, numeric refs, no header/indent
    words = [0x07230203, 0x00010200, 0, len(vals) + 3, 0, (3 << 16) | 22, 1, 32]
    for k, v in enumerate(vals):
        words += [(4 << 16) | 43, 1, 2 + k, v]
    m = st.pack(f"<{len(words)}I", *words)
    text = sk.disassemble_batch([m], sk.DisassemblerOptions(inline_names=False, no_indent=True,
                                                             no_header=True))[0]
    got = [ln.rsplit(" ", 1)[1] for ln in text.splitlines()[1:]]
    assert got == want


def test_decode_large_long_unmarked_runs(sk):
    """The parallel tile link gives up on a successor walk that crosses more than 16
    tiles without meeting a speculative chain (runs of maximal OpStrings: 65535 words
    each, their string words are not plausible instruction starts); the sequential
    link then decides.  Instructions, and the exact first error after the runs, as the
    oracle."""
    import struct
    from dataclasses import astuple
    from oracle import core
    words = [0x07230203, 0x00010100, 0, 100, 0]
    for _ in range(8):                                   # small instructions
        words += [(2 << 16) | 17, 11]                    # OpCapability 11
    for r in range(3):                                   # a run of maximal OpStrings
        for _ in range(5):
            body = [0x61616161] * 65533 + [0]            # "aaaa..." + NUL word: 65534 words
            words += [(65535 << 16) | 7, 1 + r] + body[:65533]
    for _ in range(40):
        words += [(2 << 16) | 17, 11]
    data = struct.pack(f"<{len(words)}I", *words)
    h, insts = sk.decode_module(data)
    oh, oinsts = core.decode_module(data)
    assert astuple(h) == tuple(oh)
    assert [(i.opcode, tuple(i.operands)) for i in insts] == [(op, tuple(o)) for op, o in oinsts]
    bad = list(words)
    bad[-20] = 11                                        # word count 0 after the runs
    data = struct.pack(f"<{len(bad)}I", *bad)
    with pytest.raises(Exception) as e1:
        sk.decode_module(data)
    with pytest.raises(Exception) as e2:
        core.decode_module(data)
    assert (type(e1.value).__name__, str(e1.value)) == (type(e2.value).__name__, str(e2.value))
