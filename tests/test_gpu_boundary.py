"""The reference's fine-grained boundary functions on the GPU
kernels of csrc/skg_codec.cuh and skg_disasm_refs, against golden vectors
recorded from the reference (tools/make_golden_boundary.py):
tokenize_line, encode_header / encode_instruction / encode_module /
encode_string_literal / encode_context_dependent_literal, and
format_instruction with a RenderContext."""

import gzip
import hashlib
import json
import struct
from functools import lru_cache
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).parent / "golden" / "boundary.json.gz"


@lru_cache(maxsize=None)
def golden():
    with gzip.open(GOLDEN, "rt", encoding="utf-8") as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def sk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2305_09493_b200 as sk
    return sk


def dec_val(v):
    if v is None:
        return None
    if "b" in v:
        return v["b"]
    if "f" in v:
        return float(v["f"])
    if "i" in v:
        return int(v["i"])
    return v["s"]


def ops_of(rec):
    return list(range(rec["range"])) if isinstance(rec, dict) else [int(x) for x in rec]


def check(got, want):
    """got: value or exception instance; want: {"ok": v} | {"exc": [cls, msg]}"""
    if "exc" in want:
        return isinstance(got, BaseException) and [type(got).__name__, str(got)] == want["exc"]
    return not isinstance(got, BaseException) and got == want["ok"]


def _tok(t):
    return None if t is None else [t.text, t.column, t.is_string]


def test_tokenize_lines_batch(sk):
    """every golden line in one batch (line numbers 1..n here, so they are not compared;
    test_tokenize_line_single checks them)"""
    cases = golden()["tokenize"]
    batch = sk.tokenize_lines([c["line"] for c in cases], 1)
    bad = []
    for c, r in zip(cases, batch):
        want = c["out"]
        if isinstance(r, BaseException):
            ok = "exc" in want and type(r).__name__ == want["exc"][0] and \
                [[d.column, d.message] for d in r.diagnostics] == [d[1:] for d in want["diags"]]
        elif r is None:
            ok = want == {"ok": None}
        else:
            ok = "ok" in want and want["ok"] is not None and \
                [_tok(r.result), _tok(r.opname), [_tok(t) for t in r.operands]] == \
                [want["ok"]["result"], want["ok"]["opname"], want["ok"]["operands"]]
        if not ok:
            bad.append((c["line"], want, r))
    assert not bad, bad[:5]


def test_tokenize_line_single(sk):
    cases = golden()["tokenize"]
    for c in cases[-40:] + cases[:200:5]:
        try:
            r = sk.tokenize_line(c["line"], c["lineno"])
        except Exception as exc:  # noqa: BLE001
            assert [type(exc).__name__, str(exc)] == c["out"]["exc"], c["line"]
            assert [[d.line, d.column, d.message] for d in exc.diagnostics] == c["out"]["diags"]
            continue
        want = c["out"]["ok"]
        if want is None:
            assert r is None, c["line"]
        else:
            assert [_tok(r.result), _tok(r.opname), [_tok(t) for t in r.operands], r.line] == \
                [want["result"], want["opname"], want["operands"], want["line"]], c["line"]


def test_encode_header(sk):
    for c in golden()["encode_header"]:
        h = sk.ModuleHeader(*[int(x) for x in c["h"]])
        try:
            got = sk.encode_header(h)
        except Exception as exc:  # noqa: BLE001
            got = exc
        assert check(got, c["out"]), c


def test_encode_instruction(sk):
    for c in golden()["encode_instruction"]:
        inst = sk.RawInstruction(int(c["op"]), tuple(ops_of(c["ops"])))
        try:
            got = sk.encode_instruction(inst)
        except Exception as exc:  # noqa: BLE001
            got = exc
        if "ok_sha" in c["out"]:
            assert hashlib.sha256(struct.pack(f"<{len(got)}I", *got)).hexdigest() == c["out"]["ok_sha"]
        else:
            assert check(got, c["out"]), (c["op"], c["out"])


def test_encode_modules_batch(sk):
    cases = golden()["encode_module"]
    mods = [(sk.ModuleHeader(*c["h"]), [sk.RawInstruction(o, tuple(ops_of(w))) for o, w in c["insts"]])
            for c in cases]
    got = sk.encode_modules(mods)
    for c, g in zip(cases, got):
        assert check(g.hex() if isinstance(g, bytes) else g, c["out"]), c["out"]
    for c, (h, insts) in zip(cases[:10], mods[:10]):      # single-module API
        try:
            g = sk.encode_module(h, insts).hex()
        except Exception as exc:  # noqa: BLE001
            g = exc
        assert check(g, c["out"])


def test_encode_string_literals(sk):
    cases = golden()["encode_string"]
    got = sk.encode_string_literals([c["s"] for c in cases])
    for c, g in zip(cases, got):
        assert check(g, c["out"]), c
    for c in cases[:12]:
        try:
            g = sk.encode_string_literal(c["s"])
        except Exception as exc:  # noqa: BLE001
            g = exc
        assert check(g, c["out"]), c


def test_encode_context_dependent_literals(sk):
    cases = golden()["encode_ctx"]
    items = [(dec_val(c["v"]), c["w"], c["signed"], c["floating"]) for c in cases]
    got = sk.encode_context_dependent_literals(items)
    bad = [(it, c["out"], g) for it, c, g in zip(items, cases, got) if not check(g, c["out"])]
    assert not bad, bad[:5]
    with pytest.raises(sk.CodecError):
        sk.encode_context_dependent_literal(256, 8)
    assert sk.encode_context_dependent_literal(-1, 64, signed=True) == [0xFFFFFFFF, 0xFFFFFFFF]


def test_format_instruction_with_context(sk):
    from paper_2305_09493_b200.disasm import RenderContext
    spec, ext = sk.load_pinned(), sk.load_pinned_extended()
    bad = []
    for c in golden()["format_instruction"]:
        ctx = None
        if c["ctx"] is not None:
            x = c["ctx"]
            ctx = RenderContext(refs={int(k): v for k, v in x["refs"].items()},
                                type_info={int(k): tuple(v) for k, v in x["type_info"].items()},
                                value_type={int(k): v for k, v in x["value_type"].items()},
                                import_sets={int(k): v for k, v in x["import_sets"].items()})
        try:
            got = sk.format_instruction(spec, sk.RawInstruction(c["op"], tuple(c["ops"])), ctx,
                                        ext if c["ext"] else None)
        except Exception as exc:  # noqa: BLE001
            got = exc
        if not check(got, c["out"]):
            bad.append((c, got))
    assert not bad, bad[:5]


def test_serialize_modules_batch(sk):
    """Batch builder serialization: modules built with the reference's
    builder (inputs only; oracle/_ref) serialize through skg_encode_modules to the bytes
    the builder's own ModuleScope.to_bytes writes."""
    import sys
    from pathlib import Path
    ref = Path(__file__).resolve().parents[1] / "oracle" / "_ref"
    if not (ref / "spirvkit").is_dir():
        pytest.skip("reference builder not installed (oracle/_ref)")
    sys.path.insert(0, str(ref))
    sys.path.insert(0, str(ref / "ref_tests"))
    try:
        import corpus
    except ImportError:
        pytest.skip("reference corpus not staged")
    scopes = list(corpus.crafted_modules().values()) + [corpus.random_module(s) for s in range(40)]
    got = sk.serialize_modules(scopes)
    for scope, g in zip(scopes, got):
        try:
            want = scope.to_bytes()
        except Exception as exc:  # noqa: BLE001
            assert isinstance(g, BaseException) and type(g).__name__ == type(exc).__name__ and str(g) == str(exc)
            continue
        assert g == want
