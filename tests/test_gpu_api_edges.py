"""API edges against reference-recorded goldens (tools/make_golden_api.py):
Assembler default_version (asm.py:184-206), check_capability_closure /
diagnostics_text (validate.py:223-234, 299-301) and validate_module given a
builder ModuleScope (validate.py:64-70), all through the CUDA kernels."""

import base64
import gzip
import json
from functools import lru_cache
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).parent / "golden" / "api_edges.json.gz"


@lru_cache(maxsize=None)
def gold():
    with gzip.open(GOLD, "rt", encoding="utf-8") as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def sk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2305_09493_b200 as pkg
    return pkg


def _outcome(fn):
    try:
        return {"ok": fn()}
    except Exception as exc:  # noqa: BLE001
        return {"exc": [type(exc).__name__, str(exc)]}


def test_assembler_default_version(sk):
    from paper_2305_09493_b200.asm import assemble_batch
    g = gold()
    texts = g["texts"]
    by_dv = {}
    for rec in g["default_version"]:
        by_dv.setdefault(tuple(rec["dv"]), []).append(rec)
    for dv, recs in by_dv.items():
        got = assemble_batch(texts, default_version=dv)
        for rec in recs:
            out = got[rec["text"]]
            o = {"exc": [type(out).__name__, str(out)]} if isinstance(out, BaseException) else {"ok": out.hex()}
            assert o == rec["out"], (dv, rec["text"])
        # the single-module entry point agrees with the batch
        rec = recs[0]
        assert _outcome(lambda: sk.Assembler(default_version=dv).assemble(texts[rec["text"]]).hex()) == rec["out"]


def test_check_capability_closure_and_diagnostics_text(sk):
    import golden_io
    mods = golden_io.modules()
    g = gold()
    for rec in g["closure"]:
        data = mods[rec["module"]]["bytes"]
        got = _outcome(lambda: [[d.severity, d.code, d.location, d.message]
                                for d in sk.check_capability_closure(data)])
        assert got == rec["closure"], rec["module"]
        got = _outcome(lambda: sk.diagnostics_text(sk.validate_module(data)))
        assert got == rec["text"], rec["module"]


def test_validate_module_scope(sk):
    class Scope:   # a builder ModuleScope stand-in: validate_module serializes it (validate.py:64-70)
        def __init__(self, data):
            self.data = data

        def to_bytes(self):
            return self.data

    for rec in gold()["module_scope"]:
        data = base64.b64decode(rec["data"])
        got = [[d.severity, d.code, d.location, d.message] for d in sk.validate_module(Scope(data))]
        assert got == rec["diags"], rec["name"]
    with pytest.raises(TypeError, match="validate_module expects bytes or a ModuleScope"):
        sk.validate_module(12345)
