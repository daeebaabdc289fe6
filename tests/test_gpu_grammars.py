"""Non-default grammars on the GPU path: the pinned SPIR-V 1.2
grammar and a custom GrammarSpec (edited unified1: an opcode removed, one renamed,
a capability dependency and a mask enumerant added), packed by tables.pack into
the device tables.  Disassembly (default / numeric), validation and re-assembly
against the reference's outputs under the same grammar
(tools/make_golden_grammars.py)."""

import gzip
import json
from functools import lru_cache
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).parent / "golden" / "grammars.json.gz"


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


def _spec(sk, which):
    return sk.load_pinned("1.2") if which == "1.2" else sk.load_core_grammar(golden()["custom_grammar"])


def _out(r, as_diags=False):
    if isinstance(r, BaseException):
        return {"exc": [type(r).__name__, str(r)]}
    if as_diags:
        return {"ok": [[d.severity, d.code, d.location, d.message] for d in r]}
    return {"ok": r}


def _same(got, want):
    if "exc" in want:
        return "exc" in got and got["exc"] == want["exc"]
    return got == want


@pytest.mark.parametrize("which", ["1.2", "custom"])
def test_grammar_disasm_validate_asm(sk, which):
    from golden_io import modules
    spec = _spec(sk, which)
    data = {r["name"]: r["bytes"] for r in modules()}
    from synth.families import FAMILIES, build_module
    for f in FAMILIES:
        for s in range(3):
            data[f"fam_{f}_{s}"] = build_module(f, 100 + s)
    recs = golden()["modules"]
    mods = [data[r["name"]] for r in recs]
    bad = []
    for key, opts in (("disasm", None), ("numeric", sk.DisassemblerOptions(inline_names=False))):
        got = sk.disassemble_batch(mods, opts, spec=spec)
        bad += [(r["name"], key) for r, g in zip(recs, got) if not _same(_out(g), r[which][key])]
    got = sk.validate_batch(mods, spec=spec)
    bad += [(r["name"], "validate") for r, g in zip(recs, got)
            if not _same(_out(g, True), r[which]["validate"])]
    texts = [(r, r[which]["disasm"]["ok"]) for r in recs if "asm" in r[which]]
    got = sk.assemble_batch([t for _, t in texts], spec=spec)
    bad += [(r["name"], "asm") for (r, _), g in zip(texts, got)
            if not _same(_out(g.hex() if isinstance(g, bytes) else g), r[which]["asm"])]
    assert not bad, bad[:10]


@pytest.mark.parametrize("which", ["1.2", "custom"])
def test_grammar_grid_wide_single_module_path(sk, monkeypatch, which):
    """The same goldens through the grid-wide single-module kernels (skg_disasm_large /
    skg_validate_large), which single-module calls of _native.SINGLE_LARGE_WORDS words
    and up take: forced here for every module, one call per module."""
    from golden_io import modules
    from paper_2305_09493_b200 import _native
    monkeypatch.setattr(_native, "SINGLE_LARGE_WORDS", 1)
    spec = _spec(sk, which)
    data = {r["name"]: r["bytes"] for r in modules()}
    from synth.families import FAMILIES, build_module
    for f in FAMILIES:
        for s in range(3):
            data[f"fam_{f}_{s}"] = build_module(f, 100 + s)
    bad = []
    numeric = sk.DisassemblerOptions(inline_names=False)
    for r in golden()["modules"]:
        m = data[r["name"]]
        for key, opts in (("disasm", None), ("numeric", numeric)):
            if not _same(_out(sk.disassemble_batch([m], opts, spec=spec)[0]), r[which][key]):
                bad.append((r["name"], key))
        if not _same(_out(sk.validate_batch([m], spec=spec)[0], True), r[which]["validate"]):
            bad.append((r["name"], "validate"))
    assert not bad, bad[:10]
