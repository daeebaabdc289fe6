"""Pin the CPU oracle against the reference's recorded outputs (CPU only)."""

import pytest

from golden_io import OPTION_SETS, modules, outcome, same
from oracle import core, disasm, validate

CASES = modules()


@pytest.mark.parametrize("rec", CASES, ids=[r["name"] for r in CASES])
def test_oracle_decode(rec):
    def run():
        h, insts = core.decode_module(rec["bytes"])
        return [list(h), [[op, len(w)] for op, w in insts]]
    assert same(outcome(run), rec["decode"])


@pytest.mark.parametrize("rec", CASES, ids=[r["name"] for r in CASES])
def test_oracle_disasm(rec):
    for key, opts in OPTION_SETS.items():
        got = outcome(lambda: disasm.disassemble(rec["bytes"], disasm.Options(**opts)))
        assert same(got, rec["disasm"][key]), key
    got = outcome(lambda: disasm.disassemble(rec["bytes"], strict=True))
    assert same(got, rec["disasm_strict"])


@pytest.mark.parametrize("rec", CASES, ids=[r["name"] for r in CASES])
def test_oracle_fixpoint_equals_closed_form(rec):
    a = outcome(lambda: disasm.disassemble(rec["bytes"], closed_form=False))
    b = outcome(lambda: disasm.disassemble(rec["bytes"], closed_form=True))
    assert a == b


@pytest.mark.parametrize("rec", CASES, ids=[r["name"] for r in CASES])
def test_oracle_validate(rec):
    got = outcome(lambda: [list(d) for d in validate.validate(rec["bytes"])])
    assert same(got, rec["validate"])


from golden_io import asm_texts  # noqa: E402
from oracle import asm as oasm  # noqa: E402

ASM = asm_texts()


@pytest.mark.parametrize("rec", ASM, ids=[r["name"] for r in ASM])
def test_oracle_assemble(rec):
    got = outcome(lambda: oasm.assemble(rec["text"]).hex())
    assert same(got, rec["asm"])


def test_capability_dependency_graph_golden():
    """grammar.capability_dependency_graph (host, grammar-constant) == the reference's
    DependencyReport for both pinned grammars (tests/golden/boundary.json.gz)."""
    import gzip
    import json
    from pathlib import Path
    from paper_2305_09493_b200 import capability_dependency_graph, load_pinned
    with gzip.open(Path(__file__).parent / "golden" / "boundary.json.gz", "rt", encoding="utf-8") as fh:
        want = json.load(fh)["dependency"]
    for version, rec in want.items():
        rep = capability_dependency_graph(load_pinned(version))
        assert list(rep.nodes) == rec["nodes"]
        assert {k: list(v) for k, v in rep.edges.items()} == rec["edges"]
        assert [list(c) for c in rep.cycles] == rec["cycles"]
