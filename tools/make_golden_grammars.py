"""Golden vectors for non-default grammars, recorded by running
the REFERENCE (build container only):

* the pinned SPIR-V 1.2 grammar (``load_pinned("1.2")``, grammar.py:403-413: no
  instruction classes, so the assembler's builder routing rejects module-level
  instructions);
* a custom ``GrammarSpec`` loaded with ``load_core_grammar`` from an edited copy
  of the unified1 JSON: OpFAdd removed (unknown opcode), OpIAdd renamed OpIntAdd,
  Float64 made to imply Int64 (capability closure), a FunctionControl enumerant
  added (mask rendering), the ext grammar unchanged.

For every module of tests/golden/modules.jsonl.gz plus the paper families:
disassembly (default and numeric options), validation, and re-assembly of the
default disassembly, each under both grammars.  Output:
tests/golden/grammars.json.gz (with the custom grammar's JSON text).
"""

from __future__ import annotations

import copy
import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import spirvkit as sk  # noqa: E402  (the reference)
from golden_io import modules  # noqa: E402

REF_GRAMMAR = Path("/root/reference/pkg/src/spirvkit/grammars/unified1/spirv.core.grammar.json")
OUT = ROOT / "tests" / "golden" / "grammars.json.gz"


def custom_grammar_text() -> str:
    doc = json.loads(REF_GRAMMAR.read_text(encoding="utf-8"))
    doc = copy.deepcopy(doc)
    doc["instructions"] = [i for i in doc["instructions"] if i["opname"] != "OpFAdd"]
    for i in doc["instructions"]:
        if i["opname"] == "OpIAdd":
            i["opname"] = "OpIntAdd"
    for k in doc["operand_kinds"]:
        if k["kind"] == "Capability":
            for e in k["enumerants"]:
                if e["enumerant"] == "Float64":
                    e["capabilities"] = ["Int64"]
        if k["kind"] == "FunctionControl":
            k["enumerants"].append({"enumerant": "Hot", "value": "0x0100"})
    return json.dumps(doc, indent=1)


def outcome(fn):
    try:
        return {"ok": fn()}
    except Exception as exc:  # noqa: BLE001 - every class is recorded
        return {"exc": [type(exc).__name__, str(exc)]}


def main():
    from synth.families import FAMILIES, build_module
    text = custom_grammar_text()
    grammars = {"1.2": sk.load_pinned("1.2"), "custom": sk.load_core_grammar(text)}
    mods = [(r["name"], r["bytes"]) for r in modules()]
    mods += [(f"fam_{f}_{s}", build_module(f, 100 + s)) for f in FAMILIES for s in range(3)]
    recs = []
    for name, data in mods:
        rec = {"name": name}
        for g, spec in grammars.items():
            dis = outcome(lambda: sk.disassemble_module(data, spec=spec))
            rec[g] = {
                "disasm": dis,
                "numeric": outcome(lambda: sk.disassemble_module(
                    data, sk.DisassemblerOptions(inline_names=False), spec=spec)),
                "validate": outcome(lambda: [[d.severity, d.code, d.location, d.message]
                                             for d in sk.validate_module(data, spec=spec)]),
            }
            if "ok" in dis:
                asm = outcome(lambda: sk.assemble_module(dis["ok"], spec=spec).hex())
                rec[g]["asm"] = asm
        recs.append(rec)
    with gzip.open(OUT, "wt", encoding="utf-8") as fh:
        json.dump({"custom_grammar": text, "modules": recs}, fh)
    print(len(recs), "modules")


if __name__ == "__main__":
    main()
