"""Convert Khronos SPIR-V grammar JSON into this repo's compact grammar files.

The compact files under ``paper_2305_09493_b200/grammars/`` keep exactly the
fields the codec path reads (opcode, class, operand slots, enumerants,
capabilities, composite bases) in positional arrays, plus the SHA-256 of the
Khronos source they were derived from.  The source snapshots are the ones the
reference pins (``pkg/src/spirvkit/grammars/PINNED.json``: SPIRV-Headers
@4995a2f, sdk-1.3.211.0).

Usage: python tools/pack_grammar.py [KHRONOS_GRAMMAR_DIR]
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "paper_2305_09493_b200" / "grammars"
DEFAULT_SRC = Path("/root/reference/pkg/src/spirvkit/grammars")


def _slot(o):
    return [o["kind"], o.get("quantifier", ""), o.get("name")]


def _inst(i):
    return [i["opname"], int(i["opcode"]), i.get("class", ""),
            [_slot(o) for o in i.get("operands", [])], list(i.get("capabilities", []))]


def _enum(e):
    return [e["enumerant"], e["value"], list(e.get("capabilities", [])),
            [_slot(p) for p in e.get("parameters", [])]]


def _kind(k):
    enums = [_enum(e) for e in k["enumerants"]] if "enumerants" in k else None
    return [k["category"], k["kind"], enums, k.get("bases")]


def pack_core(path: Path) -> dict:
    raw = path.read_bytes()
    doc = json.loads(raw)
    return {
        "format": "skg-core-grammar-1",
        "source_sha256": hashlib.sha256(raw).hexdigest(),
        "header": [doc.get("magic_number", "0x07230203"), doc.get("major_version", 1),
                   doc.get("minor_version", 0), doc.get("revision", 0)],
        "insts": [_inst(i) for i in doc["instructions"]],
        "kinds": [_kind(k) for k in doc["operand_kinds"]],
    }


def pack_ext(path: Path) -> dict:
    raw = path.read_bytes()
    doc = json.loads(raw)
    return {
        "format": "skg-ext-grammar-1",
        "source_sha256": hashlib.sha256(raw).hexdigest(),
        "header": [doc.get("version", 0), doc.get("revision", 0)],
        "insts": [_inst(i) for i in doc["instructions"]],
    }


def main(argv):
    src = Path(argv[1]) if len(argv) > 1 else DEFAULT_SRC
    OUT.mkdir(parents=True, exist_ok=True)
    jobs = [
        ("unified1.json", pack_core(src / "unified1" / "spirv.core.grammar.json")),
        ("1.2.json", pack_core(src / "1.2" / "spirv.core.grammar.json")),
        ("opencl.std.100.json", pack_ext(src / "unified1" / "extinst.opencl.std.100.grammar.json")),
    ]
    for name, doc in jobs:
        (OUT / name).write_text(json.dumps(doc, separators=(",", ":")) + "\n", encoding="utf-8")
        print(name, doc["source_sha256"])


if __name__ == "__main__":
    main(sys.argv)
