"""Golden vectors recorded from the reference (tools/make_golden.py)."""

import base64
import gzip
import json
from functools import lru_cache
from pathlib import Path

GOLDEN = Path(__file__).parent / "golden"
OPTION_SETS = {
    "default": {},
    "no_header": {"no_header": True},
    "numeric": {"inline_names": False},
    "highlight": {"highlight": True},
    "group_noindent": {"group": True, "no_indent": True},
    "all": {"highlight": True, "group": True, "no_header": True},
}


@lru_cache(maxsize=None)
def modules():
    out = []
    with gzip.open(GOLDEN / "modules.jsonl.gz", "rt", encoding="utf-8") as fh:
        for line in fh:
            rec = json.loads(line)
            rec["bytes"] = base64.b64decode(rec["data"])
            out.append(rec)
    return out


@lru_cache(maxsize=None)
def asm_texts():
    with gzip.open(GOLDEN / "asm.jsonl.gz", "rt", encoding="utf-8") as fh:
        return [json.loads(line) for line in fh]


def outcome(fn):
    """Same shape as tools/make_golden.py records: {"ok": v} or {"exc": [cls, msg]}."""
    try:
        return {"ok": fn()}
    except Exception as exc:  # noqa: BLE001
        return {"exc": [type(exc).__name__, str(exc)]}


def same(got, want):
    if "exc" in want:
        return "exc" in got and got["exc"][:2] == want["exc"][:2]
    return got == {"ok": want["ok"]}
