"""Golden vectors for API edges the main goldens do not exercise, recorded by
running the REFERENCE (build container only):

* ``Assembler(default_version=...)`` on texts without a ``; Version:`` header
  (asm.py:184-206): every supported default plus out-of-range ones (ValueError);
* ``check_capability_closure`` (validate.py:223-234) and ``diagnostics_text``
  (validate.py:299-301) for every module of tests/golden/modules.jsonl.gz;
* ``validate_module`` given a builder ``ModuleScope`` (validate.py:64-70), for
  the reference corpus kernels (tests/corpus.py), recorded with the module bytes.

Output: tests/golden/api_edges.json.gz
"""

from __future__ import annotations

import base64
import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, "/root/reference/pkg/tests")
sys.path.insert(2, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import spirvkit as sk  # noqa: E402  (the reference)
from golden_io import modules, outcome  # noqa: E402

OUT = ROOT / "tests" / "golden" / "api_edges.json.gz"


def diag_list(ds):
    return [[d.severity, d.code, d.location, d.message] for d in ds]


def main():
    recs = {"default_version": [], "closure": [], "module_scope": []}
    # assembler default versions: texts of the paper families without their header
    from synth.families import FAMILIES, build_module
    texts = []
    for f in FAMILIES:
        t = sk.disassemble_module(build_module(f, 1))
        body = "\n".join(ln for ln in t.splitlines() if not ln.startswith(";"))
        texts.append(body)
        texts.append("; Generator: 7; 3\n; Schema: 0\n" + body)
        texts.append("; Version: 1.3\n" + body)
    for dv in [(1, 0), (1, 2), (1, 5), (1, 6), (1, 7), (0, 9), (2, 0)]:
        for k, t in enumerate(texts):
            o = outcome(lambda: sk.Assembler(default_version=dv).assemble(t).hex())
            recs["default_version"].append({"dv": list(dv), "text": k, "out": o})
    recs["texts"] = texts
    for k, m in enumerate(modules()):
        o = outcome(lambda: diag_list(sk.check_capability_closure(m["bytes"])))
        v = outcome(lambda: sk.diagnostics_text(sk.validate_module(m["bytes"])))
        recs["closure"].append({"module": k, "closure": o, "text": v})
    import corpus
    for name in ("minimal_kernel", "if_else_kernel", "iadd_kernel", "debug_heavy_kernel",
                 "wide_constant_kernel", "switch_kernel", "extinst_kernel"):
        scope = getattr(corpus, name)()
        recs["module_scope"].append({"name": name, "data": base64.b64encode(scope.to_bytes()).decode(),
                                     "diags": diag_list(sk.validate_module(scope))})
    with gzip.open(OUT, "wt", encoding="utf-8") as fh:
        json.dump(recs, fh)
    print(f"wrote {OUT}: {len(recs['default_version'])} default-version cases, "
          f"{len(recs['closure'])} closure cases, {len(recs['module_scope'])} ModuleScope cases")


if __name__ == "__main__":
    main()
