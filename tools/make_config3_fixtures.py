"""Record full-size config-3 fixtures: SHA-256 + length of

* the REFERENCE's own ``validate_module`` -> ``diagnostics_text`` output,
* the REFERENCE's own ``disassemble_module(inline_names=False)`` text,
* the oracle's linear closed-form ``inline_names=True`` text (the reference's
  ``_assign_refs`` fixpoint is O(n^2) here: infeasible on a CPU),

for the ~91M-word module ``synth.huge.build_huge(55000)``.  Build container
only (needs /root/reference); each leg runs in its own process (RAM-heavy:
tens of GB), the results are merged into ``tests/golden/config3_<n_fn>.json``.
A mid-size module (n_fn = 640, just above the 2^20-word threshold of the
grid-wide large-module kernels) is recorded the same way for a quicker test.

usage: python tools/make_config3_fixtures.py [n_fn] [leg ...]
       legs: ref_validate ref_disasm_numeric oracle_disasm_named (default), and the same
       with a _mut suffix for the mutated module (mutate(): duplicate result ids and
       unknown opcodes)
"""

from __future__ import annotations

import hashlib
import json
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
LEGS = ("ref_validate", "ref_disasm_numeric", "oracle_disasm_named",
        "ref_validate_mut", "ref_disasm_numeric_mut", "oracle_disasm_named_mut")


def mutate(m: bytes) -> bytes:
    """Seeded mutations of the config-3 module that keep every word count: some
    OpIAdd results re-define the previous OpIAdd's result (DuplicateResultId), some
    opcodes become unknown (UnknownOpcode; OpUnknown(N) in the disassembly)."""
    import numpy as np
    w = np.frombuffer(m, dtype="<u4").copy()
    pos, starts = 5, []
    while pos < len(w):
        starts.append(pos)
        pos += int(w[pos] >> 16)
    starts = np.array(starts)
    iadd = starts[w[starts] == ((5 << 16) | 128)]
    for k in range(1, len(iadd), 997):
        w[iadd[k] + 2] = w[iadd[k - 1] + 2]
    for k in range(5, len(iadd), 1499):
        w[iadd[k]] = (5 << 16) | 0xFFF0
    return w.tobytes()


def _digest(text: str) -> dict:
    data = text.encode("utf-8")
    return {"sha256": hashlib.sha256(data).hexdigest(), "bytes": len(data),
            "lines": text.count("\n")}


def run_leg(n_fn: int, leg: str) -> dict:
    sys.path.insert(0, str(ROOT))
    from synth.huge import build_huge
    m = build_huge(n_fn)
    if leg.endswith("_mut"):
        m = mutate(m)
        leg = leg[:-4]
    t0 = time.time()
    if leg.startswith("ref_"):
        sys.path.insert(0, "/root/reference/pkg/src")
        import spirvkit as ref
        if leg == "ref_validate":
            out = ref.diagnostics_text(ref.validate_module(m))
        else:
            out = ref.disassemble_module(m, ref.DisassemblerOptions(inline_names=False))
    else:
        from oracle import disasm as odis
        out = odis.disassemble(m)
    rec = _digest(out)
    rec.update(seconds=round(time.time() - t0, 1), words=len(m) // 4,
               module_sha256=hashlib.sha256(m).hexdigest())
    return rec


def main():
    args = sys.argv[1:]
    if args and args[0] == "--leg":
        print(json.dumps(run_leg(int(args[1]), args[2])), flush=True)
        return
    n_fn = int(args[0]) if args else 55000
    legs = args[1:] or list(LEGS[:3])
    out = GOLDEN / f"config3_{n_fn}.json"
    res = json.loads(out.read_text()) if out.exists() else {}
    res["n_fn"] = n_fn
    res["generator"] = "synth.huge.build_huge(n_fn) (chain=200, seed=1)"
    procs = {leg: subprocess.Popen([sys.executable, __file__, "--leg", str(n_fn), leg],
                                   stdout=subprocess.PIPE, text=True, cwd=ROOT) for leg in legs}
    for leg, p in procs.items():
        line = p.communicate()[0].strip().splitlines()
        if p.returncode != 0 or not line:
            print(f"{leg}: failed (rc {p.returncode})", file=sys.stderr)
            continue
        res[leg] = json.loads(line[-1])
        print(leg, res[leg], flush=True)
        out.write_text(json.dumps(res, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
