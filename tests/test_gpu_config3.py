"""Config 3 at its configured size (BASELINE.json configs[2]):
one ~91M-word module (synth/huge.py, OpName on every id, long OpStrings, ids
up to ~1.1e7) disassembled and validated on the GPU through the public API,
which routes modules of 2^20 words and more to the grid-wide kernels
(skg_disasm_large / skg_validate_large) -- no monkeypatched thresholds.

The expected outputs are SHA-256 digests recorded in the build container by
tools/make_config3_fixtures.py:

* validation and ``inline_names=False`` disassembly: the REFERENCE's own
  ``validate_module`` / ``disassemble_module`` run over the full module;
* ``inline_names=True`` disassembly: the oracle's linear closed form of
  ``_assign_refs`` (the reference's fixpoint is O(n^2) here).

A mid-size module (640 functions, ~1.1M words, just above the threshold) is
pinned the same way and runs first.
"""

import hashlib
import json
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).parent / "golden"


def _fixture(n_fn):
    p = GOLDEN / f"config3_{n_fn}.json"
    if not p.exists():
        pytest.skip(f"{p.name} not recorded")
    return json.loads(p.read_text())


@pytest.fixture(scope="module")
def sk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2305_09493_b200 as sk
    return sk


def _digest(text):
    data = text.encode("utf-8") if isinstance(text, str) else bytes(text)
    return hashlib.sha256(data).hexdigest(), len(data)


@pytest.mark.parametrize("n_fn,mut", [(640, ""), (640, "_mut"), (55000, ""), (55000, "_mut")])
def test_config3_full_size(sk, n_fn, mut):
    """mut: the seeded mutations of tools/make_config3_fixtures.mutate (duplicate result
    ids, unknown opcodes): validation reports them, disassembly renders OpUnknown."""
    from paper_2305_09493_b200 import _native
    from synth.huge import build_huge
    fx = _fixture(n_fn)
    if "ref_validate" + mut not in fx:
        pytest.skip(f"config3_{n_fn}.json has no {mut or 'plain'} records")
    m = build_huge(n_fn)
    if mut:
        import sys
        sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
        from make_config3_fixtures import mutate
        m = mutate(m)
    assert hashlib.sha256(m).hexdigest() == fx["ref_validate" + mut]["module_sha256"]
    assert len(m) // 4 >= _native.LARGE_MODULE_WORDS        # the grid-wide kernels, not the warp path
    diags = sk.validate_module(m)
    text = sk.diagnostics_text(diags)
    assert _digest(text) == (fx["ref_validate" + mut]["sha256"], fx["ref_validate" + mut]["bytes"])
    got = sk.disassemble_module(m, sk.DisassemblerOptions(inline_names=False))
    want = fx["ref_disasm_numeric" + mut]
    assert _digest(got) == (want["sha256"], want["bytes"])
    del got
    got = sk.disassemble_module(m)
    want = fx["oracle_disasm_named" + mut]
    assert _digest(got) == (want["sha256"], want["bytes"])
    del got
    # the fused entry point: the text's host copy overlaps the validation kernels
    t, v = sk.disassemble_validate_batch([m])[0]
    assert _digest(t) == (want["sha256"], want["bytes"])
    assert _digest(sk.diagnostics_text(v)) == (fx["ref_validate" + mut]["sha256"], fx["ref_validate" + mut]["bytes"])
