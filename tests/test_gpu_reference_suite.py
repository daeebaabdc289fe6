"""Conformance: the reference's own test files (pkg/tests/test_{codec,disasm,asm,
validate,acceptance,cli}.py, copied to oracle/_ref/ref_tests by __graft_entry__.build)
run with every hot-path name bound to this package (tests/refsuite/refsuite_plugin.py):
decode / encode / disassemble / format / validate / tokenize / assemble all go
through the CUDA kernels; the reference builder only constructs inputs.

Expected: every test passes except the two the reference itself fails by design
(test_output.txt: criterion 1 counts generated 1.2 artefacts, criterion 5 expects
another cycle count -- neither touches the codec path).  The per-test outcome is
written to gpurun_out/refsuite_results.txt when that directory exists."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
SUITE = ROOT / "oracle" / "_ref" / "ref_tests"
FILES = ["test_codec.py", "test_disasm.py", "test_asm.py", "test_validate.py", "test_acceptance.py", "test_cli.py"]
FAIL_BY_DESIGN = {"test_acceptance.py::test_criterion_1_generator_counts",
                  "test_acceptance.py::test_criterion_5_capability_cycles"}


def test_reference_suite_on_the_gpu_path():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not (SUITE / "corpus.py").exists():
        pytest.skip("reference suite not staged (oracle/_ref/ref_tests: __graft_entry__.build())")
    env = dict(os.environ, SKG_REPO_ROOT=str(ROOT), PYTHONDONTWRITEBYTECODE="1",
               PYTHONPATH=os.pathsep.join([str(ROOT / "tests" / "refsuite"), str(SUITE)]))
    out = subprocess.run([sys.executable, "-m", "pytest", "-p", "refsuite_plugin", "-p", "no:cacheprovider",
                          "-rA", "-q", *FILES], cwd=SUITE, env=env, capture_output=True, text=True, timeout=1800)
    lines = out.stdout.splitlines()
    res = {}
    for ln in lines:
        for tag in ("PASSED", "FAILED", "ERROR", "SKIPPED"):
            if ln.startswith(tag + " "):
                res[ln.split()[1]] = tag
    rep = ROOT / "gpurun_out"
    if rep.is_dir():
        (rep / "refsuite_results.txt").write_text("\n".join(f"{v} {k}" for k, v in sorted(res.items())) + "\n"
                                                  + "\n".join(lines[-5:]) + "\n")
    assert res, out.stdout[-3000:] + out.stderr[-3000:]
    failed = {k for k, v in res.items() if v in ("FAILED", "ERROR")}
    assert failed <= FAIL_BY_DESIGN, (sorted(failed - FAIL_BY_DESIGN), out.stdout[-6000:])
    passed = sum(v == "PASSED" for v in res.values())
    assert passed >= 80, passed
