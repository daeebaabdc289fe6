"""Both code paths of the phases that run across a CTA's modules (cta_dispatch: the
assembler's encode pass 1, the validator's V2 / V3 walks) give the reference's
outputs: the default whole-CTA barrier group takes the cross-module path, barrier
groups of 8 warps (SKG_*_GROUP, read per launch) take the per-module loops.  Also
the synthetic families round-trip identically on both paths at a batch size that
fills every CTA."""

import pytest

from golden_io import asm_texts, modules, same

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2305_09493_b200 as sk
    return sk


def _asm_outcome(r):
    if isinstance(r, BaseException):
        return {"exc": [type(r).__name__, str(r)]}
    return {"ok": r.hex()}


def _val_outcome(r):
    if isinstance(r, BaseException):
        return {"exc": [type(r).__name__, str(r)]}
    return {"ok": [[d.severity, d.code, d.location, d.message] for d in r]}


@pytest.mark.parametrize("group", [None, "8"])
def test_assembler_paths(sk, monkeypatch, group):
    if group:
        monkeypatch.setenv("SKG_ASM_GROUP", group)
    recs = asm_texts()
    got = sk.assemble_batch([r["text"] for r in recs])
    bad = [r["name"] for r, g in zip(recs, got) if not same(_asm_outcome(g), r["asm"])]
    assert not bad, bad[:10]


@pytest.mark.parametrize("group", [None, "8"])
def test_validator_paths(sk, monkeypatch, group):
    if group:
        monkeypatch.setenv("SKG_VAL_GROUP", group)
    recs = modules()
    got = sk.validate_batch([r["bytes"] for r in recs])
    bad = [r["name"] for r, g in zip(recs, got) if not same(_val_outcome(g), r["validate"])]
    assert not bad, bad[:10]


def test_paths_agree_on_a_full_grid(sk, monkeypatch):
    """20k family modules (every SM's CTA full of modules, most sharing instructions):
    assembled and validated on both paths, equal results; binaries equal the inputs."""
    from synth.families import sample_batch
    b = sample_batch(20000, 500, 99)
    mods = [b.module(i) for i in range(b.n)]
    texts = sk.disassemble_batch(mods)
    out = {}
    for group in (None, "8"):
        if group:
            monkeypatch.setenv("SKG_ASM_GROUP", group)
            monkeypatch.setenv("SKG_VAL_GROUP", group)
        out[group] = (sk.assemble_batch(texts), [str(x) for x in sk.validate_batch(mods)])
    assert out[None] == out["8"]
    assert all(a == m for a, m in zip(out[None][0], mods))
