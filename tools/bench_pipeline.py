"""Config 5 on one GPU: the full decode / validate / encode pipeline over a batch
of synthetic modules resident in HBM -- skg_validate + skg_disasm + skg_asm per
step (the assembler reads the disassembler's text arena directly), bit-identical
re-assembly checked.  Per-GPU shard of the multi-GPU configuration (modules
shard with no collective; see paper_2305_09493_b200/shard.py).

usage: python tools/bench_pipeline.py [n_modules] [steps]
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    import torch
    from paper_2305_09493_b200 import _native
    from paper_2305_09493_b200.disasm import DisassemblerOptions, option_bits
    from synth.families import sample_batch
    t0 = time.time()
    b = sample_batch(n, 10_000, 20261017)
    print(f"batch: {b.n} modules, {b.words} words ({time.time() - t0:.1f}s)", flush=True)
    dev = _native.DeviceBatch.from_host(b.data, b.offsets, b.lengths)
    val = _native.DisasmPlan(dev, 0, kind="validate")
    vinfo = val.fit()
    dis = _native.DisasmPlan(dev, option_bits(DisassemblerOptions()))
    dinfo = dis.fit()
    mx = int(dis.span[1::2].max().item())
    tb = _native.DeviceBatch(dis.text, dis.span[0::2], dis.span[1::2], (mx + 3) // 4, 0)
    tb.n = dev.n
    asm = _native.AsmPlan(tb, out_cap=int(b.lengths.sum()) + 64 * dev.n + 4096, stride=2)
    asm.fit()
    assert (asm.span[1: 2 * dev.n: 2].cpu().numpy() == b.lengths).all()
    fus = _native.DisasmPlan(dev, option_bits(DisassemblerOptions()), kind="pipeline", text_cap=dis.cap)
    fus.launch()
    finfo = fus.check()
    assert not finfo["overflow"] and finfo["vtext_bytes"] == 0, finfo
    for _ in range(2):
        val.launch(); dis.launch(); asm.launch(); fus.launch()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    tv = td = ta = 0.0
    for _ in range(steps):
        ev[0].record(); val.launch(); ev[1].record(); dis.launch(); ev[2].record(); asm.launch(); ev[3].record()
        torch.cuda.synchronize()
        tv += ev[0].elapsed_time(ev[1]); td += ev[1].elapsed_time(ev[2]); ta += ev[2].elapsed_time(ev[3])
    tv, td, ta = tv / steps, td / steps, ta / steps
    ev[0].record()
    for _ in range(steps):
        fus.launch()
    ev[1].record()
    torch.cuda.synchronize()
    tf = ev[0].elapsed_time(ev[1]) / steps
    W = b.words
    print(f"validate {tv:.1f} ms ({W / tv / 1e6:.2f} Gwords/s, diagnostics {vinfo['text_bytes']} B)\n"
          f"disasm   {td:.1f} ms ({W / td / 1e6:.2f} Gwords/s, text {dinfo['text_bytes']} B)\n"
          f"asm      {ta:.1f} ms ({W / ta / 1e6:.2f} Gwords/s)\n"
          f"fused validate+disasm (skg_disasm_validate) {tf:.1f} ms vs {tv + td:.1f} ms separate\n"
          f"pipeline {tv + td + ta:.1f} ms/step: {W / (tv + td + ta) / 1e6:.2f} Gwords/s per GPU "
          f"(each word validated, disassembled and re-assembled)", flush=True)


if __name__ == "__main__":
    main()
