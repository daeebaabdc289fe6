"""Profiling driver: launch the batch disassembler / validator a few times.

ncu --set full --import-source on -k regex:disasm_kernel -s 2 -c 1 \
    -o gpurun_out/prof python tools/prof_disasm.py --modules 50000
"""

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--modules", type=int, default=50000)
    ap.add_argument("--variants", type=int, default=10000)   # the bench batch's diversity
    ap.add_argument("--launches", type=int, default=4)
    ap.add_argument("--kind", default="disasm", choices=["disasm", "validate", "asm", "pipeline"])
    ap.add_argument("--opts", type=int, default=2)
    args = ap.parse_args()
    import torch
    from paper_2305_09493_b200 import _native
    from synth.families import sample_batch
    b = sample_batch(args.modules, args.variants, 20261017)
    dev = _native.DeviceBatch.from_host(b.data, b.offsets, b.lengths)
    plan = _native.DisasmPlan(dev, args.opts, kind="disasm" if args.kind == "asm" else args.kind)
    plan.fit()
    if args.kind == "asm":   # assemble the disassembled text (stride-2 spans)
        mx = int(plan.span[1::2].max().item())
        tb = _native.DeviceBatch(plan.text, plan.span[0::2], plan.span[1::2], (mx + 3) // 4, 0)
        tb.n = dev.n
        plan = _native.AsmPlan(tb, out_cap=int(b.lengths.sum()) + 64 * dev.n + 4096, stride=2)
        plan.fit()
        assert (plan.status[: dev.n] == 0).all().item()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(args.launches):
        plan.launch()
    end.record()
    torch.cuda.synchronize()
    ms = start.elapsed_time(end) / args.launches
    print(f"{args.kind}: {b.n} modules {b.words} words: {ms:.3f} ms/launch "
          f"{b.words / ms / 1e6:.3f} Gwords/s", flush=True)


if __name__ == "__main__":
    main()
