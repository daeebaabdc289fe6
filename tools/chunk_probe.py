"""Device time of the batch kernels over the bench's 1M-module batch launched
whole vs. as K launches over contiguous module ranges (same device buffers;
inputs resident).  Question: is the whole-batch launch slower than the sum of
per-range launches (memory locality of the size-sorted order over GBs)?

usage: python tools/chunk_probe.py [modules] [K,...]
"""
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from paper_2305_09493_b200 import _native
    from paper_2305_09493_b200.disasm import DisassemblerOptions, option_bits
    from synth.families import sample_batch
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    ks = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,4,12,32").split(",")]
    b = sample_batch(n, 10_000, 20261017)
    dev = _native.DeviceBatch.from_host(b.data, b.offsets, b.lengths)
    opts = option_bits(DisassemblerOptions())
    for K in ks:
        cuts = np.linspace(0, n, K + 1).astype(int)
        plans = []
        for a, c in zip(cuts[:-1], cuts[1:]):
            lens = b.lengths[a:c]
            mwf = float(os.environ.get("MAXW_FACTOR", "1"))   # experiments: scratch slot spacing
            sub = _native.DeviceBatch(dev.data, dev.off[a:c], dev.len[a:c], int(int(lens.max()) // 4 * mwf),
                                      int(lens.sum()))
            dp = _native.DisasmPlan(sub, opts)
            dp.fit()
            mt = int(dp.span[1::2].max().item())
            tb = _native.DeviceBatch(dp.text, dp.span[0::2], dp.span[1::2], (mt + 3) // 4, 0)
            tb.n = c - a
            slot = int(os.environ.get("SLOT_KB", "0")) * 1024 or None
            ap = _native.AsmPlan(tb, out_cap=int(lens.sum()) + 64 * (c - a) + 4096, stride=2, slot_bytes=slot)
            ap.fit()
            st = ap.status[: c - a].cpu().numpy()
            print(f"   asm slot {ap.slot} B, {(st == _native.ST_INTERNAL).sum()} modules over it, "
                  f"{(st != 0).sum()} not ok", flush=True)
            plans.append((dp, ap))
        best_d = best_a = 1e9
        for _ in range(4):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record()
            for dp, _ in plans:
                dp.launch()
            e[1].record()
            for _, ap in plans:
                ap.launch()
            e[2].record()
            torch.cuda.synchronize()
            best_d = min(best_d, e[0].elapsed_time(e[1]))
            best_a = min(best_a, e[1].elapsed_time(e[2]))
        print(f"K={K:3d}: disasm {best_d:7.1f} ms  asm {best_a:7.1f} ms  sum {best_d + best_a:7.1f} ms "
              f"({b.words / (best_d + best_a) / 1e6:.3f} Gw/s)", flush=True)
        del plans
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
