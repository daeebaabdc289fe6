"""Per-phase cycle breakdown of skg_asm (debug build with -DSKG_PHASE_TIMING).

Builds paper_2305_09493_b200/libskgpu_timing.so and runs the assembler over a
disassembled synthetic batch; prints the share of warp-cycles per phase."""
import ctypes
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
LIB = ROOT / "paper_2305_09493_b200" / "libskgpu_timing.so"
PH = ["A split", "alloc+init", "B tokenize", "C header", "D results", "E opname/widths", "F encode1",
      "G state", "H layout", "I write"]


def build():
    import __graft_entry__ as g
    cmd = [g._nvcc(), *g.NVCC_FLAGS, "-DSKG_PHASE_TIMING", "-o", str(LIB), str(g.CSRC / "skg_api.cu")]
    subprocess.run(cmd, check=True)


def main():
    if "--build" in sys.argv:
        build()
        return
    os.environ["SKGPU_LIB"] = str(LIB)
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
    import torch
    from paper_2305_09493_b200 import _native
    from synth.families import sample_batch
    b = sample_batch(n, min(n, 10000), 20261017)
    dev = _native.DeviceBatch.from_host(b.data, b.offsets, b.lengths)
    plan = _native.DisasmPlan(dev, 2)
    plan.fit()
    mx = int(plan.span[1::2].max().item())
    tb = _native.DeviceBatch(plan.text, plan.span[0::2], plan.span[1::2], (mx + 3) // 4, 0)
    tb.n = dev.n
    ap = _native.AsmPlan(tb, out_cap=int(b.lengths.sum()) + 64 * dev.n + 4096, stride=2)
    ap.fit()
    torch.cuda.synchronize()
    L = _native.lib()
    L.skg_debug_asm_phases.argtypes = [ctypes.c_void_p]
    arr = (ctypes.c_ulonglong * 16)()
    L.skg_debug_asm_phases(arr)
    tot = sum(arr) or 1
    for k, name in enumerate(PH):
        print(f"{name:18s} {100 * arr[k] / tot:6.2f}%  {arr[k] / n:12.0f} cycles/module")


if __name__ == "__main__":
    main()
