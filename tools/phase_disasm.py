"""Per-phase cycle breakdown + quick timing of skg_disasm.

  python tools/phase_disasm.py --build          # build libskgpu_timing.so (-DSKG_PHASE_TIMING)
  python tools/phase_disasm.py phases [N]       # per-phase share of warp-cycles (timing build)
  python tools/phase_disasm.py time [N] [opts]  # CUDA-event time of the normal build
"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
LIB = ROOT / "paper_2305_09493_b200" / "libskgpu_timing.so"
PH = ["P0 load+boundary", "P1 tables+prescan", "P2 classify", "P3 errors", "P4 names",
      "P5 refs+size", "P6 write"]


def build():
    import __graft_entry__ as g
    cmd = [g._nvcc(), *g.NVCC_FLAGS, "-DSKG_PHASE_TIMING", "-o", str(LIB), str(g.CSRC / "skg_api.cu")]
    subprocess.run(cmd, check=True)


def batch(n):
    import numpy as np
    from paper_2305_09493_b200 import _native
    from synth.families import sample_batch
    if n < 0:   # one config-3 module of -n functions (synth/huge.py)
        from synth.huge import build_huge
        m = build_huge(-n)

        class B:
            words = len(m) // 4
        data = np.frombuffer(m + b"\0" * 16, dtype=np.uint8)
        return B, _native.DeviceBatch.from_host(data, np.array([0], np.int64), np.array([len(m)], np.int64))
    b = sample_batch(n, min(n, 10000), 20261017)
    return b, _native.DeviceBatch.from_host(b.data, b.offsets, b.lengths)


def main():
    if "--build" in sys.argv:
        build()
        return
    mode = sys.argv[1] if len(sys.argv) > 1 else "phases"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
    opts = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    if mode == "phases":
        os.environ["SKGPU_LIB"] = str(LIB)
    import ctypes
    import torch
    from paper_2305_09493_b200 import _native
    b, dev = batch(n)
    plan = _native.DisasmPlan(dev, opts)
    info = plan.fit()
    torch.cuda.synchronize()
    if mode == "phases":
        L = _native.lib()
        L.skg_debug_disasm_phases.argtypes = [ctypes.c_void_p]
        arr = (ctypes.c_ulonglong * 16)()
        L.skg_debug_disasm_phases(arr)
        tot = sum(arr) or 1
        for k, name in enumerate(PH):
            print(f"{name:20s} {100 * arr[k] / tot:6.2f}%  {arr[k] / abs(n):12.0f} warp-cycles/module")
        return
    for _ in range(3):
        plan.launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = 5
    e0.record()
    for _ in range(k):
        plan.launch()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    print(f"disasm n={n} words={b.words} text={info['text_bytes']} {ms:.3f} ms "
          f"{b.words / ms / 1e6:.3f} Gwords/s env={{{', '.join(f'{k}={v}' for k, v in os.environ.items() if k.startswith('SKG_'))}}}")


if __name__ == "__main__":
    main()
