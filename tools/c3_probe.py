"""Host-side timing of the config-3 step parts (disassembly, validation) on the GPU box."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch
    from paper_2305_09493_b200 import _native
    from paper_2305_09493_b200.disasm import DisassemblerOptions, option_bits
    from synth.huge import build_huge
    m = build_huge(int(sys.argv[1]) if len(sys.argv) > 1 else 55000)
    data = np.frombuffer(m + b"\0" * 16, dtype=np.uint8)
    dev = _native.DeviceBatch.from_host(data, np.array([0], np.int64), np.array([len(m)], np.int64))
    opts = option_bits(DisassemblerOptions())
    for it in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _native._disasm_large(dev, 0, len(m), opts, None, None, view=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        _native._validate_large(dev, 0, len(m), None)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"iter {it}: disasm {1e3 * (t1 - t0):.1f} ms  validate {1e3 * (t2 - t1):.1f} ms", flush=True)


if __name__ == "__main__":
    main()
