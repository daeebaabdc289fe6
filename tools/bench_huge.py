"""Config 3: disassembly + validation of ONE large module (synth/huge.py) on
cuda:0, inputs resident in HBM; prints words/s for each kernel.

usage: python tools/bench_huge.py <n_functions> [chain] [--batch-path]   (~1660 words per function)
       (--batch-path also times the one-warp batch kernels on the same module)
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    n_fn = int(args[0]) if len(args) > 0 else 5000
    chain = int(args[1]) if len(args) > 1 else 200
    import numpy as np
    import torch
    from paper_2305_09493_b200 import _native
    from synth.huge import build_huge
    t0 = time.time()
    m = build_huge(n_fn, chain)
    W = len(m) // 4
    print(f"module: {W} words, {len(m) / 1e6:.1f} MB (built in {time.time() - t0:.1f}s)", flush=True)
    data = np.frombuffer(m + b"\0" * 16, dtype=np.uint8)
    dev = _native.DeviceBatch.from_host(data, np.array([0], np.int64), np.array([len(m)], np.int64))
    from paper_2305_09493_b200 import decode_module
    for rep in range(2):   # decode_module end to end (host bytes in, host objects out; 2nd run timed)
        t2 = time.time()
        h, insts = decode_module(m)
        if rep:
            print(f"decode_module (tiled boundary pass, incl. H2D/D2H + Python objects): "
                  f"{len(insts)} instructions {time.time() - t2:.2f} s", flush=True)
    from paper_2305_09493_b200 import _native as nat
    dd = torch.frombuffer(bytearray(m + b"\0" * 16), dtype=torch.uint8).cuda()
    nat._run_decode_large(dd, len(m))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    nat._run_decode_large(dd, len(m))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"decode (skg_decode_large, device + result copies): {ms:.1f} ms {W / ms / 1e3:.1f} Mwords/s",
          flush=True)
    for rep in range(2):   # validate, whole GPU on the one module (skg_validate_large), device-resident
        torch.cuda.synchronize()
        t3 = time.time()
        r = nat._validate_large(dev, 0, len(m), None)
        torch.cuda.synchronize()
        if rep:
            print(f"validate (skg_validate_large, grid-wide, incl. host syncs): {time.time() - t3:.3f} s "
                  f"{W / (time.time() - t3) / 1e6:.1f} Mwords/s -> {len(r) if isinstance(r, bytes) else r}",
                  flush=True)
    from paper_2305_09493_b200.disasm import DisassemblerOptions, option_bits
    for rep in range(2):   # disassembly, whole GPU on the one module (skg_disasm_large), device-resident
        torch.cuda.synchronize()
        t4 = time.time()
        r = nat._disasm_large(dev, 0, len(m), option_bits(DisassemblerOptions()), None, None)
        torch.cuda.synchronize()
        if rep:
            dt = time.time() - t4
            print(f"disasm (skg_disasm_large, grid-wide, default options, incl. host syncs + text D2H): "
                  f"{dt:.3f} s {W / dt / 1e6:.1f} Mwords/s -> {len(r) if isinstance(r, bytes) else r} bytes",
                  flush=True)
    if "--batch-path" not in sys.argv:
        return
    for kind in ("disasm", "validate"):
        plan = _native.DisasmPlan(dev, 2, kind=kind, text_cap=24 * len(m) + 4096)
        t1 = time.time()
        info = plan.fit()
        st = int(plan.status[0].item())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.launch()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"{kind}: status {st} out {info['text_bytes']} B  {ms:.1f} ms  {W / ms / 1e3:.2f} Mwords/s "
              f"(fit {time.time() - t1:.1f}s)", flush=True)


if __name__ == "__main__":
    main()
