"""Single-module calls: one-warp batch path vs the grid-wide large-module path
(skg_disasm_large / skg_validate_large) by module size, to place
_native.LARGE_MODULE_WORDS at the crossover.  Both outputs are compared.

usage: python tools/large_threshold_probe.py
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def per_call(fn, reps):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e3


def main():
    from synth.families import build_module
    from synth.huge import build_huge
    from paper_2305_09493_b200 import _native
    from paper_2305_09493_b200.disasm import DisassemblerOptions, option_bits
    opts = option_bits(DisassemblerOptions())
    mods = [("saxpy", build_module("saxpy", 0))]
    for nfn, chain, s in ((1, 20, ()), (4, 50, ()), (8, 200, (1,)), (32, 200, (1,)), (128, 200, (1, 8)),
                          (512, 200, (1, 8)), (2048, 200, (1, 8, 64))):
        mods.append((f"huge({nfn},{chain})", build_huge(nfn, chain=chain, string_kib=s)))
    print(f"{'module':18s} {'words':>9s} | disasm batch / large ms | validate batch / large ms")
    for name, m in mods:
        b = _native.DeviceBatch.from_modules([m])
        W = len(m) // 4
        reps = 20 if W < 200000 else 3
        db = lambda: _native.fetch_texts(_native.run_disasm(b, opts, None, None), 1)[0]
        dl = lambda: _native._disasm_large(b, 0, len(m), opts, None, None)
        vb = lambda: _native.fetch_texts(_native.run_validate(b, None), 1)[0]
        vl = lambda: _native._validate_large(b, 0, len(m), None)
        same_d = bytes(db()) == bytes(dl())
        same_v = bytes(vb()) == bytes(vl())
        print(f"{name:18s} {W:9d} | {per_call(db, reps):8.3f} / {per_call(dl, reps):8.3f} "
              f"{'=' if same_d else 'DIFF'} | {per_call(vb, reps):8.3f} / {per_call(vl, reps):8.3f} "
              f"{'=' if same_v else 'DIFF'}", flush=True)


if __name__ == "__main__":
    main()
