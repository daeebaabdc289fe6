"""Per-call latency of the single-module public API on the GPU (one module per
call: H2D, launch, sync, D2H inside every call) against the reference's CPU
time for the same call on one core (configs[0]: the saxpy kernel).

usage: python tools/latency_probe.py [--calls N] [--family saxpy]
"""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def timeit(fn, calls):
    for _ in range(5):
        fn()
    t0 = time.perf_counter()
    for _ in range(calls):
        fn()
    return (time.perf_counter() - t0) / calls * 1e6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=300)
    ap.add_argument("--family", default="saxpy")
    args = ap.parse_args()
    from synth.families import build_module
    m = build_module(args.family, 0)
    import paper_2305_09493_b200 as sk
    text = sk.disassemble_module(m)
    rows = {
        "disassemble_module": lambda: sk.disassemble_module(m),
        "validate_module": lambda: sk.validate_module(m),
        "assemble_module": lambda: sk.assemble_module(text),
        "round trip": lambda: sk.assemble_module(sk.disassemble_module(m)),
    }
    ours = {k: timeit(f, args.calls) for k, f in rows.items()}
    ref = {}
    sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
    try:
        import spirvkit as R
        rrows = {
            "disassemble_module": lambda: R.disassemble_module(m),
            "validate_module": lambda: R.validate_module(m),
            "assemble_module": lambda: R.assemble_module(text),
            "round trip": lambda: R.assemble_module(R.disassemble_module(m)),
        }
        ref = {k: timeit(f, max(20, args.calls // 10)) for k, f in rrows.items()}
    except ImportError as exc:
        print(f"reference not importable: {exc}")
    print(f"{args.family}: {len(m) // 4} words, {len(text)} text bytes")
    for k in rows:
        r = ref.get(k)
        print(f"{k:20s} gpu {ours[k]:9.1f} us/call   reference (1 core) "
              + (f"{r:9.1f} us/call   ratio {r / ours[k]:6.2f}x" if r else "n/a"))


if __name__ == "__main__":
    main()
