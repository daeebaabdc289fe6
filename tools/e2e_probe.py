"""Where the RoundTripSession e2e time goes (GPU box): whole-call wall time for
several pipeline depths and arena bounds on the bench's 1M-module batch.

usage: e2e_probe.py [modules] [chunks,...] [text_factor,...]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from paper_2305_09493_b200.asm import RoundTripSession
    from synth.families import sample_batch
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    chunk_list = [int(c) for c in (sys.argv[2] if len(sys.argv) > 2 else "8").split(",")]
    factors = [int(c) for c in (sys.argv[3] if len(sys.argv) > 3 else "6").split(",")]
    b = sample_batch(n, 10_000, 20261017)
    h = torch.from_numpy(b.data).pin_memory()
    for f in factors:
        RoundTripSession.TEXT_FACTOR = f
        for chunks in chunk_list:
            sess = RoundTripSession(chunks=chunks)
            sess.run(h, b.offsets, b.lengths)
            best = 1e9
            for _ in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                sess.run(h, b.offsets, b.lengths)
                best = min(best, time.perf_counter() - t0)
            sess.kernel_events = []
            sess.run(h, b.offsets, b.lengths)
            torch.cuda.synchronize()
            kd = sum(e0.elapsed_time(e1) for e0, e1, _ in sess.kernel_events)
            ka = sum(e1.elapsed_time(e2) for _, e1, e2 in sess.kernel_events)
            span = sess.kernel_events[0][0].elapsed_time(sess.kernel_events[-1][2])
            print(f"factor {f} chunks {chunks}: {best * 1e3:.1f} ms  {b.words / best / 1e9:.3f} Gw/s  "
                  f"kernels: disasm {kd:.1f} ms asm {ka:.1f} ms, first start -> last end {span:.1f} ms", flush=True)
            del sess
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
