"""Where the RoundTripSession e2e time goes (GPU box): whole-call wall time for
several pipeline depths and arena bounds on the bench's 1M-module batch.

usage: e2e_probe.py [modules] [chunks,...] [text_factor,...] [taper a/b,...]"""
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
    tapers = [tuple(float(x) for x in t.split("/") if x) for t in
              (sys.argv[4] if len(sys.argv) > 4 else "0.5").split(",")]
    b = sample_batch(n, 10_000, 20261017)
    h = torch.from_numpy(b.data).pin_memory()
    for f, chunks, taper in [(f, c, t) for f in factors for c in chunk_list for t in tapers]:
        RoundTripSession.TEXT_FACTOR = f
        RoundTripSession.TAPER = taper
        if True:
            sess = RoundTripSession(chunks=chunks)
            sess.run(h, b.offsets, b.lengths)
            best = 1e9
            for _ in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                sess.run(h, b.offsets, b.lengths)
                best = min(best, time.perf_counter() - t0)
            sess.kernel_events = []
            ev_start = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ev_start.record()
            sess.run(h, b.offsets, b.lengths)
            t_call = (time.perf_counter() - t0) * 1e3
            torch.cuda.synchronize()
            head = ev_start.elapsed_time(sess.kernel_events[0][0])
            kd = sum(e0.elapsed_time(e1) for e0, e1, _ in sess.kernel_events)
            ka = sum(e1.elapsed_time(e2) for _, e1, e2 in sess.kernel_events)
            span = sess.kernel_events[0][0].elapsed_time(sess.kernel_events[-1][2])
            print(f"factor {f} chunks {chunks} taper {taper}: {best * 1e3:.1f} ms  {b.words / best / 1e9:.3f} Gw/s  "
                  f"kernels: disasm {kd:.1f} ms asm {ka:.1f} ms, first start -> last end {span:.1f} ms; "
                  f"this call {t_call:.1f} ms = head {head:.1f} + kernels {span:.1f} + tail "
                  f"{t_call - head - span:.1f}", flush=True)
            m0 = sess.marks[0][1]
            print("   host marks (ms): " + ", ".join(f"{k} {1e3 * (t - m0):.1f}" for k, t in sess.marks), flush=True)
            del sess
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
