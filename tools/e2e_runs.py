"""Run-to-run e2e times of RoundTripSession on the bench batch, with the allocator
segments each run adds (a cudaMalloc inside a run synchronises the pipeline)."""
import sys, time
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import torch
from paper_2305_09493_b200.asm import RoundTripSession
from synth.families import sample_batch
b = sample_batch(1_000_000, 10_000, 20261017)
h = torch.from_numpy(b.data).pin_memory()
# hold device memory like the bench does (the 1M batch + text + asm out)
hold = [torch.empty(int(3e9), dtype=torch.uint8, device="cuda"), torch.empty(int(9e9), dtype=torch.uint8, device="cuda"),
        torch.empty(int(3e9), dtype=torch.uint8, device="cuda")]
sess = RoundTripSession(chunks=8)
for k in range(8):
    torch.cuda.synchronize()
    s0 = torch.cuda.memory_stats()
    t0 = time.perf_counter()
    sess.run(h, b.offsets, b.lengths)
    dt = time.perf_counter() - t0
    s1 = torch.cuda.memory_stats()
    print(f"run {k}: {dt*1e3:.1f} ms  cudaMalloc retries {s1.get('num_alloc_retries',0)-s0.get('num_alloc_retries',0)} "
          f"segments +{s1.get('segment.all.allocated',0)-s0.get('segment.all.allocated',0)} "
          f"reserved {s1.get('reserved_bytes.all.current',0)/1e9:.1f} GB", flush=True)
