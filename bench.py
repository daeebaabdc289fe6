"""Benchmark: SPIR-V words/s disassembled + assembled on B200 (BASELINE.json
configs[1] disassembly and configs[3] assembler round trip of the same batch).

Workload (N=1): a batch of 1,000,000 synthetic modules drawn (seeded) from
10,000 builder-canonical variants of the paper's benchmark kernels (saxpy,
matmul, DFT, n-body, Black-Scholes; synth/families.py).  One step = the CUDA
disassembler (skg_disasm, default options) over the whole batch followed by the
CUDA assembler (skg_asm) over the produced text, back to binaries that must be
bit-identical to the input; inputs resident in HBM.  value = words per step /
step time (each word is disassembled once and assembled once).  N>1 (torchrun,
one process per GPU): every rank round-trips its own 1M-module batch (weak
scaling, no collective on the data path); value = all ranks' words /
max-over-ranks time.

Extra keys: roofline (HBM; algorithmic bytes 4W+T per launch for either
kernel; the dominant kernel is reported, both are listed), cpu_baseline (the
reference's own CPU implementation, oracle/_ref, timed on this box's host cores
on a bounded sample), e2e (host buffers through RoundTripSession: pinned H2D of
the binaries + both kernels + D2H of the text and the binaries, pipelined over
16 module chunks on three streams), gpu_launches,
clocks.

``--impl reference`` times the reference's CPU implementation instead (rank 0
only, all host cores, bounded sample per step) and prints the same JSON line
with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SPIR-V words/sec disassembled+assembled (1/2/4/8 B200); % of HBM roofline"
SEED = 20261017


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# -- CPU reference (bounded sample) ------------------------------------------------
_REF_MOD = None


def _ref_init():
    global _REF_MOD
    ref = ROOT / "oracle" / "_ref"
    if (ref / "spirvkit").is_dir():
        sys.path.insert(0, str(ref))
        import spirvkit
        _REF_MOD = ("reference", spirvkit.disassemble_module, spirvkit.assemble_module)
    else:
        from oracle import asm as oasm, disasm as odis
        _REF_MOD = ("port", odis.disassemble, oasm.assemble)


def _ref_work(mods):
    dis, asm = _REF_MOD[1], _REF_MOD[2]
    words = 0
    for m in mods:
        back = asm(dis(m))
        assert back == m
        words += len(m) // 4
    return words


def ref_kind():
    return "reference" if (ROOT / "oracle" / "_ref" / "spirvkit").is_dir() else "port"


class CpuReference:
    """The reference disassembler + assembler on all host cores (multiprocessing).

    Workers are spawned (fresh interpreters), not forked: a fork of the GPU arm's
    process would carry its CUDA context, pinned buffers and the 1M-module batch,
    and ran measurably slower than the driver's reference arm."""

    def __init__(self, cores=None):
        import multiprocessing as mp
        self.cores = cores or len(os.sched_getaffinity(0))
        self.pool = mp.get_context("spawn").Pool(self.cores, initializer=_ref_init)

    def run(self, mods):
        chunks = [mods[i::self.cores] for i in range(self.cores)]
        t0 = time.perf_counter()
        words = sum(self.pool.map(_ref_work, chunks))
        return words, time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()


def sample_modules(batch, n):
    idx = np.linspace(0, batch.n - 1, num=min(n, batch.n)).astype(np.int64)
    return [batch.module(int(i)) for i in idx]


# -- clocks ------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        sm = [float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for k, name in enumerate(names):
                if len(s) > 3 + k and s[3 + k].lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:  # noqa: BLE001
            pass
    return 6650.0, "fallback"


def profile_traffic():
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:  # noqa: BLE001
            return None
    return None


def _issue_roofline(inst, ms):
    if not inst or not ms:
        return None
    peak = 148 * 4 * 1.965e9
    ach = inst / (ms / 1e3)
    return {"warp_inst_per_launch": inst, "achieved_warp_inst_per_s": ach, "peak_warp_inst_per_s": peak,
            "frac": ach / peak, "source": "profiles/traffic.json (ncu smsp__inst_executed.sum)"}


# -- the GPU arm ---------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    from paper_2305_09493_b200 import _native
    from paper_2305_09493_b200.asm import RoundTripSession
    from paper_2305_09493_b200.disasm import DisassemblerOptions, option_bits
    from synth.families import sample_batch

    t0 = time.perf_counter()
    batch = sample_batch(args.modules, args.variants, SEED + rank)
    words = batch.words
    log(f"[rank {rank}] batch: {batch.n} modules, {words} words, {batch.data.nbytes} bytes "
        f"({time.perf_counter() - t0:.1f}s)")
    dev = _native.DeviceBatch.from_host(batch.data, batch.offsets, batch.lengths)
    plan = _native.DisasmPlan(dev, option_bits(DisassemblerOptions()))
    info = plan.fit()
    status = plan.status[: dev.n].cpu().numpy()
    assert info["errors"] == 0 and not info["overflow"] and (status == 0).all(), info
    text_bytes = info["text_bytes"]
    max_text = int(plan.span[1::2].max().item())
    tb = _native.DeviceBatch(plan.text, plan.span[0::2], plan.span[1::2], (max_text + 3) // 4, 0)
    tb.n = dev.n
    aplan = _native.AsmPlan(tb, out_cap=int(batch.lengths.sum()) + 64 * dev.n + 4096, stride=2)
    ainfo = aplan.fit()
    astatus = aplan.status[: dev.n].cpu().numpy()
    assert not ainfo["overflow"] and (astatus == 0).all(), (ainfo, np.unique(astatus))
    out_bytes = ainfo["bytes"]
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        plan.launch()
        aplan.launch()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps + 1)]
    with ClockSampler(local_rank) as clocks:
        ev[0].record(stream)
        for k in range(args.steps):
            plan.launch()
            ev[2 * k + 1].record(stream)
            aplan.launch()
            ev[2 * k + 2].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[-1])
    ms_dis = sum(ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(args.steps)) / args.steps
    ms_asm = sum(ev[2 * k + 1].elapsed_time(ev[2 * k + 2]) for k in range(args.steps)) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    total_words = words * world
    value = total_words / (ms_step / 1e3)

    # parity of the timed configuration: every module round-trips bit-identically
    # (length totals on all, bytes on an even sample) and the text matches the oracle
    astatus = aplan.status[: dev.n].cpu().numpy()
    assert (astatus == 0).all()
    aspan = aplan.span[: 2 * dev.n].cpu().numpy().reshape(-1, 2)
    assert (aspan[:, 1] == batch.lengths).all(), "re-assembled sizes differ from the inputs"
    if rank == 0:
        from oracle import disasm as odis
        txt = plan.text[: text_bytes].cpu().numpy()
        span = plan.span.cpu().numpy()
        outb = aplan.out[: out_bytes].cpu().numpy()
        for i in np.linspace(0, dev.n - 1, 2000).astype(int):
            m = batch.module(int(i))
            assert outb[aspan[i, 0]:aspan[i, 0] + aspan[i, 1]].tobytes() == m, f"module {i} round trip"
            if i % 97 == 0:
                got = txt[span[2 * i]:span[2 * i] + span[2 * i + 1]].tobytes().decode()
                assert got == odis.disassemble(m), f"module {i} differs from oracle"

    # e2e through the host-buffer public API: RoundTripSession.run on the batch in pinned
    # host memory -- no sizing pass (capacity-bounded arenas, per-chunk counters read
    # back before each D2H), H2D of the binaries and D2H of text + binaries timed
    sess = RoundTripSession(chunks=int(os.environ.get("SKG_RT_CHUNKS", "16")))   # pipeline depth (experiments)
    h_batch = torch.from_numpy(batch.data).pin_memory()
    sess.run(h_batch, batch.offsets, batch.lengths)          # warm-up: buffer allocation
    e2e_steps = max(1, min(args.steps, 3))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t1 = time.perf_counter()
    e2e_runs = []
    for _ in range(e2e_steps):
        tr = time.perf_counter()
        text, tspan, tst, binv, bspan, bst = sess.run(h_batch, batch.offsets, batch.lengths)
        e2e_runs.append(time.perf_counter() - tr)
    e2e_s = (time.perf_counter() - t1) / e2e_steps
    log(f"[rank {rank}] e2e runs (ms): " + " ".join(f"{1e3 * r:.1f}" for r in e2e_runs))
    et = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_s = float(et.item())
    assert len(text) == text_bytes and (bst == 0).all()
    h2d = batch.data.nbytes + 16 * batch.n
    d2h = text_bytes + 16 * batch.n + 4 * batch.n + len(binv) + 16 * batch.n + 4 * batch.n + 64

    if rank != 0:
        return None
    peak, peak_src = peak_hbm()
    alg_bytes = 4 * words + text_bytes           # either direction: read one form, write the other
    per_kernel = {
        "skg_disasm": {"ms": ms_dis, "achieved_gbs": alg_bytes / (ms_dis / 1e3) / 1e9,
                       "words_per_s": words / (ms_dis / 1e3)},
        "skg_asm": {"ms": ms_asm, "achieved_gbs": alg_bytes / (ms_asm / 1e3) / 1e9,
                    "words_per_s": words / (ms_asm / 1e3)},
    }
    dom = max(per_kernel, key=lambda k: per_kernel[k]["ms"])
    achieved = per_kernel[dom]["achieved_gbs"]
    traffic = profile_traffic() or {}
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "words/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic: seeded builder-canonical paper-family modules (synth/families.py)",
        "config": {
            "workload": "configs[1]+configs[3]: batch of 1M synthetic modules (saxpy/matmul/DFT/"
                        "n-body/Black-Scholes variants) disassembled (default options) and the "
                        "text re-assembled to bit-identical binaries on 1 B200; step = skg_disasm "
                        "+ skg_asm over the whole batch",
            "modules_per_gpu": batch.n, "variants": args.variants, "words_per_gpu": words,
            "input_bytes_per_gpu": 4 * words, "text_bytes_per_gpu": text_bytes,
            "l2": "inputs (%.2f GB) and text (%.2f GB) exceed the 126 MB L2; no flush needed" %
                  (batch.data.nbytes / 1e9, text_bytes / 1e9),
            "parallelism": f"module-sharded x{world}",
        },
        "roofline": {
            "bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": alg_bytes,
            "traffic": (traffic.get(dom) or {}).get("bytes_per_launch"),
            "frac_of_nominal_8TBs": achieved / 8000.0,
            "per_kernel": per_kernel,
            # the bound these kernels actually sit against: instruction issue (warp instructions
            # per launch from the ncu capture in profiles/, like traffic; the peak is 148 SMs x
            # 4 schedulers x 1 warp instruction per cycle at 1965 MHz)
            "issue": _issue_roofline((traffic.get(dom) or {}).get("warp_inst_per_launch"),
                                     per_kernel[dom]["ms"]),
        },
        "e2e": {"value": total_words / e2e_s, "unit": "words/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "paper_2305_09493_b200.asm.RoundTripSession.run (fresh batch: no sizing "
                       "pass, host arrays of the results returned)"},
        # per step: skg_disasm + skg_asm, each = 3 scheduling kernels (size sort) + the main kernel
        "gpu_launches": 8 * args.steps,
        "clocks": clocks.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        ref = CpuReference()
        try:
            sample = sample_modules(batch, ref.cores * args.cpu_per_core)
            ref.run(sample[: ref.cores])          # fork + import warm-up
            w, dt = ref.run(sample)
        finally:
            ref.close()
        line["cpu_baseline"] = {"value": w / dt, "unit": "words/s", "cores": ref.cores,
                                "kind": ref_kind(),
                                "sample": f"{len(sample)} modules ({w} words) evenly spaced "
                                          f"through the batch, assemble_module(disassemble_module(m)) "
                                          f"each"}
    return line


# -- config 5: decode / validate / encode pipeline over one sharded 10M-module batch ------
def device_chunk(pool_dev, pool_off, pool_len, pick):
    """Synthetic input construction (untimed): the modules `pick` of the variant pool,
    packed on the device in 16-byte units (module starts 16-byte aligned)."""
    import torch
    from paper_2305_09493_b200 import _native
    dev = pool_dev.device
    pk = torch.from_numpy(pick.astype(np.int64)).to(dev)
    lengths = pool_len[pk]
    units = (lengths + 15) // 16
    starts = torch.cumsum(units, 0) - units
    U = int(units.sum().item())
    rep = torch.repeat_interleave(torch.arange(len(pick), device=dev), units)
    src = (pool_off[pk] // 16)[rep] + (torch.arange(U, device=dev) - starts[rep])
    data = torch.zeros(16 * U + 16, dtype=torch.uint8, device=dev)
    data[: 16 * U].view(-1, 16)[:] = pool_dev[: pool_dev.numel() // 16 * 16].view(-1, 16)[src]
    del rep, src
    b = _native.DeviceBatch(data, 16 * starts, lengths, int(lengths.max().item()) // 4,
                            int(lengths.sum().item()))
    return b


def config5_shard(n_modules, n_variants, rank, world, seed=SEED):
    """The global config-5 batch (module i = variant pick[i] of a seeded pool, as
    synth.families.sample_batch draws it) and this rank's contiguous module range
    [m0, m1) from shard.shard_ranges: (pool, pick, lengths, m0, m1)."""
    from paper_2305_09493_b200.shard import shard_ranges
    from synth.families import pack, variants
    pool = pack(variants(n_variants, seed))
    rng = np.random.default_rng(seed)
    pick = rng.integers(0, n_variants, size=n_modules)
    lengths = pool.lengths[pick]
    m0, m1 = shard_ranges(lengths, world)[rank]
    return pool, pick, lengths, m0, m1


def run_config5(args, rank, world, local_rank):
    """BASELINE configs[4]: one seeded batch of args.modules modules (default 10M), split
    across the ranks by shard.shard_ranges (contiguous module ranges balanced by bytes, no
    collective on the data path); every rank runs validate + disassemble + re-assemble over
    its shard in device-resident chunks.  value = all words / max-over-ranks step time."""
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    from paper_2305_09493_b200 import _native
    from paper_2305_09493_b200.disasm import DisassemblerOptions, option_bits

    t0 = time.perf_counter()
    pool, pick, lengths, m0, m1 = config5_shard(args.modules, args.variants, rank, world)
    pool_dev = torch.from_numpy(pool.data.copy()).cuda()
    pool_off = torch.from_numpy(pool.offsets.astype(np.int64)).cuda()
    pool_len = torch.from_numpy(pool.lengths.astype(np.int64)).cuda()
    chunks = []
    for c0 in range(m0, m1, args.chunk):
        chunks.append((c0, device_chunk(pool_dev, pool_off, pool_len, pick[c0:min(m1, c0 + args.chunk)])))
    words = int(lengths[m0:m1].sum()) // 4
    log(f"[rank {rank}] config 5 shard [{m0}, {m1}) of {args.modules}: {words} words in "
        f"{len(chunks)} chunks ({time.perf_counter() - t0:.1f}s)")
    opts = option_bits(DisassemblerOptions())
    # plans per chunk; the text / binary arenas and workspaces are shared (chunks run in order)
    max_bytes = max(b.total_bytes for _, b in chunks)
    max_n = max(b.n for _, b in chunks)
    text = torch.empty(4 * max_bytes + 4096, dtype=torch.uint8, device="cuda")
    out = torch.empty(max_bytes + 64 * max_n + 4096, dtype=torch.uint8, device="cuda")
    vtext = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")   # clean batch: no diagnostics

    def asm_plan(b, span, aws):
        mx = int(span[1::2].max().item())
        tb = _native.DeviceBatch(text, span[0::2], span[1::2], (mx + 3) // 4, 0)
        tb.n = b.n
        ap = _native.AsmPlan(tb, out_cap=16, stride=2, ws=aws)
        ap.out, ap.cap = out, out.numel()
        return ap

    plans, ws, aws = [], None, None
    for c0, b in chunks:
        # fused: decode -> validate -> disassemble in one pass (skg_disasm_validate), then asm
        fp = _native.DisasmPlan(b, opts, kind="pipeline", text_cap=16, ws=ws)
        ws = fp.ws
        fp.text, fp.cap, fp.vtext, fp.vcap = text, text.numel(), vtext, vtext.numel()
        fp.launch()
        finfo = fp.check()
        assert not finfo["overflow"] and finfo["errors"] == 0 and finfo["vtext_bytes"] == 0, finfo
        apf = asm_plan(b, fp.span, aws)
        aws = apf.ws
        apf.launch()
        ainfo = apf.check()
        st_ok = bool((fp.status[: b.n] == 0).all() and (fp.vstatus[: b.n] == 0).all()
                     and (apf.status[: b.n] == 0).all())
        assert st_ok and not ainfo["overflow"], (finfo, ainfo)
        # unfused, for comparison: skg_validate + skg_disasm + skg_asm
        vp = _native.DisasmPlan(b, 0, kind="validate", text_cap=1 << 20, ws=ws)
        vp.text, vp.cap = vtext, vtext.numel()
        dp = _native.DisasmPlan(b, opts, text_cap=16, ws=ws)
        dp.text, dp.cap = text, text.numel()
        dp.launch()
        apu = asm_plan(b, dp.span, aws)
        plans.append((b, fp, apf, vp, dp, apu))

    def step():
        for b, fp, apf, vp, dp, apu in plans:
            fp.launch()
            apf.launch()

    def step_unfused():
        for b, fp, apf, vp, dp, apu in plans:
            vp.launch()
            dp.launch()
            apu.launch()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    for _ in range(2):
        step_unfused()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        step_unfused()
    e1.record()
    torch.cuda.synchronize()
    tu = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tu, op=dist.ReduceOp.MAX)
    ms_unfused = float(tu.item()) / args.steps
    # parity of the fused step (sampled): validation clean, text == oracle, binaries == inputs
    from oracle import disasm as odis, validate as oval
    checked, text_bytes = 0, 0
    for ci, (b, dp, ap, _, _, _) in enumerate(plans):
        dp.launch()               # the arenas are shared: re-run this chunk, then check it
        info = dp.check()
        assert info["vtext_bytes"] == 0 and (dp.vstatus[: b.n] == 0).all()
        text_bytes += int(info["text_bytes"])
        ap.launch()
        torch.cuda.synchronize()
        dspan = dp.span[: 2 * b.n].cpu().numpy().reshape(-1, 2)
        aspan = ap.span[: 2 * b.n].cpu().numpy().reshape(-1, 2)
        assert (aspan[:, 1] == b.len.cpu().numpy()).all(), "re-assembled sizes differ"
        offs = b.off.cpu().numpy()
        for i in np.linspace(0, b.n - 1, max(2, 400 // len(plans))).astype(int):
            m = b.data[offs[i]:offs[i] + aspan[i, 1]].cpu().numpy().tobytes()
            got_bin = ap.out[aspan[i, 0]:aspan[i, 0] + aspan[i, 1]].cpu().numpy().tobytes()
            assert got_bin == m, f"chunk {ci} module {i}: round trip"
            txt = dp.text[dspan[i, 0]:dspan[i, 0] + dspan[i, 1]].cpu().numpy().tobytes().decode()
            if i % 5 == 0:
                assert txt == odis.disassemble(m), f"chunk {ci} module {i}: text differs from the oracle"
                assert not oval.validate(m)
            checked += 1
    tw = torch.tensor([words], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tw, op=dist.ReduceOp.SUM)
    total_words = int(tw.item())
    if rank != 0:
        return None
    peak, peak_src = peak_hbm()
    alg = 4 * words + text_bytes + text_bytes + 4 * words   # fused validate+disasm, then asm
    ach = alg / (ms_step / 1e3) / 1e9
    return {
        "metric": METRIC, "value": total_words / (ms_step / 1e3), "unit": "words/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic: seeded builder-canonical paper-family modules (synth/families.py)",
        "config": {
            "workload": "configs[4]: full decode/validate/encode pipeline over ONE seeded batch "
                        f"of {args.modules} modules split across {world} GPU(s) by "
                        "shard.shard_ranges; per rank, per device-resident chunk of "
                        f"{args.chunk} modules: the fused decode->validate->disassemble pass "
                        "(skg_disasm_validate) + skg_asm on its text",
            "ms_per_step_unfused": ms_unfused,
            "unfused": "skg_validate + skg_disasm + skg_asm (three reads of every module)",
            "modules_total": args.modules, "modules_rank0": m1 - m0, "words_total": total_words,
            "chunks_rank0": len(chunks), "parity_sampled_rank0": checked,
            "l2": "inputs and text exceed the 126 MB L2; no flush needed",
            "parallelism": f"module-sharded x{world} (no collective on the data path)",
        },
        "roofline": {"bound": "hbm", "kernel": "pipeline (fused validate+disasm, then asm)",
                     "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                     "peak_source": peak_src, "traffic": None,
                     "algorithmic_bytes_per_step_rank0": alg},
        "gpu_launches": 2 * 4 * len(chunks) * args.steps,
        "clocks": clocks.summary(),
    }


# -- config 3: one ~91M-word module, disassembled and validated over the whole GPU ----------
def run_config3(args, rank, world, local_rank):
    """BASELINE configs[2]: the synth/huge.py module (55,000 functions, ~91M words, an
    OpName on every id, long OpStrings) disassembled (default options: friendly names)
    and validated by the grid-wide kernels (skg_disasm_large / skg_validate_large),
    the module resident in HBM.  One step = disassembly + validation; value = words /
    step time.  The text is checked against the recorded SHA-256 (reference validate,
    oracle closed-form named disassembly: tests/golden/config3_55000.json).  Replicas
    only: every rank runs its own copy (the module does not shard)."""
    import hashlib
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    from paper_2305_09493_b200 import _native
    from paper_2305_09493_b200.disasm import DisassemblerOptions, option_bits
    from synth.huge import build_huge
    t0 = time.perf_counter()
    m = build_huge(args.functions)
    W = len(m) // 4
    log(f"[rank {rank}] config 3 module: {W} words ({time.perf_counter() - t0:.1f}s)")
    data = np.frombuffer(m + b"\0" * 16, dtype=np.uint8)
    dev = _native.DeviceBatch.from_host(data, np.array([0], np.int64), np.array([len(m)], np.int64))
    opts = option_bits(DisassemblerOptions())

    def step(view=True):
        # the text lands in pinned host memory (a numpy view of the staging buffer: no
        # further host-side copy into a Python object inside the timed step); its copy
        # runs on a side stream while the validation kernels run (the path
        # disassemble_validate_batch takes for one large module)
        return _native._disasm_validate_large(dev, 0, len(m), opts, None, None, view=view)

    for _ in range(args.warmup):
        step()
    text, diags = step(view=False)
    fx = ROOT / "tests" / "golden" / f"config3_{args.functions}.json"
    checked = None
    if fx.exists():
        rec = json.loads(fx.read_text())
        checked = (hashlib.sha256(text).hexdigest() == rec["oracle_disasm_named"]["sha256"]
                   and hashlib.sha256(diags).hexdigest() == rec["ref_validate"]["sha256"])
        assert checked, "config-3 output differs from the recorded digests"
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    if rank != 0:
        return None
    peak, peak_src = peak_hbm()
    alg = 4 * W + len(text) + 4 * W
    ach = alg / (ms_step / 1e3) / 1e9
    return {
        "metric": METRIC, "value": world * W / (ms_step / 1e3), "unit": "words/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic: synth/huge.py (seeded; canonicality checked on slices against the reference)",
        "config": {"workload": "configs[2]: one ~91M-word module (OpName on every id, long OpStrings, ids > "
                               "2^16) disassembled (default options) + validated on the GPU, module resident "
                               "in HBM; step = skg_disasm_large + skg_validate_large (the text's "
                               "copy into pinned host memory inside the step, overlapped with the validation)",
                   "functions": args.functions, "words": W, "text_bytes": len(text),
                   "digests_match_recorded": checked, "parallelism": f"replicas x{world}"},
        "roofline": {"bound": "hbm", "kernel": "skg_disasm_large + skg_validate_large", "achieved": ach,
                     "peak": peak, "unit": "GB/s", "frac": ach / peak, "peak_source": peak_src, "traffic": None,
                     "algorithmic_bytes_per_step": alg},
        "clocks": clocks.summary(),
    }


def run_config1(args, rank, world, local_rank):
    """BASELINE configs[0]: one saxpy-family module (synth/families.py, seed
    --c1-seed) disassembled and re-assembled through the public single-module API,
    assemble_module(disassemble_module(m)), one call pair per step: every step
    copies the module to the device, launches both kernels, and reads the text
    and the binary back (per-call latency, host buffers).  cpu_baseline: the
    reference's own disassemble_module / assemble_module on one host core, same
    module.  Replicas only: each rank makes its own calls."""
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    import paper_2305_09493_b200 as sk
    from synth.families import build_module
    m = build_module("saxpy", args.c1_seed)
    W = len(m) // 4

    def step():
        return sk.assemble_module(sk.disassemble_module(m))

    for _ in range(max(args.warmup, 20)):
        out = step()
    assert out == m, "config 1: round trip is not bit-identical"
    text = sk.disassemble_module(m)
    calls = max(args.steps, 200)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        e0.record()
        t0 = time.perf_counter()
        for _ in range(calls):
            step()
        t_host = time.perf_counter() - t0
        e1.record()
        torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_call = float(t.item()) / calls
    if rank != 0:
        return None
    cpu = None
    sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
    try:
        import spirvkit as R
        assert R.assemble_module(R.disassemble_module(m)) == m
        n_ref = 0
        r0 = time.perf_counter()
        while time.perf_counter() - r0 < args.c1_cpu_seconds:
            R.assemble_module(R.disassemble_module(m))
            n_ref += 1
        r_dt = (time.perf_counter() - r0) / n_ref
        cpu = {"value": W / r_dt, "unit": "words/s", "cores": 1, "kind": "reference",
               "sample": f"{n_ref} calls of spirvkit assemble_module(disassemble_module(m)) on the same "
                         f"module, one core ({1e6 * r_dt:.0f} us per call)"}
    except ImportError as exc:
        log(f"config 1: reference not importable ({exc}); no cpu_baseline")
    value = world * W / (ms_call / 1e3)
    return {
        "metric": METRIC, "value": value, "unit": "words/s", "n_gpus": world,
        "steps": calls, "warmup": max(args.warmup, 20), "ms_per_step": ms_call, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic: synth/families.py saxpy module (builder-canonical, seeded)",
        "config": {"workload": "configs[0]: one saxpy module, assemble_module(disassemble_module(m)) per step "
                               "through the public single-module API (per-call latency: H2D, both kernels, "
                               "D2H of text and binary inside every call)",
                   "seed": args.c1_seed, "words": W, "text_bytes": len(text),
                   "us_per_call": 1e3 * ms_call, "host_us_per_call": 1e6 * t_host / calls,
                   "parallelism": f"replicas x{world}"},
        "e2e": {"value": value, "unit": "words/s", "h2d_bytes_per_step": len(m) + len(text),
                "d2h_bytes_per_step": len(text) + len(m)},
        "gpu_launches": 2 * calls,   # per call pair: disasm_kernel + asm_kernel (one module: no scheduling sort)
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
    }


def run_reference(args, rank):
    if rank != 0:
        return None
    from synth.families import sample_batch
    batch = sample_batch(max(2000, args.ref_modules), min(args.variants, 2000), SEED)
    ref = CpuReference()
    try:
        per_step = ref.cores * args.cpu_per_core
        sample = sample_modules(batch, batch.n)
        words_total, t_total = 0, 0.0
        cursor = 0

        def take():
            nonlocal cursor
            out = [sample[(cursor + k) % len(sample)] for k in range(per_step)]
            cursor += per_step
            return out

        for _ in range(args.warmup):
            ref.run(take())
        for _ in range(args.steps):
            w, dt = ref.run(take())
            words_total += w
            t_total += dt
    finally:
        ref.close()
    value = words_total / t_total
    return {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": "words/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic: seeded builder-canonical paper-family modules (synth/families.py)",
        "config": {"workload": "configs[1]+configs[3] (bounded CPU sample): reference spirvkit "
                               "assemble_module(disassemble_module(m)) per module on all host cores",
                   "modules_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": "words/s", "cores": ref.cores,
                         "kind": ref_kind(),
                         "sample": f"{per_step} modules per step from a 2000-variant pool"},
        "e2e": {"value": value, "unit": "words/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--modules", type=int, default=1_000_000)
    ap.add_argument("--variants", type=int, default=10_000)
    ap.add_argument("--cpu-per-core", type=int, default=60)
    ap.add_argument("--ref-modules", type=int, default=4000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 5],
                    help="2: configs[1]+[3] round trip per GPU (default); 1: configs[0] one saxpy module "
                         "per call (latency); 3: configs[2] one huge module; 5: configs[4] sharded pipeline")
    ap.add_argument("--c1-seed", type=int, default=0, help="config 1: saxpy variant seed")
    ap.add_argument("--c1-cpu-seconds", type=float, default=5.0, help="config 1: reference timing budget")
    ap.add_argument("--functions", type=int, default=55000, help="config 3: functions of the module")
    ap.add_argument("--chunk", type=int, default=1_000_000, help="config 5: modules per device chunk")
    args = ap.parse_args()
    if args.config == 5 and "--modules" not in sys.argv:
        args.modules = 10_000_000
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch this command under torch.distributed.run
        import socket
        with socket.socket() as sock:
            sock.bind(("127.0.0.1", 0))
            port = sock.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
               os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "ours" and world != args.gpus:
        log(f"note: --gpus {args.gpus} but WORLD_SIZE={world}; n_gpus reports the real rank count")
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.impl == "ours":
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    if args.impl == "reference":
        line = run_reference(args, rank)
    elif args.config == 5:
        line = run_config5(args, rank, world, local_rank)
    elif args.config == 3:
        line = run_config3(args, rank, world, local_rank)
    elif args.config == 1:
        line = run_config1(args, rank, world, local_rank)
    else:
        line = run_ours(args, rank, world, local_rank)
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
