"""Seeded synthetic SPIR-V modules replicating the paper's benchmark kernels.

The paper's evaluation kernels (saxpy, DFT, Black-Scholes: PAPER.md:786-789;
matmul and n-body from the TornadoVM suite) are emitted here as
OpenCL-style compute kernels in *builder-canonical* layout, i.e. the exact
section order ``ModuleScope.serialize`` produces (reference
``builder.py:39-43, 187-197``) with builder-style literal encodings
(``codec.py:132-168``).  Canonical modules re-assemble byte-identically from
their disassembly, which is what the round-trip benchmark relies on
(SURVEY.md appendix A.5).  ``tests/test_synth.py`` checks canonicality against
the reference builder/assembler when the reference is available.

Each family is an unstructured loop: entry -> header (2x OpPhi) -> body ->
back-edge -> exit, with the family's arithmetic unrolled a random number of
times, random 32/64-bit integer and f16/f32/f64 constants (normal,
log-uniform, subnormal and signed-zero magnitudes), OpName on a random share
of ids from a collision-prone vocabulary, and an OpString of 0-256 bytes.

Pure Python + numpy; no reference code is imported, so this also runs on the
GPU box (``bench.py`` builds its batches from it).
"""

from __future__ import annotations

import math
import random
import struct

import numpy as np

from paper_2305_09493_b200 import grammar

MAGIC = 0x07230203
FAMILIES = ("saxpy", "matmul", "dft", "nbody", "blackscholes")
SECTIONS = ("capabilities", "extensions", "ext_imports", "memory_model", "entry_points",
            "execution_modes", "debug_sources", "debug_names", "debug_processed",
            "annotations", "globals")
VOCAB = ("x", "x", "i", "acc", "tmp", "a b", "3d", "x_0", "sum", "sum", "tmp!", "",
         "val", "ptr", "gid", "idx", "re", "im", "résultat", "n")


def _pack_string(text: str) -> list[int]:
    data = text.encode("utf-8") + b"\x00"
    data += b"\x00" * (-len(data) % 4)
    return list(struct.unpack(f"<{len(data) // 4}I", data))


class Writer:
    """Minimal canonical emitter: section buckets + functions, ids by counter."""

    def __init__(self, spec, minor=2):
        self.spec = spec
        self.minor = minor
        self.sec = {s: [] for s in SECTIONS}
        self.functions = []           # list of word lists
        self.counter = 0

    def new_id(self) -> int:
        self.counter += 1
        return self.counter

    def enum(self, kind, name) -> int:
        return self.spec.kind(kind).enumerant(name).value

    def inst(self, opname, *ops) -> list[int]:
        words = []
        for o in ops:
            if isinstance(o, str):
                words.extend(_pack_string(o))
            elif isinstance(o, (list, tuple)):
                words.extend(int(w) & 0xFFFFFFFF for w in o)
            else:
                words.append(int(o) & 0xFFFFFFFF)
        opcode = self.spec.instruction(opname).opcode
        return [((len(words) + 1) << 16) | opcode] + words

    def add(self, section, opname, *ops):
        self.sec[section].extend(self.inst(opname, *ops))

    def words(self) -> list[int]:
        out = [MAGIC, (1 << 16) | (self.minor << 8), 32 << 16, self.counter + 1, 0]
        for s in SECTIONS:
            out.extend(self.sec[s])
        for f in self.functions:
            out.extend(f)
        return out


class Function:
    def __init__(self, w: Writer, ret_t, fn_id, fn_t, control="None"):
        self.w = w
        self.words = w.inst("OpFunction", ret_t, fn_id, w.enum("FunctionControl", control), fn_t)

    def param(self, t):
        pid = self.w.new_id()
        self.words += self.w.inst("OpFunctionParameter", t, pid)
        return pid

    def label(self, lid):
        self.words += self.w.inst("OpLabel", lid)

    def op(self, opname, *ops):
        self.words += self.w.inst(opname, *ops)

    def value(self, opname, t, *ops):
        rid = self.w.new_id()
        self.words += self.w.inst(opname, t, rid, *ops)
        return rid

    def end(self):
        self.words += self.w.inst("OpFunctionEnd")
        self.w.functions.append(self.words)


def _float_bits(value: float, width: int) -> list[int]:
    if width == 64:
        lo, hi = struct.unpack("<2I", struct.pack("<d", value))
        return [lo, hi]
    fmt = "<f" if width == 32 else "<e"
    raw = struct.pack(fmt, value)
    return [struct.unpack("<I", raw.ljust(4, b"\x00"))[0]]


def _random_float(rng: random.Random, width: int) -> float:
    r = rng.random()
    if r < 0.05:
        return rng.choice((0.0, -0.0, 1.0, -1.0, 0.5, 2.0, 0.1))
    if r < 0.10:    # subnormals of the target width
        tiny = {16: 2.0 ** -24, 32: 2.0 ** -149, 64: 5e-324}[width]
        return tiny * rng.randint(1, 1000) * rng.choice((1, -1))
    if r < 0.55:
        v = rng.gauss(0.0, 10.0)
    else:           # log-uniform magnitudes within the width's finite range
        span = {16: 14, 32: 37, 64: 300}[width]
        v = rng.choice((1, -1)) * 10.0 ** rng.uniform(-span, span)
    if width == 16:
        v = max(-65000.0, min(65000.0, v))
    # round to the storage width so encode/decode is the identity
    return struct.unpack("<d", struct.pack("<d", v))[0] if width == 64 else \
        struct.unpack("<f" if width == 32 else "<e", struct.pack("<f" if width == 32 else "<e", v))[0]


def build_module(family: str, seed: int, spec=None) -> bytes:
    """One builder-canonical module of ``family`` (deterministic in ``seed``)."""
    spec = spec if spec is not None else grammar.load_pinned()
    rng = random.Random(f"{family}:{seed}")
    w = Writer(spec, minor=rng.choice((0, 1, 2, 2, 2)))
    use_f64 = rng.random() < 0.4
    use_f16 = rng.random() < 0.2
    caps = ["Addresses", "Linkage", "Kernel", "Int64", "Int8"]      # PAPER.md Listing 6
    caps += ["Float64"] if use_f64 else []
    caps += ["Float16"] if use_f16 else []
    for c in caps:
        w.add("capabilities", "OpCapability", w.enum("Capability", c))
    ext = w.new_id()
    w.add("ext_imports", "OpExtInstImport", ext, "OpenCL.std")
    w.add("memory_model", "OpMemoryModel", w.enum("AddressingModel", "Physical64"),
          w.enum("MemoryModel", "OpenCL"))

    void_t, bool_t, u32, u64, u8 = (w.new_id() for _ in range(5))
    f32 = w.new_id()
    f64 = w.new_id() if use_f64 else None
    f16 = w.new_id() if use_f16 else None
    v3u64, ptr_in, ptr_gl, fn_t = (w.new_id() for _ in range(4))
    gid = w.new_id()
    kernel = w.new_id()
    name_pool = {}

    # entry point + debug
    kname = f"{family}_k{seed % 97}"
    w.add("entry_points", "OpEntryPoint", w.enum("ExecutionModel", "Kernel"), kernel, kname, gid)
    w.add("debug_sources", "OpSource", w.enum("SourceLanguage", "OpenCL_C"), 120)
    slen = rng.choice((0, 0, 8, 32, 64, 256))
    src = w.new_id()
    w.add("debug_sources", "OpString", src,
          "".join(rng.choice("abcdefghijklmnopqrstuvwxyz _(){};*+=\\\"é") for _ in range(slen)))
    w.add("annotations", "OpDecorate", gid, w.enum("Decoration", "BuiltIn"),
          w.enum("BuiltIn", "GlobalInvocationId"))
    w.add("annotations", "OpDecorate", gid, w.enum("Decoration", "Constant"))
    w.add("annotations", "OpDecorate", gid, w.enum("Decoration", "LinkageAttributes"),
          "__spirv_BuiltInGlobalInvocationId", w.enum("LinkageType", "Import"))
    name_pool[gid] = "__spirv_BuiltInGlobalInvocationId"
    name_pool[kernel] = kname

    # types
    w.add("globals", "OpTypeVoid", void_t)
    w.add("globals", "OpTypeBool", bool_t)
    w.add("globals", "OpTypeInt", u32, 32, 0)
    w.add("globals", "OpTypeInt", u64, 64, 0)
    w.add("globals", "OpTypeInt", u8, 8, 0)
    w.add("globals", "OpTypeFloat", f32, 32)
    if f64:
        w.add("globals", "OpTypeFloat", f64, 64)
    if f16:
        w.add("globals", "OpTypeFloat", f16, 16)
    w.add("globals", "OpTypeVector", v3u64, u64, 3)
    w.add("globals", "OpTypePointer", ptr_in, w.enum("StorageClass", "Input"), v3u64)
    w.add("globals", "OpTypePointer", ptr_gl, w.enum("StorageClass", "CrossWorkgroup"), f32)
    n_params = {"saxpy": 4, "matmul": 4, "dft": 4, "nbody": 3, "blackscholes": 5}[family]
    w.add("globals", "OpTypeFunction", fn_t, void_t, *([ptr_gl] * (n_params - 1) + [u32]))

    # constants
    consts_u32 = []
    for _ in range(rng.randint(3, 8)):
        c = w.new_id()
        w.add("globals", "OpConstant", u32, c, rng.choice((0, 1, 2, 4, rng.getrandbits(32))))
        consts_u32.append(c)
    one64 = w.new_id()
    w.add("globals", "OpConstant", u64, one64, (1, 0))
    for _ in range(rng.randint(0, 3)):
        v = rng.getrandbits(64)
        w.add("globals", "OpConstant", u64, w.new_id(), (v & 0xFFFFFFFF, v >> 32))
    fconsts = []
    for _ in range(rng.randint(2, 8)):
        c = w.new_id()
        w.add("globals", "OpConstant", f32, c, _float_bits(_random_float(rng, 32), 32))
        fconsts.append(c)
    if f64:
        for _ in range(rng.randint(1, 4)):
            w.add("globals", "OpConstant", f64, w.new_id(), _float_bits(_random_float(rng, 64), 64))
    if f16:
        for _ in range(rng.randint(1, 3)):
            w.add("globals", "OpConstant", f16, w.new_id(), _float_bits(_random_float(rng, 16), 16))
    w.add("globals", "OpVariable", ptr_in, gid, w.enum("StorageClass", "Input"))

    # the kernel
    fn = Function(w, void_t, kernel, fn_t)
    params = [fn.param(ptr_gl) for _ in range(n_params - 1)]
    n_arg = fn.param(u32)
    for p in params:
        w.add("annotations", "OpDecorate", p, w.enum("Decoration", "Alignment"), 4)
    entry, header, body, exit_ = (w.new_id() for _ in range(4))
    fn.label(entry)
    g3 = fn.value("OpLoad", v3u64, gid, w.enum("MemoryAccess", "Aligned"), 32)
    g0 = fn.value("OpCompositeExtract", u64, g3, 0)
    gi = fn.value("OpUConvert", u32, g0)
    fn.op("OpBranch", header)
    fn.label(header)
    i_phi, acc_phi = w.new_id(), w.new_id()
    i_next_id, acc_next_id = w.new_id(), w.new_id()
    fn.op("OpPhi", u32, i_phi, consts_u32[0], entry, i_next_id, body)
    fn.op("OpPhi", f32, acc_phi, fconsts[0], entry, acc_next_id, body)
    cond = fn.value("OpULessThan", bool_t, i_phi, n_arg)
    fn.op("OpBranchConditional", cond, body, exit_)
    fn.label(body)

    def load(ptr_param, index):
        p = fn.value("OpInBoundsPtrAccessChain", ptr_gl, ptr_param, index)
        return fn.value("OpLoad", f32, p, w.enum("MemoryAccess", "Aligned"), 4)

    def ext_call(name, *args):
        return fn.value("OpExtInst", f32, ext, grammar.load_pinned_extended().instruction(name).opcode, *args)

    acc = acc_phi
    idx = fn.value("OpIAdd", u32, gi, i_phi)
    unroll = rng.randint(1, {"saxpy": 6, "matmul": 10, "dft": 8, "nbody": 8, "blackscholes": 6}[family])
    for k in range(unroll):
        idx = fn.value("OpIAdd", u32, idx, rng.choice(consts_u32))
        if family == "saxpy":
            x = load(params[0], idx)
            y = load(params[1], idx)
            ax = fn.value("OpFMul", f32, rng.choice(fconsts), x)
            r = fn.value("OpFAdd", f32, ax, y)
            p = fn.value("OpInBoundsPtrAccessChain", ptr_gl, params[2], idx)
            fn.op("OpStore", p, r, w.enum("MemoryAccess", "Aligned"), 4)
            acc = fn.value("OpFAdd", f32, acc, r)
        elif family == "matmul":
            row = fn.value("OpIMul", u32, idx, n_arg)
            col = fn.value("OpIAdd", u32, row, rng.choice(consts_u32))
            a = load(params[0], row)
            b = load(params[1], col)
            acc = fn.value("OpFAdd", f32, acc, fn.value("OpFMul", f32, a, b))
        elif family == "dft":
            x = load(params[0], idx)
            ang = fn.value("OpFMul", f32, x, rng.choice(fconsts))
            c = ext_call("cos", ang)
            s = ext_call("sin", ang)
            re = fn.value("OpFMul", f32, x, c)
            im = fn.value("OpFMul", f32, x, s)
            acc = fn.value("OpFAdd", f32, acc, fn.value("OpFSub", f32, re, im))
        elif family == "nbody":
            px = load(params[0], idx)
            py = load(params[1], idx)
            dx = fn.value("OpFSub", f32, px, acc)
            dy = fn.value("OpFSub", f32, py, acc)
            d2 = fn.value("OpFAdd", f32, fn.value("OpFMul", f32, dx, dx), fn.value("OpFMul", f32, dy, dy))
            inv = ext_call("rsqrt", fn.value("OpFAdd", f32, d2, rng.choice(fconsts)))
            acc = fn.value("OpFAdd", f32, acc, fn.value("OpFMul", f32, inv, dx))
        else:  # blackscholes
            s = load(params[0], idx)
            kx = load(params[1], idx)
            lg = ext_call("log", fn.value("OpFDiv", f32, s, kx))
            sq = ext_call("sqrt", fn.value("OpFAdd", f32, rng.choice(fconsts), lg))
            ex = ext_call("exp", fn.value("OpFSub", f32, lg, sq))
            d = fn.value("OpFMul", f32, ex, ext_call("fabs", sq))
            acc = fn.value("OpFAdd", f32, acc, d)
            p = fn.value("OpInBoundsPtrAccessChain", ptr_gl, params[2 + k % 2], idx)
            fn.op("OpStore", p, d, w.enum("MemoryAccess", "Aligned"), 4)
    # close the loop: i_next / acc_next are the pre-reserved phi operands
    fn.words += w.inst("OpIAdd", u32, i_next_id, i_phi, consts_u32[min(1, len(consts_u32) - 1)])
    fn.words += w.inst("OpFAdd", f32, acc_next_id, acc, fconsts[-1])
    fn.op("OpBranch", header)
    fn.label(exit_)
    out = fn.value("OpInBoundsPtrAccessChain", ptr_gl, params[-1], gi)
    fn.op("OpStore", out, acc_phi, w.enum("MemoryAccess", "Aligned"), 4)
    fn.op("OpReturn")
    fn.end()

    # debug names on a random share of ids (OpName bucket is pre-annotations)
    share = rng.choice((0.0, 0.1, 0.3, 0.6, 1.0))
    for ident in range(1, w.counter + 1):
        if ident in name_pool and rng.random() < 0.8:
            w.add("debug_names", "OpName", ident, name_pool[ident])
        elif rng.random() < share:
            w.add("debug_names", "OpName", ident, rng.choice(VOCAB))
    words = w.words()
    return struct.pack(f"<{len(words)}I", *words)


def variants(n: int, seed: int = 20261017) -> list[bytes]:
    """n distinct modules, families in equal shares."""
    return [build_module(FAMILIES[i % len(FAMILIES)], seed * 1000003 + i) for i in range(n)]


class Batch:
    """A packed batch: one byte arena, module starts 16-byte aligned."""

    def __init__(self, data: np.ndarray, offsets: np.ndarray, lengths: np.ndarray):
        self.data, self.offsets, self.lengths = data, offsets, lengths

    @property
    def n(self):
        return len(self.offsets)

    @property
    def words(self) -> int:
        return int(self.lengths.sum() // 4)

    def module(self, i) -> bytes:
        o, n = int(self.offsets[i]), int(self.lengths[i])
        return self.data[o:o + n].tobytes()


def pack(modules: list[bytes]) -> Batch:
    lengths = np.array([len(m) for m in modules], dtype=np.int64)
    padded = (lengths + 15) // 16 * 16
    offsets = np.zeros(len(modules), dtype=np.int64)
    if len(modules) > 1:
        offsets[1:] = np.cumsum(padded)[:-1]
    data = np.zeros(int(padded.sum()) + 16, dtype=np.uint8)
    for m, o in zip(modules, offsets):
        data[o:o + len(m)] = np.frombuffer(m, dtype=np.uint8)
    return Batch(data, offsets, lengths)


def sample_batch(n_modules: int, n_variants: int = 10000, seed: int = 20261017) -> Batch:
    """n_modules drawn (seeded) from n_variants distinct variants, packed."""
    base = pack(variants(n_variants, seed))
    rng = np.random.default_rng(seed)
    pick = rng.integers(0, n_variants, size=n_modules)
    lengths = base.lengths[pick]
    padded = (lengths + 15) // 16 * 16
    offsets = np.zeros(n_modules, dtype=np.int64)
    offsets[1:] = np.cumsum(padded)[:-1]
    total = int(padded.sum()) + 16
    data = np.zeros(total, dtype=np.uint8)
    # gather in 16-byte units: every module is padded to 16 bytes in both arenas
    src16 = base.data[: len(base.data) // 16 * 16].view(np.uint32).reshape(-1, 4)
    dst16 = data[: total // 16 * 16].view(np.uint32).reshape(-1, 4)
    units = padded // 16
    src_unit = base.offsets[pick] // 16
    starts = offsets // 16
    rep = np.repeat(np.arange(n_modules), units)
    within = np.arange(int(units.sum())) - np.repeat(starts, units)
    dst16[starts[rep] + within] = src16[src_unit[rep] + within]
    return Batch(data, offsets, lengths)
