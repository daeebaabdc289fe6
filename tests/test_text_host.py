"""Host build of the assembler's CPython text semantics (csrc/skg_text.cuh)
against CPython itself: int(s, 0) / int(s), float(s), repr(s) (+ the %.200R
truncation), struct.pack('<e' / '<f').  Runs the exact device code compiled
for the host (tests/native/text_check.cpp); no GPU needed."""

import random
import shutil
import struct
import subprocess
import sys
from decimal import Decimal, getcontext
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "native" / "text_check.cpp"


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    d = tmp_path_factory.mktemp("textcheck")
    exe = d / "text_check"
    subprocess.run(["g++", "-O2", "-std=c++17", "-x", "c++", str(SRC), "-o", str(exe)], check=True)
    sys.path.insert(0, str(ROOT))
    from paper_2305_09493_b200 import tables
    blob = d / "blob.bin"
    blob.write_bytes(np.ascontiguousarray(tables.pack().blob, dtype="<u4").tobytes())

    def run(lines):
        out = subprocess.run([str(exe), str(blob)], input="\n".join(lines) + "\n", capture_output=True,
                             text=True, check=True).stdout.splitlines()
        assert len(out) == len(lines)
        return out
    return run


def hx(s: str) -> str:
    return s.encode("utf-8", "surrogatepass").hex()


def py_int(s, base):
    try:
        v = int(s, base)
    except ValueError as exc:
        if "Exceeds the limit" in str(exc):
            return "LIMIT " + str(exc).split("value has ")[1].split(" ")[0]
        return "INVALID"
    try:
        d = str(v)
    except ValueError:
        d = "LIMITSTR"
    return f"OK {d} {v:#x}"


def py_float(s):
    try:
        return struct.pack("<d", float(s))[::-1].hex()
    except ValueError:
        return "INVALID"


UNI_DIGITS = ["٠", "١", "१", "３", "\U0001d7ce", "৩"]
UNI_SPACES = [" ", " ", "　", "\x1f", "\x1c", " "]


def int_cases(rng):
    fixed = ["0", "00", "0_0", "0_", "_0", "01", "0b101", "-0b101", "0B1_0", "0o17", "0O_7", "0x_1f",
             "0x", "0x_", "0x__1", "1__0", "1_0", "+5", "-0", "- 5", "", " ", "+", "-", "5 ", " 5",
             " 5　", "5\x1f", "٣", "١٢٣", "1٢3", "²", "0x1F", "0XfF", "18446744073709551615",
             "18446744073709551616", "-18446744073709551616", "99999999999999999999999", "0" * 4301,
             "0" + "1" * 4301, "1" * 4300, "1" * 4301, "1" * 4301 + "x", "1_" * 2200 + "1",
             "0x" + "f" * 5000, "0x" + "1" * 3600, "0b" + "1" * 20000, "0o" + "7" * 5000, "12a", "a12",
             "0x1g", "0b2", "0o8", "1e5", "1.0", "\x00", "1\x00", "１２"]
    out = [(s, b) for s in fixed for b in (0, 10)]
    for _ in range(3000):
        v = rng.choice([rng.randrange(0, 1 << 70), rng.randrange(0, 100), rng.randrange(1 << 63, 1 << 65),
                        rng.randrange(0, 10 ** rng.randrange(1, 60))])
        form = rng.choice(["d", "x", "X", "o", "b"])
        s = {"d": str(v), "x": f"0x{v:x}", "X": f"0X{v:X}", "o": f"0o{v:o}", "b": f"0b{v:b}"}[form]
        if rng.random() < 0.3:
            i = rng.randrange(len(s) + 1)
            s = s[:i] + "_" + s[i:]
        if rng.random() < 0.2:
            s = rng.choice("+-") + s
        if rng.random() < 0.1:
            s = rng.choice(UNI_SPACES + [" "]) + s + rng.choice(UNI_SPACES + ["", " "])
        if rng.random() < 0.1:
            s = "".join(rng.choice(UNI_DIGITS) if c.isdigit() and rng.random() < 0.5 else c for c in s)
        if rng.random() < 0.05:
            s = s.replace("0", "O", 1)
        out.append((s, rng.choice((0, 10))))
    return out


def float_cases(rng):
    fixed = ["1", "1.", ".5", ".", "-.5", "+.5e3", "1e", "1e+", "1e-5", "1E5", "e5", "inf", "-inf", "+inf",
             "Infinity", "-iNfInItY", "infinit", "nan", "-nan", "NaN", "+nan", "nan1", "1_0.5", "1_.5",
             "1._5", "_1.5", "1.5_", "1e1_0", "1_e5", "0x10", " 1.5 ", " 1.5", "١.٥", "1 .5", "",
             "  ", "1e999999999999999999", "1e-999999999999999999", "0e999999", "-0.0", "0.000",
             "4.9406564584124654e-324", "2.4703282292062327e-324", "2.4703282292062328e-324",
             "1.7976931348623157e308", "1.7976931348623158e308", "1.7976931348623159e308",
             "2.2250738585072011e-308", "2.2250738585072012e-308", "9007199254740993",
             "9007199254740992.5", "9007199254740993.0000000000000000000000000000001",
             "0." + "0" * 400 + "1", "1" + "0" * 400, "1" * 900 + "e-600", "\x00", "1\x00"]
    out = list(fixed)
    getcontext().prec = 1200
    for _ in range(4000):
        kind = rng.randrange(6)
        if kind == 0:
            x = struct.unpack("<d", struct.pack("<Q", rng.getrandbits(64)))[0]
            out.append(repr(x))
        elif kind == 1:
            x = struct.unpack("<f", struct.pack("<I", rng.getrandbits(32)))[0]
            out.append(repr(x))
        elif kind == 2:   # exact halfway points between adjacent doubles, +/- tiny
            b = rng.getrandbits(63) & ~(0x7FF << 52) | (rng.randrange(1, 2046) << 52)
            lo = struct.unpack("<d", struct.pack("<Q", b))[0]
            hi = struct.unpack("<d", struct.pack("<Q", b + 1))[0]
            mid = (Decimal(lo) + Decimal(hi)) / 2
            s = format(mid, "f") if rng.random() < 0.3 else format(mid, "e")
            t = rng.randrange(3)
            if t == 1:
                s = s.replace("e", "0000000000000000000001e") if "e" in s else s + "0000000001"
            out.append(s)
        elif kind == 3:
            digits = "".join(rng.choice("0123456789") for _ in range(rng.randrange(1, 40)))
            dot = rng.randrange(len(digits) + 1)
            s = digits[:dot] + "." + digits[dot:]
            if rng.random() < 0.7:
                s += f"e{rng.randrange(-340, 320)}"
            out.append(s)
        elif kind == 4:   # subnormal / tiny
            x = struct.unpack("<d", struct.pack("<Q", rng.getrandbits(52)))[0]
            out.append(repr(x) if rng.random() < 0.5 else f"{x:.30e}")
        else:
            out.append(f"{rng.uniform(-1e6, 1e6):.{rng.randrange(0, 20)}f}")
    return out


def repr_cases(rng):
    alphabet = ["a", "'", '"', "\\", "\t", "\n", "\r", "\x00", "\x7f", "\x85", "\xa0", "é", "​",
                " ", "\ud800", "\udfff", "\U0001f600", "\U000e0001", "￿", "\x1b", " ", "%",
                "͸", "\U0010ffff", "中"]
    out = []
    for _ in range(2000):
        s = "".join(rng.choice(alphabet) for _ in range(rng.randrange(0, 12)))
        out.append(s)
    out.append("x" * 300)
    out.append("é" * 300)
    return out


def test_int_parse(checker):
    rng = random.Random(7)
    cases = int_cases(rng)
    got = checker([f"I {b} {hx(s)}" for s, b in cases])
    bad = [(s[:60], b, g[:80], py_int(s, b)[:80]) for (s, b), g in zip(cases, got) if g != py_int(s, b)]
    assert not bad, bad[:10]


def test_float_parse(checker):
    rng = random.Random(11)
    cases = float_cases(rng)
    got = checker([f"F {hx(s)}" for s in cases])
    bad = [(s[:80], g, py_float(s)) for s, g in zip(cases, got) if g != py_float(s)]
    assert not bad, bad[:10]


def test_repr(checker):
    rng = random.Random(3)
    cases = repr_cases(rng)
    lines = [f"R 0 {hx(s)}" for s in cases] + [f"R 200 {hx(s)}" for s in cases]
    got = checker(lines)
    want = [hx(repr(s)) for s in cases] + [hx(repr(s)[:200]) for s in cases]
    bad = [(c, g, w) for c, g, w in zip(cases + cases, got, want) if g != w]
    assert not bad, bad[:10]


def test_pack_half_single(checker):
    rng = random.Random(5)
    vals = [0.0, -0.0, 65504.0, 65519.99, 65520.0, -65520.0, 6e-8, 2.98e-8, 2.9802322387695312e-08,
            5.960464477539063e-08, 3.4028235e38, 3.4028235677973366e+38, 3.402823669209385e+38,
            1e39, float("inf"), float("-inf"), float("nan"), -float("nan"), 1e-320, 5e-324]
    for _ in range(5000):
        vals.append(struct.unpack("<d", struct.pack("<Q", rng.getrandbits(64)))[0])
        vals.append(rng.uniform(-70000, 70000))
        vals.append(rng.uniform(-1e-4, 1e-4))
    lines = [f"P {struct.unpack('<Q', struct.pack('<d', v))[0]:016x}" for v in vals]
    got = checker(lines)

    def want(v):
        try:
            h = struct.pack("<e", v)[::-1].hex()
        except OverflowError:
            h = "OVF"
        try:
            f = struct.pack("<f", v)[::-1].hex()
        except OverflowError:
            f = "OVF"
        return f"{h} {f}"
    bad = [(v, g, want(v)) for v, g in zip(vals, got) if g != want(v)]
    assert not bad, bad[:10]
