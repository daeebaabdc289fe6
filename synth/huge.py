"""Config-3 generator: one large module emitted with numpy.

The reference builder is far too slow at this size, so the module is tiled
from a per-function template: `n_fn` functions, each a parameter, a label, a
chain of `chain` OpIAdd instructions and OpReturn, every id named by an OpName
(collision-prone vocabulary, so name de-duplication and demotion are
exercised) and a few long OpString literals.  Ids grow to ~n_fn * (chain + 3),
so operand words have non-zero high halves once that passes 2^16.  The
layout follows the builder's section order (debug, annotations, types,
functions), so the module validates clean; its disassembly and validation are
checked against the oracle on small instances (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import struct

import numpy as np

VOCAB = ("x", "tmp", "acc", "sum", "x_0", "i", "3d", "a b", "val", "sum_1", "n", "résumé"[:5])


def _name_words(text: str) -> list[int]:
    data = text.encode("utf-8") + b"\x00"
    data += b"\x00" * (-len(data) % 4)
    return list(struct.unpack(f"<{len(data) // 4}I", data))


def _inst(op: int, *ops: int) -> list[int]:
    return [((1 + len(ops)) << 16) | op, *ops]


def build_huge(n_fn: int, chain: int = 200, seed: int = 1, string_kib=(1, 8, 64)) -> bytes:
    rng = np.random.default_rng(seed)
    # fixed ids: 1 OpenCL.std, 2 void, 3 int32, 4 ptr, 5 fn type, 6 const 1, 7.. strings
    n_str = len(string_kib)
    first = 7 + n_str
    per_fn = 3 + chain                       # function, parameter, label, chain values
    bound = first + n_fn * per_fn
    head = [0x07230203, 0x00010200, 0x00200000, bound, 0]
    body: list[int] = []
    for cap in (4, 5, 6):                    # Addresses, Linkage, Kernel
        body += _inst(17, cap)
    body += _inst(11, 1, *_name_words("OpenCL.std"))
    body += _inst(14, 2, 2)                  # Physical64 OpenCL
    body += _inst(15, 6, first, *_name_words("k"))          # OpEntryPoint Kernel %f0 "k"
    for j, kib in enumerate(string_kib):     # OpString: long literals (debug section)
        text = ("spirv" * (kib * 1024 // 5 + 1))[: kib * 1024 - 1]
        body += _inst(7, 7 + j, *_name_words(text))
    # OpName for every id of the functions (vectorised; 1- or 2-word names)
    vw = [_name_words(v) for v in VOCAB]
    vlen = np.array([len(w) for w in vw], dtype=np.int64)
    v0 = np.array([w[0] for w in vw], dtype=np.uint32)
    v1 = np.array([w[1] if len(w) > 1 else 0 for w in vw], dtype=np.uint32)
    ids = np.arange(first, bound, dtype=np.uint32)
    pick = rng.integers(0, len(VOCAB), size=len(ids))
    nw = 2 + vlen[pick]
    start = np.concatenate([[0], np.cumsum(nw)[:-1]])
    names = np.zeros(int(nw.sum()), dtype=np.uint32)
    names[start] = (nw.astype(np.uint32) << 16) | 5
    names[start + 1] = ids
    names[start + 2] = v0[pick]
    two = vlen[pick] == 2
    names[start[two] + 3] = v1[pick[two]]
    types = []
    types += _inst(19, 2)                    # OpTypeVoid %2
    types += _inst(21, 3, 32, 0)             # OpTypeInt %3 32 0
    types += _inst(32, 4, 5, 3)              # OpTypePointer %4 CrossWorkgroup %3
    types += _inst(33, 5, 2, 4)              # OpTypeFunction %5 %2 %4
    types += _inst(43, 3, 6, 1)              # OpConstant %3 %6 1
    # function template with ids relative to the function base
    t = []
    t += _inst(54, 2, 0, 0, 5)               # OpFunction %2 %f None %5
    t += _inst(55, 4, 1)                     # OpFunctionParameter %4 %p
    t += _inst(248, 2)                       # OpLabel %l
    prev_rel, prev_abs = None, 6
    for c in range(chain):
        if prev_rel is None:
            t += _inst(128, 3, 3 + c, prev_abs, 6)     # OpIAdd %3 %v %6 %6
        else:
            t += _inst(128, 3, 3 + c, prev_rel, 6)
        prev_rel = 3 + c
    t += _inst(253)                          # OpReturn
    t += _inst(56)                           # OpFunctionEnd
    tmpl = np.array(t, dtype=np.uint32)
    rel = np.zeros(len(tmpl), dtype=bool)    # words holding function-relative ids
    # mark relative id positions: OpFunction result (1), parameter result (5+2), label (8+1), chains
    rel[[2, 7, 9]] = True
    base = 10
    for c in range(chain):
        rel[base + 2] = True                 # result
        if c > 0:
            rel[base + 3] = True             # previous value
        base += 5
    offs = first + per_fn * np.arange(n_fn, dtype=np.uint32)
    fns = np.tile(tmpl, (n_fn, 1))
    fns[:, rel] += offs[:, None]
    words = np.concatenate([np.array(head + body, dtype=np.uint32), names,
                            np.array(types, dtype=np.uint32), fns.reshape(-1)])
    return words.astype("<u4").tobytes()
