"""Decoder of the pass records produced by the fusion planner
(paper_2401_06861_b200/csrc/engine.hpp: PassHdr / MOp; nq_plan_debug).

Used for planner introspection (tests, bench statistics).  It does not execute
anything.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field
from typing import List

import numpy as np

MOP_NAMES = {0: "dense", 1: "diag", 2: "xperm", 3: "swap", 4: "depol", 5: "layout"}
HDR_FMT = "<iiiiqIIII16b56b16bi16b3i"
HDR_SIZE = struct.calcsize(HDR_FMT)
MOP_FMT = "<BB8bHII4xQ"
MOP_SIZE = struct.calcsize(MOP_FMT)
assert HDR_SIZE == 160 and MOP_SIZE == 32


@dataclass
class MicroOp:
    type: str
    k: int
    pos: List[int]
    gq: List[int]
    mat: int
    cmask_tile: int
    cmask_glob: int


@dataclass
class Pass:
    m: int
    nloc: int
    ntiles: int
    q: List[int]
    rest: List[int]
    qst: List[int] = field(default_factory=list)  # store position of tile bit i (relabelling pass)
    lab: List[int] = field(default_factory=list)  # stored content of tile bit i carries tile bit lab[i]'s label
    ops: List[MicroOp] = field(default_factory=list)
    pool: np.ndarray = None


def decode(buf: bytes) -> List[Pass]:
    out = []
    at = 0
    while at < len(buf):
        f = struct.unpack_from(HDR_FMT, buf, at)
        m, nops, nloc, nrest, ntiles, op_off, pool_off, pool_n, nbytes = f[:9]
        q = list(f[9:9 + 16])[:m]
        rest = list(f[25:25 + 56])[:nrest]
        qst = list(f[81:81 + 16])[:m]
        lab = list(f[98:98 + 16])[:m]
        p = Pass(m=m, nloc=nloc, ntiles=ntiles, q=q, rest=rest, qst=qst, lab=lab)
        for i in range(nops):
            f2 = struct.unpack_from(MOP_FMT, buf, at + op_off + i * MOP_SIZE)
            t, k = f2[0], f2[1]
            pos = list(f2[2:10])
            mat, cmt, cmg = f2[11], f2[12], f2[13]
            p.ops.append(MicroOp(MOP_NAMES[t], k, pos[:max(k, 1)], [], mat, cmt, cmg))
        p.pool = np.frombuffer(buf, dtype=np.complex128, count=pool_n, offset=at + pool_off).copy()
        out.append(p)
        at += nbytes
    return out
