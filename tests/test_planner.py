"""Host-side fusion planner, CPU only (no GPU needed).

The planner's output (pass records, nq_plan_debug) is executed here by a
numpy emulator of the micro-op semantics documented in csrc/engine.hpp and
compared with the oracle.  This validates pass windows (commutation-safe
deferral), tile bit selection, fusion and serialisation independently of the
kernels; the GPU tests then validate the kernels on the same plans.
"""
import numpy as np
import pytest

from paper_2401_06861_b200 import abi, plan_format


def ins0(w, b):
    return ((w >> b) << (b + 1)) | (w & ((1 << b) - 1))


def deposit(v, pos):
    r = 0
    for j, p in enumerate(pos):
        if (v >> j) & 1:
            r |= 1 << p
    return r


def run_plan(n, passes, amps):
    """Numpy emulator of the pass records (semantics of csrc/engine.hpp).
    Relabelling passes store tile bit i at qst[i]; the result is returned in
    logical qubit order (the final layout undone)."""
    a = amps.copy()
    p2l = list(range(n))  # physical bit -> logical qubit
    for p in passes:
        size = 1 << p.m
        offs = np.array([deposit(e, p.q) for e in range(size)], dtype=np.int64)
        qst = p.qst if p.qst else p.q
        assert sorted(qst) == sorted(p.q)
        offs_st = np.array([deposit(e, qst) for e in range(size)], dtype=np.int64)
        lab = p.lab if p.lab else list(range(p.m))
        new = list(p2l)
        for i in range(p.m):
            new[qst[i]] = p2l[p.q[lab[i]]]
        p2l = new
        assert p.ops[0].type == "layout"
        for r in range(p.ntiles):
            base = deposit(r, p.rest)
            t = a[base + offs].copy()
            lay = None
            for op in p.ops:
                if op.type == "layout":
                    lay = op.pos[: op.k]
                    assert lay == sorted(lay)
                    continue
                apply_mop(op, t, p.pool, base, p.m, lay)
            a[base + offs_st] = t
    if p2l != list(range(n)):
        l2p = [0] * n
        for ph, lq in enumerate(p2l):
            l2p[lq] = ph
        idx = np.array([deposit(x, l2p) for x in range(1 << n)], dtype=np.int64)
        a = a[idx]
    return a


def apply_mop(op, t, pool, full, m, lay):
    size = 1 << m
    e = np.arange(size)
    # register-slot ops address tile bits through the current layout
    tp = [lay[s] for s in op.pos[: op.k]] if op.type in ("dense", "xperm", "swap", "depol") else None
    if op.type == "dense":
        assert op.pos[: op.k] == sorted(op.pos[: op.k])
        k = op.k
        D = 1 << k
        U = pool[op.mat:op.mat + D * D].reshape(D, D)
        mask = sum(1 << b for b in tp)
        bases = e[(e & mask) == 0]
        idx = np.stack([bases | deposit(l, tp) for l in range(D)])  # D x G
        t[idx] = U @ t[idx]
    elif op.type == "diag":
        k = op.k
        tab = pool[op.mat:op.mat + (1 << k)]
        idx = np.zeros(size, dtype=np.int64)
        for j in range(k):
            if op.pos[j] >= 0:
                idx |= ((e >> op.pos[j]) & 1) << j
            else:
                idx |= ((full >> (-1 - op.pos[j])) & 1) << j
        t *= tab[idx]
    elif op.type == "xperm":
        if (full & op.cmask_glob) != op.cmask_glob:
            return
        b = 1 << tp[0]
        sel = e[((e & b) == 0) & ((e & op.cmask_tile) == op.cmask_tile)]
        t[sel], t[sel | b] = t[sel | b].copy(), t[sel].copy()
    elif op.type == "swap":
        b0, b1 = 1 << tp[0], 1 << tp[1]
        sel = e[((e & b0) != 0) & ((e & b1) == 0)]
        other = (sel & ~b0) | b1
        t[sel], t[other] = t[other].copy(), t[sel].copy()
    else:
        raise AssertionError(op.type)


@pytest.mark.parametrize("n,tile", [(3, 12), (6, 4), (8, 5), (10, 6), (12, 8), (12, 12)])
@pytest.mark.parametrize("fuse", [True, False])
def test_plan_emulation_matches_oracle(port, n, tile, fuse):
    for seed in range(3):
        ops = port.random_circuit(5000 + 10 * n + seed, n, 150)
        passes = plan_format.decode(abi.plan_debug(n, ops, tile_qubits=tile, fuse=fuse))
        a0 = np.zeros(1 << n, dtype=complex)
        a0[0] = 1
        got = run_plan(n, passes, a0)
        np.testing.assert_allclose(got, port.sv_run(n, ops), atol=1e-10, rtol=0)


@pytest.mark.parametrize("n,tile", [(12, 8), (14, 9), (16, 11), (13, 6)])
def test_relabelling_plans_match_oracle(port, n, tile):
    """Relabelling stores (low physical bits hold a per-pass choice of
    qubits): emulated plan, final layout undone, equals the oracle; the
    relabelled plan never needs more passes than the plain one."""
    for seed in range(3):
        ops = port.random_circuit(7100 + n + seed, n, 200)
        plain = plan_format.decode(abi.plan_debug(n, ops, tile_qubits=tile))
        passes = plan_format.decode(abi.plan_debug(n, ops, tile_qubits=tile, relabel=True))
        assert any(p.qst != p.q for p in passes)
        lb = max(0, min(4, tile - 4))
        for p in passes:
            assert p.q[:lb] == list(range(lb))  # the physical low bits stay in every tile
        a0 = np.zeros(1 << n, dtype=complex)
        a0[0] = 1
        got = run_plan(n, passes, a0)
        np.testing.assert_allclose(got, port.sv_run(n, ops), atol=1e-10, rtol=0)
        assert len(passes) <= len(plain) + 1


def test_tile_sets_respect_coalescing_and_capacity(port):
    n, tile = 20, 10
    ops = port.random_circuit(1, n, 300)
    passes = plan_format.decode(abi.plan_debug(n, ops, tile_qubits=tile))
    for p in passes:
        assert p.m == tile
        assert p.q[:4] == [0, 1, 2, 3]  # >= 4 contiguous low bits: 256-byte runs
        assert sorted(p.q) == p.q and len(set(p.q)) == tile
        assert set(p.q).isdisjoint(p.rest) and len(p.q) + len(p.rest) == n
        for op in p.ops:
            if op.type in ("dense", "xperm", "swap"):
                assert all(0 <= x < tile for x in op.pos[: op.k])


def test_fusion_reduces_passes_and_microops(port):
    n = 24
    ops = port.random_circuit(2024, n, 200)
    fused = plan_format.decode(abi.plan_debug(n, ops, tile_qubits=12, fuse=True))
    unfused = plan_format.decode(abi.plan_debug(n, ops, tile_qubits=12, fuse=False))
    assert len(fused) == len(unfused)
    assert sum(len(p.ops) for p in fused) < sum(len(p.ops) for p in unfused)
    assert len(fused) < 200 / 5  # far fewer state sweeps than gates


def test_diagonals_never_force_tile_bits():
    # a run of RZ/CZ on high qubits fits in one pass with only low tile bits
    n = 20
    ops = [("rz", [q], [0.1 * q]) for q in range(n)] + [("cz", [q, (q + 7) % n]) for q in range(n)]
    passes = plan_format.decode(abi.plan_debug(n, ops, tile_qubits=8))
    assert len(passes) == 1
    assert passes[0].q == list(range(8))


def test_plan_rejects_bad_ops():
    with pytest.raises(abi.ContractError):
        abi.plan_debug(4, [("cx", [0, 4])])
    with pytest.raises(abi.ContractError):
        abi.plan_debug(4, [("measure", [0])])


def test_cancelled_permutation_pairs_respect_dense_work_on_controls(port):
    """P U P with U dense on a control of P does not cancel (regression: the
    sandwich check once only looked at pending work on the target;
    CX(c,t) U3(c) CX(c,t) was folded into U3(c))."""
    n = 5
    circ = [("h", [2], []), ("cx", [0, 2], []), ("u3", [0], [-0.6, -2.75, 1.79]), ("cx", [0, 2], []),
            ("ccx", [0, 1, 3], []), ("ry", [1], [0.7]), ("ccx", [0, 1, 3], [])]
    a0 = np.zeros(1 << n, dtype=complex)
    a0[0] = 1
    for tile in (3, 4, 5):
        passes = plan_format.decode(abi.plan_debug(n, circ, tile_qubits=tile))
        np.testing.assert_allclose(run_plan(n, passes, a0), port.sv_run(n, circ), atol=1e-12, rtol=0)


@pytest.mark.parametrize("block", range(4))
def test_plan_fuzz_against_oracle(port, block):
    """Seeded random plans (uniform gate mix and permutation-heavy mixes,
    random qubit counts and tile sizes, with and without relabelling) emulated
    against the oracle."""
    from oracle import ops_to_list

    kinds = [("cx", 2, 0), ("cx", 2, 0), ("ccx", 3, 0), ("swap", 2, 0), ("x", 1, 0), ("y", 1, 0), ("ry", 1, 1),
             ("u3", 1, 3), ("h", 1, 0), ("t", 1, 0), ("rz", 1, 1), ("cz", 2, 0), ("s", 1, 0)]
    for seed in range(block * 25, block * 25 + 25):
        rng = np.random.default_rng(1000 + seed)
        n = int(rng.integers(5, 10))
        tile = int(rng.integers(3, min(n, 8) + 1))
        if seed % 2:
            circ = []
            for _ in range(150):
                k, ar, npar = kinds[int(rng.integers(len(kinds)))]
                qs = [int(q) for q in rng.choice(n, size=ar, replace=False)]
                circ.append((k, qs, [float(v) for v in rng.uniform(-3, 3, size=npar)]))
        else:
            circ = [tuple(x) for x in ops_to_list(port.random_circuit(seed, n, 150))]
        a0 = np.zeros(1 << n, dtype=complex)
        a0[0] = 1
        want = port.sv_run(n, circ)
        for relabel in (False, True):
            passes = plan_format.decode(abi.plan_debug(n, circ, tile_qubits=tile, relabel=relabel))
            err = np.max(np.abs(run_plan(n, passes, a0) - want))
            assert err <= 1e-10, (seed, n, tile, relabel, err)
