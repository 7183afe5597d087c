"""Multi-GPU layer, host side, on CPU (no GPU, no NCCL).

The sharded flush's schedule (csrc/shard.cpp: segments of local work in
PHYSICAL bits + global<->local exchanges + the exchanges restoring the
identity map) comes from nq_shard_debug.  Here it is executed by a numpy
model of the ranks -- in one process, and over torch.distributed "gloo" with
world size 2 exchanging real half-shards -- and the assembled state must equal
the oracle's.  This validates victim selection, the qubit map, controls and
diagonals on global bits (rank-extended indices) and the exchange index math
(which half is sent, where it lands) independently of the CUDA kernels.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_06861_b200 import abi


def apply_elem(a, rank, nloc, op):
    """One elementary op on rank's shard (local array a), physical bits."""
    kind, k, bits, ctrl, mat = op
    L = len(a)
    loc = np.arange(L, dtype=np.int64)
    full = (rank << nloc) | loc
    if kind == "nop":
        return
    if kind == "diag":
        idx = np.zeros(L, dtype=np.int64)
        for j, b in enumerate(bits):
            idx |= ((full >> b) & 1) << j
        a *= mat[idx]
        return
    if kind == "xperm":
        t = 1 << bits[0]
        assert bits[0] < nloc
        sel = loc[((loc & t) == 0) & ((full & ctrl) == ctrl)]
        a[sel], a[sel | t] = a[sel | t].copy(), a[sel].copy()
        return
    if kind == "swap":
        b0, b1 = 1 << bits[0], 1 << bits[1]
        assert max(bits) < nloc
        sel = loc[((loc & b0) != 0) & ((loc & b1) == 0)]
        o = (sel & ~b0) | b1
        a[sel], a[o] = a[o].copy(), a[sel].copy()
        return
    if kind == "dense":
        assert max(bits) < nloc
        D = 1 << k
        U = mat.reshape(D, D)
        mask = sum(1 << b for b in bits)
        base = loc[(loc & mask) == 0]
        idx = np.stack([base | sum(((l >> j) & 1) << b for j, b in enumerate(bits)) for l in range(D)])
        a[idx] = U @ a[idx]
        return
    raise AssertionError(kind)


def half_indices(nloc, v, val):
    k = np.arange(1 << (nloc - 1), dtype=np.int64)
    return ((k >> v) << (v + 1)) | (val << v) | (k & ((1 << v) - 1))


def run_schedule_single(n, world, acts):
    g = world.bit_length() - 1
    nloc = n - g
    shards = [np.zeros(1 << nloc, dtype=complex) for _ in range(world)]
    shards[0][0] = 1.0
    exchanges = 0
    for act in acts:
        if act[0] == "segment":
            for r in range(world):
                for op in act[1]:
                    apply_elem(shards[r], r, nloc, op)
        else:
            _, gb, v = act
            j = gb - nloc
            assert j >= 0 and v < nloc
            exchanges += 1
            new = [s.copy() for s in shards]
            for r in range(world):
                p = r ^ (1 << j)
                b = (r >> j) & 1
                mine = half_indices(nloc, v, 1 - b)
                theirs = half_indices(nloc, v, 1 - ((p >> j) & 1))
                new[r][mine] = shards[p][theirs]
            shards = new
    return np.concatenate(shards), exchanges


@pytest.mark.parametrize("n,world", [(6, 2), (8, 2), (8, 4), (10, 8), (12, 4), (16, 4)])
def test_sharded_schedule_matches_oracle(port, n, world):
    for seed in range(3):
        ops = port.random_circuit(70 + 13 * n + seed, n, 120)
        acts = abi.shard_debug(n, world, ops)
        state, ex = run_schedule_single(n, world, acts)
        np.testing.assert_allclose(state, port.sv_run(n, ops), atol=1e-10, rtol=0)
        assert ex > 0  # the random circuits do touch global qubits


@pytest.mark.parametrize("n,world,seed", [(16, 4, 0), (16, 4, 2), (20, 4, 2)])
def test_rebalanced_segments_match_oracle(port, n, world, seed):
    """Ops moved across an exchange (csrc/shard.cpp rebalance: bits translated
    g <-> v, order kept) give the same state; these cases do move ops."""
    ops = port.random_circuit(70 + 13 * n + seed, n, 120)
    plain = abi.shard_debug(n, world, ops, rebalance=False)
    moved = abi.shard_debug(n, world, ops, rebalance=True)
    sizes = lambda acts: [len(a[1]) if a[0] == "segment" else "X" for a in acts]  # noqa: E731
    assert sizes(plain) != sizes(moved)
    assert sum(len(a[1]) for a in plain if a[0] == "segment") == sum(len(a[1]) for a in moved if a[0] == "segment")
    want = port.sv_run(n, ops)
    for acts in (plain, moved):
        state, _ = run_schedule_single(n, world, acts)
        np.testing.assert_allclose(state, want, atol=1e-10, rtol=0)


def test_diagonal_and_control_on_global_bits_need_no_exchange(port):
    n, world = 10, 4
    ops = [("h", [q]) for q in range(8)] + [("rz", [9], [0.3]), ("cz", [8, 2]), ("cx", [9, 1]), ("ccx", [8, 9, 0]),
                                           ("t", [8]), ("u1", [9], [1.1])]
    acts = abi.shard_debug(n, world, ops)
    assert all(a[0] == "segment" for a in acts)
    state, ex = run_schedule_single(n, world, acts)
    assert ex == 0
    np.testing.assert_allclose(state, port.sv_run(n, ops), atol=1e-12, rtol=0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, n, seed, result_path):
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    from oracle import Port

    ops = Port().random_circuit(seed, n, 150)
    acts = abi.shard_debug(n, world, ops)
    nloc = n - (world.bit_length() - 1)
    a = np.zeros(1 << nloc, dtype=complex)
    if rank == 0:
        a[0] = 1.0
    for act in acts:
        if act[0] == "segment":
            for op in act[1]:
                apply_elem(a, rank, nloc, op)
            continue
        _, gb, v = act
        j = gb - nloc
        partner = rank ^ (1 << j)
        idx = half_indices(nloc, v, 1 - ((rank >> j) & 1))
        send = torch.from_numpy(np.ascontiguousarray(a[idx]).view(np.float64).copy())
        recv = torch.empty_like(send)
        reqs = [dist.isend(send, partner), dist.irecv(recv, partner)]
        for rq in reqs:
            rq.wait()
        a[idx] = recv.numpy().view(np.complex128)
    parts = [torch.empty(2 * len(a), dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(a.view(np.float64).copy()))
    if rank == 0:
        full = np.concatenate([p.numpy().view(np.complex128) for p in parts])
        np.save(result_path, full)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_schedule_over_gloo(port, tmp_path, world):
    n, seed = 9, 4242
    out = str(tmp_path / "state.npy")
    mp.start_processes(_gloo_worker, args=(world, _free_port(), n, seed, out), nprocs=world, start_method="spawn")
    got = np.load(out)
    np.testing.assert_allclose(got, port.sv_run(n, port.random_circuit(seed, n, 150)), atol=1e-10, rtol=0)
