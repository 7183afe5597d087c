"""Sharded state vector against the oracle.

Each rank is a process; the communicator id is created in the parent.  With
>= world visible GPUs every rank owns one GPU and the ranks talk NCCL; on a
box with fewer GPUs the same cases run with every rank on GPU 0 and
NQ_COMM=host (ranks coordinate through host shared memory; exchanges still go
through CUDA-IPC peer memory), except the forms that need one GPU per rank
(staged exchanges: two ranks' cooperative grids cannot share a GPU; NCCL).
"""
import os
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2401_06861_b200 import abi

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _uid(shared):
    """The communicator id, made the way the ranks will use it (NQ_COMM is
    read when the id is made: an NCCL id, or random bytes naming the
    shared-memory block)."""
    old = os.environ.get("NQ_COMM")
    if shared:
        os.environ["NQ_COMM"] = "host"
    try:
        return abi.comm_unique_id()
    finally:
        if old is None:
            os.environ.pop("NQ_COMM", None)
        else:
            os.environ["NQ_COMM"] = old


def _mode(world, fused="1", exchange="p2p"):
    """(shared_gpu, skip reason): one GPU per rank when there are enough,
    else every rank on GPU 0 with host coordination."""
    if abi.device_count() >= world:
        return False, None
    if fused == "staged" or exchange == "nccl":
        return True, f"needs {world} GPUs ({fused} / {exchange})"
    return True, None


def _setup_rank(rank, shared):
    if shared:
        os.environ["NQ_COMM"] = "host"
    return 0 if shared else rank


def _rank_main(rank, world, uid, n, seed, outdir, fused="1", exchange="p2p", shared=False):
    os.environ["NQ_FUSED_EXCHANGE"] = fused
    os.environ["NQ_EXCHANGE"] = exchange
    dev = _setup_rank(rank, shared)
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    from oracle import Port
    from paper_2401_06861_b200 import abi as A

    port = Port()
    ops = port.random_circuit(seed, n, 300)
    sv = A.SV.sharded(n, rank, world, uid, device=dev)
    sv.apply(ops)
    norm = sv.norm_sq()
    rng = np.random.default_rng(seed)
    terms = [("".join(rng.choice(list("IXYZ"), size=n)), float(rng.uniform(-1, 1))) for _ in range(12)]
    g = world.bit_length() - 1
    terms.append(("X" * (n - g) + "Z" * g, 0.5))  # flips every local qubit's worth
    ex = sv.expectations(terms)
    u = np.sort(port.rng_double(99, 4000))
    idx, cnt = sv.sample_sorted(u)
    amps = sv.amplitudes()
    probs = sv.probabilities()
    # set_amplitudes: every rank passes the whole vector, then more gates
    srng = np.random.default_rng(seed + 1)
    psi = srng.normal(size=1 << n) + 1j * srng.normal(size=1 << n)
    psi /= np.linalg.norm(psi)
    sv.set_amplitudes(psi)
    more = port.random_circuit(seed + 2, n, 120)
    sv.apply(more)
    after = sv.amplitudes()
    stats = sv.comm_stats()
    np.savez(os.path.join(outdir, f"r{rank}.npz"), norm=norm, ex=ex, idx=idx, cnt=cnt, amps=amps, probs=probs,
             psi=psi, after=after,
             exchanges=stats["exchanges"], fused=stats["fused"], alt=stats["alt_buffer"], staged=stats["staged"],
             letters=np.array([t[0] for t in terms]),
             coeff=np.array([t[1] for t in terms]))


@pytest.mark.parametrize("n,world,fused,exchange", [(14, 2, "1", "p2p"), (20, 2, "1", "p2p"),
                                                    (20, 2, "staged", "p2p"), (21, 2, "staged", "p2p"),
                                                    (20, 2, "0", "p2p"), (20, 2, "0", "nccl"),
                                                    (22, 4, "1", "p2p"), (22, 4, "staged", "p2p"),
                                                    (22, 4, "0", "p2p"), (22, 4, "0", "nccl")])
def test_sharded_gpus(port, tmp_path, n, world, fused, exchange):
    """Sharded run == oracle (amplitudes, norm, expectations, sampling), with
    exchanges fused into the preceding pass (out-of-place exchange stores into
    the partner's second buffer, or staged: in place + staging ring + pusher
    kernel, the form used when no second copy fits), as standalone peer-memory swaps, or through
    the NCCL send/recv fallback (NQ_EXCHANGE=nccl: pack, send/recv through
    bounce buffers, unpack -- the path taken when CUDA IPC is unavailable)."""
    shared, why = _mode(world, fused, exchange)
    if why:
        pytest.skip(why)
    seed = 808 + n
    uid = _uid(shared)
    mp.start_processes(_rank_main, args=(world, uid, n, seed, str(tmp_path), fused, exchange, shared), nprocs=world,
                       start_method="spawn")
    ops = port.random_circuit(seed, n, 300)
    want = port.sv_run(n, ops)
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        assert int(d["exchanges"]) > 0
        if fused == "1":
            assert bool(d["alt"]) and int(d["fused"]) > 0, (d["alt"], d["fused"])
        elif fused == "staged":
            assert bool(d["staged"]) and not bool(d["alt"]) and int(d["fused"]) > 0
        else:
            assert int(d["fused"]) == 0
        np.testing.assert_allclose(d["amps"], want, atol=1e-10, rtol=0)
        np.testing.assert_allclose(d["probs"], np.abs(want) ** 2, atol=1e-12, rtol=0)
        more = port.random_circuit(seed + 2, n, 120)
        np.testing.assert_allclose(d["after"], port.sv_apply(d["psi"].copy(), more), atol=1e-10, rtol=0)
        assert abs(float(d["norm"]) - 1.0) < 1e-10
        ref = [port.expectation(want, str(L), float(c)) for L, c in zip(d["letters"], d["coeff"])]
        np.testing.assert_allclose(d["ex"], ref, atol=1e-10, rtol=0)
        dense = np.zeros(1 << n, dtype=np.uint64)
        dense[d["idx"].astype(np.int64)] = d["cnt"]
        assert np.array_equal(dense, port.sample_distribution(np.abs(want) ** 2, 4000, 99))


def _env_rank(rank, world, uid, outdir, shared=False):
    # rank 1 plans with a different tile size: the ranks' flushes would diverge
    dev = _setup_rank(rank, shared)
    if rank == 1:
        os.environ["NQ_TILE_SV"] = "10"
    sys.path[:0] = [ROOT]
    from paper_2401_06861_b200 import abi as A

    try:
        A.SV.sharded(16, rank, world, uid, device=dev)
        msg = "created"
    except A.ContractError as e:
        msg = str(e)
    with open(os.path.join(outdir, f"env{rank}.txt"), "w") as f:
        f.write(msg)


def test_ranks_must_share_the_environment(tmp_path):
    """Every rank plans its own flushes, so creation fails on every rank (a
    contract error, not a later collective hang) when the plan-shaping NQ_*
    options differ between ranks."""
    shared, _ = _mode(2)
    uid = _uid(shared)
    mp.start_processes(_env_rank, args=(2, uid, str(tmp_path), shared), nprocs=2, start_method="spawn")
    for r in range(2):
        msg = (tmp_path / f"env{r}.txt").read_text()
        assert "different NQ_* options" in msg, msg


def _repeat_rank(rank, world, uid, n, seed, outdir, fused, shared=False):
    os.environ["NQ_FUSED_EXCHANGE"] = fused
    dev = _setup_rank(rank, shared)
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    from oracle import Port
    from paper_2401_06861_b200 import abi as A

    ops = Port().random_circuit(seed, n, 200)
    sv = A.SV.sharded(n, rank, world, uid, device=dev)
    for _ in range(4):  # the same circuit flushed again and again (benchmark / iterative shape)
        sv.apply(ops)
        sv.norm_sq()
    stats = sv.comm_stats()
    np.savez(os.path.join(outdir, f"rep{rank}.npz"), amps=sv.amplitudes(), exchanges=stats["exchanges"],
             fused=stats["fused"])


@pytest.mark.parametrize("n,world,fused", [(20, 2, "1"), (20, 2, "staged"), (22, 4, "staged"), (22, 4, "0")])
def test_sharded_repeated_flushes(port, tmp_path, n, world, fused):
    """Repeated flushes of one circuit carry the qubit map from flush to flush
    and move the next flush's opening exchange to the end of the current one
    (where it fuses into the last pass): the state after four repetitions
    equals the oracle's."""
    shared, why = _mode(world, fused)
    if why:
        pytest.skip(why)
    seed = 909 + n
    uid = _uid(shared)
    mp.start_processes(_repeat_rank, args=(world, uid, n, seed, str(tmp_path), fused, shared), nprocs=world,
                       start_method="spawn")
    ops = port.random_circuit(seed, n, 200)
    want = port.sv_run(n, np.concatenate([ops] * 4))
    for r in range(world):
        d = np.load(tmp_path / f"rep{r}.npz")
        np.testing.assert_allclose(d["amps"], want, atol=1e-10, rtol=0)
        assert int(d["exchanges"]) > 0
