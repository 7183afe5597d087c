"""Sharded state vector over 2 GPUs (NCCL) against the oracle.

Needs >= 2 visible GPUs (gpurun --gpus 2); skipped otherwise.  Each rank is a
process owning one GPU; the NCCL unique id is created in the parent.
"""
import os
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2401_06861_b200 import abi

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rank_main(rank, world, uid, n, seed, outdir, fused=True):
    os.environ["NQ_FUSED_EXCHANGE"] = "1" if fused else "0"
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    from oracle import Port
    from paper_2401_06861_b200 import abi as A

    port = Port()
    ops = port.random_circuit(seed, n, 300)
    sv = A.SV.sharded(n, rank, world, uid, device=rank)
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
             exchanges=stats["exchanges"], fused=stats["fused"], alt=stats["alt_buffer"],
             letters=np.array([t[0] for t in terms]),
             coeff=np.array([t[1] for t in terms]))


@pytest.mark.parametrize("n,world,fused", [(14, 2, True), (20, 2, True), (20, 2, False), (22, 4, True),
                                           (22, 4, False)])
def test_sharded_gpus(port, tmp_path, n, world, fused):
    """Sharded run == oracle (amplitudes, norm, expectations, sampling), with
    exchanges fused into the preceding pass (out-of-place exchange stores into
    the partner's second buffer) or as standalone peer-memory swaps."""
    if abi.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    seed = 808 + n
    uid = abi.comm_unique_id()
    mp.start_processes(_rank_main, args=(world, uid, n, seed, str(tmp_path), fused), nprocs=world,
                       start_method="spawn")
    ops = port.random_circuit(seed, n, 300)
    want = port.sv_run(n, ops)
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        assert int(d["exchanges"]) > 0
        if fused:
            assert bool(d["alt"]) and int(d["fused"]) > 0
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
