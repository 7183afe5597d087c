"""Regenerate the golden fixtures in tests/golden/ (run in the build container).

Sources -- never the code under test:
* every_gate_numpy_model.npy: the reference's own independent numpy model,
  executed from /root/reference/proj/tests/python/test_reference.py
  (its ``reference_state()``; the module's ``import naqs`` is stripped).
* ref_*.npz: the reference engine compiled unmodified from its sources
  (oracle/_ref/libnaqs_ref.so, oracle/Makefile) on seeded inputs.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import NoiseSpec, Ref  # noqa: E402

REF_PY = "/root/reference/proj/tests/python/test_reference.py"


def every_gate():
    src = open(REF_PY).read().replace("import naqs\n", "")
    ns = {}
    exec(compile(src, REF_PY, "exec"), ns)
    return ns["reference_state"]()


def main():
    ref = Ref()
    files = {}
    np.save(os.path.join(HERE, "every_gate_numpy_model.npy"), every_gate())
    files["every_gate_numpy_model.npy"] = "proj/tests/python/test_reference.py:48-124 reference_state()"

    # state vector: test_util random circuits
    for n, seed, depth in [(10, 2024, 200), (16, 4040, 300)]:
        ops = ref.random_circuit(seed, n, depth)
        amps = ref.sv_run(n, ops)
        rng = np.random.default_rng(seed)
        terms = [("".join(rng.choice(list("IXYZ"), size=n)), float(rng.uniform(-2, 2))) for _ in range(24)]
        vals = ref.sv_expectations(n, ops, terms)
        counts = ref.sv_sample(n, ops, 20000, 7)
        name = f"ref_sv_n{n}_s{seed}_d{depth}.npz"
        np.savez_compressed(os.path.join(HERE, name), ops=ops, amps=amps, letters=np.array([t[0] for t in terms]),
                            coeff=np.array([t[1] for t in terms]), expect=vals, counts=counts)
        files[name] = f"reference sv_run / expectation / sample(20000, 7) on random_circuit(Rng({seed}), {n}, {depth})"

    # density matrix with the synthetic calibration
    for n, seed in [(4, 11), (6, 12)]:
        ops = ref.random_circuit(seed, n, 60, 2)
        noise = NoiseSpec(n)
        rho = ref.dm_run_noisy(n, ops, noise)
        rng = np.random.default_rng(seed)
        terms = [("".join(rng.choice(list("IXYZ"), size=n)), float(rng.uniform(-2, 2))) for _ in range(16)]
        scal, ex, probs = ref.dm_noisy_reductions(n, ops, noise, terms)
        name = f"ref_dm_noisy_n{n}_s{seed}.npz"
        np.savez_compressed(os.path.join(HERE, name), ops=ops, rho=rho, scalars=scal, expect=ex, probs=probs,
                            letters=np.array([t[0] for t in terms]), coeff=np.array([t[1] for t in terms]))
        files[name] = f"reference dm_run_noisy + trace/purity/hermiticity/expectation/probabilities, n={n}"

    # readout
    rng = np.random.default_rng(5)
    p = rng.random(1 << 8)
    p /= p.sum()
    p01 = rng.uniform(0, 0.08, 8)
    p10 = rng.uniform(0, 0.08, 8)
    out = ref.readout_apply_dist(p, p01, p10)
    np.savez_compressed(os.path.join(HERE, "ref_readout_n8.npz"), dist=p, p01=p01, p10=p10, out=out)
    files["ref_readout_n8.npz"] = "reference readout_apply_dist on a random 8-qubit distribution"

    with open(os.path.join(HERE, "MANIFEST.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py", "files": files}, f, indent=1)


if __name__ == "__main__":
    main()
