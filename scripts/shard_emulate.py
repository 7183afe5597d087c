"""CPU emulation of the steady state of repeated sharded flushes (no GPU).

Restates csrc/shard.cpp::schedule() (Belady victim: the local qubit whose next
non-diagonal use is farthest, ties to the highest bit; the qubit map carried
from flush to flush) for the benchmark's random circuit, runs it for a number
of repetitions, and plans each steady-state segment with the real planner
(abi.plan_debug) to count passes.  Usage:

    python scripts/shard_emulate.py [local_qubits] [global_qubits] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_06861_b200 import abi, plan_format, workloads  # noqa: E402

DIAG = {"z", "s", "sdg", "t", "tdg", "rz", "u1", "cz", "id", "barrier"}


def need(op):
    k, qs, _ = op
    if k in DIAG:
        return set()
    if k == "cx":
        return {qs[1]}
    if k == "ccx":
        return {qs[2]}
    return set(qs)


def steady(nl, g, reps, seed=2024, depth=200):
    n = nl + g
    ops = workloads.random_circuit(seed, n, depth)
    needs = [need(o) for o in ops]
    l2p, p2l = list(range(n)), list(range(n))
    for rep in range(reps):
        segs, cur, exch = [], [], []
        for i, nb in enumerate(needs):
            glob = sorted(l2p[q] for q in nb if l2p[q] >= nl)
            if glob:
                segs.append(cur)
                cur = []
            for gp in glob:
                best, bd = -1, -1
                for v in range(nl - 1, -1, -1):
                    lq = p2l[v]
                    if lq in nb:
                        continue
                    d = next((j for j in range(i + 1, len(ops)) if lq in needs[j]), len(ops) + 1)
                    if d > bd:
                        best, bd = v, d
                la, lb = p2l[gp], p2l[best]
                p2l[gp], p2l[best] = lb, la
                l2p[la], l2p[lb] = best, gp
                exch.append((i, gp, best))
            k, qs, ps = ops[i]
            cur.append((k, [l2p[q] for q in qs], ps))
        segs.append(cur)
        yield rep, segs, exch


def passes(n, seg):
    return len(plan_format.decode(abi.plan_debug(n, abi.make_ops(seg), 11))) if seg else 0


if __name__ == "__main__":
    nl = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    g = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 12
    n = nl + g
    for rep, segs, exch in steady(nl, g, reps):
        print(f"rep {rep}: exchanges {len(exch)} at ops {[e[0] for e in exch]}; segment passes "
              f"{[passes(n, s) for s in segs]} (before rebalancing)")
    print("unsharded plan of the same circuit:", passes(n, workloads.random_circuit(2024, n, 200)), "passes")
