#!/usr/bin/env python
"""Benchmark of the B200 SV/DM simulation core (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Headline workload: the reference's seeded random circuit
(proj/tests/test_util.hpp generator, Rng(2024)), 30 qubits, depth 200, on one
B200.  One step = the whole circuit applied to the HBM-resident 2^30-amplitude
state through the C ABI (fusion planning + fused passes).  Metric: source
gates per second (whole job), plus achieved HBM GB/s.

* value     device time of K steps (CUDA events on the library's stream),
            barrier + synchronize on both sides, max over ranks.
* e2e       the same steps through the reference-facing C ABI with host
            buffers: each step copies its op list host->device (pinned
            staging) and reads a <Z_0> expectation back device->host; timed
            on the host clock around synchronised steps, max over ranks.
* roofline  the fused-pass kernel: algorithmic bytes per launch (32 * 2^n:
            every amplitude read and written once) / its average CUDA-event
            duration inside the timed region, against MEASURED_PEAKS.json.
* cpu_baseline  the reference engine compiled from its own sources
            (oracle/_ref, kind "reference"; the C restatement "port" if that
            build is absent), on the host cores, on a bounded prefix of the
            same circuit.
For N > 1 (torchrun) the state is ONE sharded state of 30 + log2(N) qubits
(2^30 amplitudes per GPU: weak scaling); non-diagonal gates on the log2(N)
global qubits trigger half-shard exchanges over NVLink peer memory, fused into
the preceding pass when a second copy of the shard fits.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--qubits", type=int, default=30)
    ap.add_argument("--depth", type=int, default=200)
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--cpu-ops", type=int, default=12, help="ops of the circuit prefix timed on the CPU")
    return ap.parse_args()


# ---------------------------------------------------------------------------
def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as td

        torch.cuda.set_device(local)
        td.init_process_group("nccl")
        dist = td
    return world, rank, local, dist


def barrier(dist, local):
    if dist is not None:
        import torch

        dist.barrier(device_ids=[local])
        torch.cuda.synchronize()


def max_over_ranks(dist, local, v: float) -> float:
    if dist is None:
        return v
    import torch

    t = torch.tensor([v], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []  # (host time, csv line)
        self.t_start = self.t_end = None

    # nvidia-smi needs ~1 s to start streaming: the sampler is started before
    # the warm-up and only samples stamped inside [mark_start, mark_end] count.
    def mark_start(self):
        self.t_start = time.time()

    def mark_end(self):
        self.t_end = time.time()

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.device)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lo = self.t_start if self.t_start is not None else -1e30
        hi = (self.t_end if self.t_end is not None else 1e30) + 0.05
        window = [ln for t, ln in self.lines if lo <= t <= hi]
        for ln in window:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def traffic_from_profiles():
    """dram bytes per pass launch from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------
def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def host_mem_gib() -> float:
    try:
        with open("/proc/meminfo") as f:
            for ln in f:
                if ln.startswith("MemAvailable:"):
                    return int(ln.split()[1]) / (1 << 20)
    except OSError:
        pass
    return 0.0


def cpu_reference_rate(n: int, ops, n_ops: int, reps: int):
    """Gates/s of the reference engine on the host: `reps` timed runs of the
    first `n_ops` ops on one persistent n-qubit state (all host threads)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    from oracle import Port, Ref, list_to_ops  # checker / baseline only

    need = (16 << n) / (1 << 30) * 1.3 + 2
    if host_mem_gib() < need:
        return None, f"host RAM {host_mem_gib():.0f} GiB < {need:.0f} GiB needed for n={n}"
    arr = list_to_ops(ops[:n_ops])
    cores = cpu_threads()
    if Ref.available():
        ref = Ref()
        ref.set_threads(cores)
        h = ref.sv_new(n)
        try:
            times = [ref.sv_run_timed(h, arr) for _ in range(reps)]
        finally:
            ref.sv_free(h)
        kind = "reference"
    else:
        port = Port()
        amps = np.zeros(1 << n, dtype=np.complex128)
        amps[0] = 1
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            port.sv_apply(amps, arr)
            times.append((time.perf_counter() - t0) * 1e3)
        kind, cores = "port", 1
    ms = statistics.median(times)
    return {"value": n_ops / (ms / 1e3), "unit": "gates/s", "cores": cores, "kind": kind,
            "sample": f"first {n_ops} ops of random_circuit(Rng(2024), n={n}, depth=200) on one persistent "
                      f"2^{n} state, median of {reps} runs, OMP threads={cores}",
            "ms_per_run": ms}, None


def run_reference_arm(args, world, rank):
    if rank != 0:
        return 0
    from paper_2401_06861_b200 import workloads

    # The b200 arm runs 30 + log2(N) qubits on N GPUs and reports 30-qubit
    # gate equivalents (a gate on 2^(30+g) amplitudes counts 2^g).  The
    # reference rejects n > 30 (proj/include/naqs/statevector.hpp:22), so it is
    # timed at n = 30, where its rate is already in that unit.
    n = args.qubits
    ops = workloads.random_circuit(args.seed, n, args.depth)
    # bounded sample: fewer ops per step as the state doubles (a few s per step)
    k = max(1, min(args.cpu_ops >> max(0, n - 30), len(ops)))
    total_steps = args.warmup + args.steps
    res, why = cpu_reference_rate(n, ops, k, total_steps)
    base = {"metric": "SV gates/s (random circuit, depth 200)", "unit": "gates/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "config": {"workload": f"random_circuit(Rng({args.seed})) n={args.qubits} depth={args.depth} "
                                   f"(proj/tests/test_util.hpp generator)",
                       "qubits": args.qubits,
                       "unit_note": "30-qubit gate equivalents; the reference accepts n <= 30 only, so for "
                                    "N > 1 it is timed at n = 30 (the b200 arm runs 30 + log2 N qubits)"}}
    if res is None:
        emit({"impl": "reference", "unavailable": why})
        return 0
    base.update({"value": res["value"], "ms_per_step": res["ms_per_run"], "dtype": "c128",
                 "data": "synthetic", "scaling": "weak",
                 "cpu_baseline": {k2: res[k2] for k2 in ("value", "unit", "cores", "kind", "sample")},
                 "e2e": {"value": res["value"], "unit": "gates/s", "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0}})
    emit(base)
    return 0


# ---------------------------------------------------------------------------
def secondary_workloads(abi, workloads, device):
    """Quick numbers for the other BASELINE.json configurations (device time)."""
    out = {}
    # C2b: QFT-30
    n = 30
    ops = abi.make_ops(workloads.qft(n))
    sv = abi.SV(n, device=device)
    sv.apply(ops).flush()
    abi.jit_wait()
    sv.apply(ops).flush()
    sv.synchronize()
    abi.profile_begin(device, per_pass_events=False)
    reps = 2
    for _ in range(reps):
        sv.apply(ops).flush()
    p = abi.profile_end(device)
    st = sv.stats()
    out["qft30"] = {"gates_per_s": reps * len(ops) / (p["region_ms"] / 1e3), "ms_per_circuit": p["region_ms"] / reps,
                    "gates": len(ops), "passes_per_circuit": st["passes"]}
    sv.close()
    # C4: noisy TFIM, DM n=14 (synthetic calibration), wall time of the schedule
    from paper_2401_06861_b200 import naqs

    nd = 14
    cal = {"name": "synthetic", "qubits": [{"t1_us": 60.0, "t2_us": 40.0, "readout_p01": 0.02, "readout_p10": 0.02}] * nd,
           "default_1q": {"error": 0.001, "duration_ns": 50.0}, "default_2q": {"error": 0.01, "duration_ns": 300.0}}
    model = naqs.load_calibration(json.dumps(cal))
    circ = naqs.Circuit(nd)
    for name, qs, ps in workloads.tfim_trotter(nd, 1.0, steps=10):
        circ.add(name, qs, ps)
    naqs.density_expectation(circ, "Z" + "I" * (nd - 1), model)  # warm: plan + queue kernels
    abi.jit_wait()
    naqs.density_expectation(circ, "Z" + "I" * (nd - 1), model)
    t0 = time.perf_counter()
    z = naqs.density_expectation(circ, "Z" + "I" * (nd - 1), model)
    dt = time.perf_counter() - t0
    # C4: noisy QAOA-MaxCut ring (p = 2), same calibration, <Z0 Z1>
    qc = naqs.Circuit(nd)
    for name, qs, ps in workloads.qaoa_ring(nd, 2):
        qc.add(name, qs, ps)
    zz = "ZZ" + "I" * (nd - 2)
    naqs.density_expectation(qc, zz, model)
    abi.jit_wait()
    naqs.density_expectation(qc, zz, model)
    t0 = time.perf_counter()
    zzq = naqs.density_expectation(qc, zz, model)
    out["dm_noisy_qaoa14"] = {"wall_s": time.perf_counter() - t0, "z0z1": zzq, "gates": len(qc),
                              "note": "QAOA-MaxCut ring p=2 (h; cx.rz.cx per edge; rx), end to end via "
                                      "naqs.density_expectation"}
    # C4 upper end: n = 16 (4^16 entries = 69 GB; beyond the reference's
    # 14-qubit guard, so GPU only)
    nd16 = 16
    cal16 = dict(cal, qubits=cal["qubits"][:1] * nd16)
    model16 = naqs.load_calibration(json.dumps(cal16))
    circ16 = naqs.Circuit(nd16)
    for name, qs, ps in workloads.tfim_trotter(nd16, 1.0, steps=10):
        circ16.add(name, qs, ps)
    naqs.density_expectation(circ16, "Z" + "I" * (nd16 - 1), model16, max_qubits=16)
    abi.jit_wait()
    t0 = time.perf_counter()
    z16 = naqs.density_expectation(circ16, "Z" + "I" * (nd16 - 1), model16, max_qubits=16)
    out["dm_noisy_tfim16"] = {"wall_s": time.perf_counter() - t0, "z0": z16, "cpu": None,
                              "note": "beyond the reference's 14-qubit guard: no CPU baseline"}
    dm_cpu = dm_cpu_sample(workloads, nd)
    out["dm_noisy_tfim14"] = {"wall_s": dt, "cpu": dm_cpu,
                              "items": len(circ) * 3 + sum(1 for o in circ.ops() if len(o[1]) == 2),
                              "z0": z, "note": "end-to-end via naqs.density_expectation: attach_noise, superoperator "
                                               "compile, fused passes, expectation"}
    # C5: VQE n=28 energy evaluations (exact, 193 gates + 55 terms)
    nv, layers = 28, 3
    params = workloads.vqe_initial_params(nv, layers)
    vops = abi.make_ops(workloads.vqe_ansatz(nv, layers, params))
    terms = workloads.tfim_hamiltonian(nv)
    sv = abi.SV(nv, device=device)
    sv.apply(vops)
    e = float(sum(sv.expectations(terms)))
    abi.jit_wait()
    sv.reset()
    sv.apply(vops)
    e = float(sum(sv.expectations(terms)))
    reps = 3
    t0 = time.perf_counter()
    for _ in range(reps):
        sv.reset()
        sv.apply(vops)
        e = float(sum(sv.expectations(terms)))
    dt = (time.perf_counter() - t0) / reps
    out["vqe28"] = {"evals_per_s": 1.0 / dt, "ms_per_eval": dt * 1e3, "energy": e, "terms": len(terms),
                    "gates": len(vops)}
    sv.close()
    # f1: batched Monte-Carlo trajectories (one launch) vs the reference's
    # sequential loop (acceptance 5 shape, and a 10-qubit noisy TFIM)
    out["trajectories"] = trajectory_workloads(workloads)
    out["tfim4_sweep"] = tfim4_sweep(workloads)
    return out


def abi_wait():
    from paper_2401_06861_b200 import abi

    abi.jit_wait()  # no compilations competing for the host during the timing


def tfim4_sweep(workloads):
    """C1: the n = 4 TFIM magnetization sweep (31 rows, ideal + noisy with
    example_5q.json), end to end: all rows' state vectors in one launch and all
    rows' noisy density matrices in another (naqs.batch_*), vs the reference's
    own row loop on the host."""
    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Ref  # CPU baseline only
    from paper_2401_06861_b200 import naqs

    cal = open(os.path.join(ROOT, "tests", "golden", "example_5q.json")).read()
    model = naqs.load_calibration(cal)
    abi_wait()
    workloads.tfim_sweep_rows_batched(naqs, 4, model)  # warm
    workloads.tfim_sweep_rows_batched(naqs, 4, model)
    reps = 3
    t0 = time.perf_counter()
    for _ in range(reps):
        rows = np.array(workloads.tfim_sweep_rows_batched(naqs, 4, model))
    gpu_s = (time.perf_counter() - t0) / reps
    res = {"rows": len(rows), "gpu_wall_s": gpu_s, "gates": 60671, "note": "SV ideal + DM noisy columns, shots = 0"}
    if Ref.available():
        ref = Ref()
        threads = ref.set_threads(cpu_threads())
        _, ideal, noisy, ms = ref.tfim_sweep(cal, 4)
        res.update({"cpu_wall_s": ms / 1e3, "cpu_threads": threads,
                    "max_abs_diff_vs_cpu": float(max(np.max(np.abs(rows[:, 1] - ideal)),
                                                     np.max(np.abs(rows[:, 2] - noisy))))})
    return res


def dm_cpu_sample(workloads, nd):
    """The reference's noisy density-matrix run (dm_run_noisy, all host
    threads) on a prefix of the same n = 14 TFIM circuit: seconds per source
    gate, and that rate times the full circuit (an extrapolation, labelled)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import NoiseSpec, Ref  # CPU baseline only

    if not Ref.available():
        return None
    ops = list(workloads.tfim_trotter(nd, 1.0, steps=10))
    k = 3  # one ZZ bond (cx, rz, cx): each noisy 2-qubit gate costs the reference ~10 s at n = 14
    spec = NoiseSpec(nd, t1=60.0, t2=40.0, p01=0.02, p10=0.02, e1=0.001, d1=50.0, e2=0.01, d2=300.0)
    ref = Ref()
    threads = ref.set_threads(cpu_threads())
    ms = ref.dm_time_noisy(nd, ops[:k], spec, 1)
    per_gate = float(ms[0]) / 1e3 / k
    return {"sample": f"first {k} of {len(ops)} gates (with their noise channels), reference dm_run_noisy, "
                      f"{threads} threads", "s_per_gate": per_gate, "extrapolated_wall_s": per_gate * len(ops)}


def trajectory_workloads(workloads):
    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import NoiseSpec, Ref  # CPU baseline only
    from paper_2401_06861_b200 import naqs

    res = {}
    cases = [("acc5_n3", 3, [("h", [0], []), ("cx", [0, 1], []), ("cx", [1, 2], []), ("rx", [0], [0.4]),
                             ("rz", [1], [0.9]), ("cx", [0, 2], [])], 10000, 10000,
              NoiseSpec(3, t1=60.0, t2=40.0, p01=0.0, p10=0.0, e1=0.02, d1=100.0, e2=0.02, d2=100.0)),
             ("tfim_n10_5steps", 10, list(workloads.tfim_trotter(10, 0.5, steps=5)), 10000, 200,
              NoiseSpec(10))]
    for name, n, ops, ntraj, ncpu, spec in cases:
        c = naqs.Circuit(n)
        for g, qs, ps in ops:
            c.add(g, qs, ps)
        model = naqs.load_calibration(spec.calibration_json())
        obs = ["Z" + "I" * (n - 1)]
        naqs.trajectory_expectations(c, obs, model, 16, 1)  # warm
        t0 = time.perf_counter()
        z = naqs.trajectory_expectations(c, obs, model, ntraj, 505)[:, 0]
        gpu_s = time.perf_counter() - t0
        row = {"trajectories": ntraj, "gpu_wall_s": gpu_s, "gpu_traj_per_s": ntraj / gpu_s, "z0_mean": float(z.mean())}
        if Ref.available():
            ms, zref = Ref().traj_time(n, ops, spec, ncpu, 505)
            row.update({"cpu_traj_per_s": ncpu / (ms / 1e3), "cpu_sample": f"first {ncpu} trajectories of the reference's "
                        "sequential run_trajectory loop (shared Rng) on the host",
                        "max_abs_diff_vs_cpu": float(np.max(np.abs(z[:ncpu] - zref)))})
        res[name] = row
    return res


_JSON_OUT = None


def claim_stdout():
    """Keep stdout for the one JSON line: anything else written to fd 1 (NCCL's
    version banner, native or library prints) is sent to stderr instead."""
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(obj):
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(obj) + "\n")
    out.flush()


def main():
    claim_stdout()
    args = parse_args()
    world, rank, local, dist = dist_setup(args)
    if args.impl == "reference":
        rc = run_reference_arm(args, world, rank)
        if dist is not None:
            dist.destroy_process_group()
        return rc

    from paper_2401_06861_b200 import abi, workloads

    if abi.device_count() < 1:
        raise SystemExit("bench.py: no CUDA device")
    dev = local
    g = world.bit_length() - 1
    if (1 << g) != world:
        raise SystemExit("bench.py: the sharded state needs a power-of-two number of GPUs")
    n_local, depth = args.qubits, args.depth
    n = n_local + g  # weak scaling: 2^n_local amplitudes per GPU
    ops_list = workloads.random_circuit(args.seed, n, depth)
    ops = abi.make_ops(ops_list)
    if world == 1:
        sv = abi.SV(n, device=dev, tile_qubits=args.tile, max_qubits=max(30, n))
    else:
        import torch

        uid = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{local}")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(abi.comm_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        sv = abi.SV.sharded(n, rank, world, bytes(uid.cpu().numpy().tobytes()), device=dev,
                            tile_qubits=args.tile, max_qubits=n)

    clk = ClockSampler(dev).__enter__()
    # warm-up: the first step plans the passes and queues their specialised
    # kernels for compilation (jit.cpp); wait for them, then warm the rest
    # Warm-up: at least W steps, continued (up to 16) while steps still meet
    # pass structures that had to be compiled -- a sharded state carries its
    # qubit map from step to step and settles into a short cycle of layouts.
    # All ranks take the same decision (the flushes are collective).
    warm = 0
    while True:
        before = abi.jit_stats()["compiled"]
        sv.apply(ops).flush()
        abi.jit_wait()
        warm += 1
        fresh = abi.jit_stats()["compiled"] > before
        if dist is not None:
            import torch

            flag = torch.tensor([1.0 if fresh else 0.0], device=f"cuda:{local}")
            dist.all_reduce(flag, op=dist.ReduceOp.MAX)
            fresh = flag.item() > 0
        if warm >= max(args.warmup, 3) and (not fresh or warm >= 16):
            break
    sv.synchronize()
    jit = abi.jit_stats()
    stats = sv.stats()

    # ---- value: device time of K steps
    barrier(dist, local)
    sv.synchronize()
    clk.mark_start()
    abi.profile_begin(dev, per_pass_events=True)
    for _ in range(args.steps):
        sv.apply(ops).flush()
    prof = abi.profile_end(dev)
    clk.mark_end()
    clk.__exit__(None, None, None)
    barrier(dist, local)
    ms = max_over_ranks(dist, local, prof["region_ms"])
    # one circuit on the whole (sharded) state; weak scaling: a gate on the
    # 2^(n_local+g)-amplitude state counts 2^g gate equivalents of n_local qubits
    gates_total = args.steps * depth * world
    value = gates_total / (ms / 1e3)
    pass_avg_ms = prof["pass_ms"] / max(prof["pass_launches"], 1)
    bytes_per_launch = prof["pass_bytes"] / max(prof["pass_launches"], 1)
    achieved = bytes_per_launch / (pass_avg_ms / 1e3) / 1e9
    peak, peak_kind = measured_peaks()
    step_gbs = prof["pass_bytes"] / (prof["region_ms"] / 1e3) / 1e9

    # ---- e2e: host buffers in, result out, every step
    e2e_term = [("Z" + "I" * (n - 1), 1.0)]
    sv.apply(ops)
    sv.expectations(e2e_term)  # warm: expectation kernel compiled, collectives connected
    abi.jit_wait()
    sv.apply(ops)
    sv.expectations(e2e_term)
    barrier(dist, local)
    sv.synchronize()
    abi.profile_begin(dev, per_pass_events=False)
    t0 = time.perf_counter()
    lap = []
    for _ in range(args.steps):
        sv.apply(ops)  # host op array -> planner -> pinned staging -> H2D
        sv.expectations(e2e_term)  # D2H of the step's result
        lap.append(time.perf_counter())
    t_e2e = time.perf_counter() - t0
    if os.environ.get("NQ_BENCH_LAPS") == "1":
        print(f"rank {rank} e2e step ms:", [round((b - a) * 1e3, 2) for a, b in zip([t0] + lap[:-1], lap)],
              file=sys.stderr)
    prof_e2e = abi.profile_end(dev)
    t_e2e = max_over_ranks(dist, local, t_e2e)
    laps_ms = sorted((b - a) * 1e3 for a, b in zip([t0] + lap[:-1], lap))
    e2e = {"value": gates_total / t_e2e, "unit": "gates/s",
           "h2d_bytes_per_step": int(prof_e2e["h2d_bytes"] / args.steps),
           "d2h_bytes_per_step": int(prof_e2e["d2h_bytes"] / args.steps),
           "step_ms_median_rank0": laps_ms[len(laps_ms) // 2], "step_ms_max_rank0": laps_ms[-1]}
    jit_end = abi.jit_stats()

    out = None
    if rank == 0:
        out = {
            "metric": "SV gates/s (random circuit, depth 200)",
            "value": value,
            "unit": "gates/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "c128",
            "data": "synthetic",
            "config": {"workload": f"random_circuit(Rng({args.seed})) n={n} depth={depth} "
                                   f"(proj/tests/test_util.hpp generator)",
                       "qubits": n, "depth": depth, "state_bytes": 16 << n,
                       "parallelism": "single" if world == 1 else
                       f"sharded x{world}: {g} global qubits; half-shard exchanges over NVLink peer memory, fused into the preceding pass",
                       "local_qubits": n_local,
                       "warmup_steps_run": warm,
                       "unit_note": (f"gates/s of {n_local}-qubit gate equivalents: each gate on the {n}-qubit "
                                     f"state counts {world} (2^{g}); whole-job aggregate over {world} GPU(s)"),
                       "comm": sv.comm_stats() if world > 1 else None,
                       "l2": "state (16 GiB) >> L2 (126 MB): every pass streams from HBM"},
            "hbm_gbs": step_gbs,
            "hbm_frac_step": step_gbs / peak,
            "passes_per_step": stats["passes"],
            "microops_per_step": stats["microops"],
            "gpu_launches": prof["kernel_launches"],
            "jit": jit,
            "jit_end": jit_end,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic_from_profiles(),
                         "kernel": ("nqjit (pass-specialised fused pass, NVRTC)" if jit.get("launches", 0) > 0
                                    else "pass_kernel (fused pass interpreter)"), "bytes_per_launch": bytes_per_launch,
                         "avg_launch_ms": pass_avg_ms, "launches": prof["pass_launches"],
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"},
            "clocks": clk.summary(),
            "e2e": e2e,
        }
    sv.close()
    if rank == 0 and world == 1 and not args.no_secondary:
        try:
            out["secondary"] = secondary_workloads(abi, workloads, dev)
        except Exception as exc:  # secondary numbers never hide the headline
            out["secondary"] = {"error": repr(exc)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res, why = cpu_reference_rate(n, ops_list, args.cpu_ops, 3)
        out["cpu_baseline"] = (
            {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")} if res else {"unavailable": why})
    if rank == 0:
        emit(out)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
