"""Time the sharded phases (flush, expectation) per rank.  torchrun, N GPUs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2401_06861_b200 import abi, workloads  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
g = world.bit_length() - 1
nl = int(os.environ.get("NL", "30"))
n = nl + g
ops = abi.make_ops(workloads.random_circuit(2024, n, 200))
uid = torch.zeros(128, dtype=torch.uint8, device=f"cuda:{local}")
if rank == 0:
    uid.copy_(torch.frombuffer(bytearray(abi.comm_unique_id()), dtype=torch.uint8))
dist.broadcast(uid, 0)
sv = abi.SV.sharded(n, rank, world, bytes(uid.cpu().numpy().tobytes()), device=local, max_qubits=n)
sv.apply(ops).flush()
abi.jit_wait()
sv.apply(ops).flush()
term = [("Z" + "I" * (n - 1), 1.0)]
sv.expectations(term)
abi.jit_wait()
sv.synchronize()
dist.barrier()


def timed(label, fn, reps=3):
    fn()
    abi.jit_wait()
    dist.barrier()
    sv.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    sv.synchronize()
    dt = (time.perf_counter() - t0) / reps * 1e3
    c0 = sv.comm_stats()
    if rank == 0:
        print(f"{label}: {dt:.2f} ms  comm={c0} jit={abi.jit_stats()}", flush=True)


timed("flush", lambda: sv.apply(ops).flush())
timed("flush", lambda: sv.apply(ops).flush())
timed("expect", lambda: sv.expectations(term))
timed("apply+expect", lambda: (sv.apply(ops), sv.expectations(term)))
if rank == 0:
    print("jit", abi.jit_stats())
dist.destroy_process_group()
