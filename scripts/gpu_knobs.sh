run() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 8 --warmup 3 --no-secondary --no-cpu-baseline $EXTRA > gpurun_out/knob_$name.json 2> gpurun_out/knob_$name.err; echo "$name rc=$?"
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['passes_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])" gpurun_out/knob_$name.json; }
run base NQ_X=0
run pf_minb3 NQ_JIT_PREFETCH=1 NQ_JIT_MINB=3
run pf_minb2 NQ_JIT_PREFETCH=1 NQ_JIT_MINB=2
run minb3 NQ_JIT_MINB=3
EXTRA="--tile 10" run t10 NQ_X=0
EXTRA="--tile 10" run t10_pf NQ_JIT_PREFETCH=1
EXTRA="--tile 12" run t12 NQ_X=0
timeout 600 python - <<'PY'
import time, sys
sys.path.insert(0, '.')
from paper_2401_06861_b200 import abi, workloads
nv, layers = 28, 3
params = workloads.vqe_initial_params(nv, layers)
vops = abi.make_ops(workloads.vqe_ansatz(nv, layers, params))
terms = workloads.tfim_hamiltonian(nv)
sv = abi.SV(nv, device=0)
for _ in range(3):
    sv.reset(); sv.apply(vops); sum(sv.expectations(terms))
abi.jit_wait()
for _ in range(2):
    sv.reset(); sv.apply(vops); sum(sv.expectations(terms))
sv.synchronize()
def t(fn, k=5):
    sv.synchronize(); t0 = time.perf_counter()
    for _ in range(k): fn(); sv.synchronize()
    return (time.perf_counter() - t0) / k * 1e3
print("reset ms", t(lambda: sv.reset()))
print("reset+flush ms", t(lambda: (sv.reset(), sv.apply(vops).flush())))
sv.reset(); sv.apply(vops).flush()
print("expectations ms", t(lambda: sv.expectations(terms)))
print("full eval ms", t(lambda: (sv.reset(), sv.apply(vops), sv.expectations(terms))))
abi.profile_begin(0, per_pass_events=True)
sv.reset(); sv.apply(vops).flush(); sv.synchronize()
p = abi.profile_end(0)
print("profile", {k: p[k] for k in ("region_ms", "pass_ms", "pass_launches")}, sv.stats())
PY
