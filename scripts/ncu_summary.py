"""Summarise ncu reports / launch lists into profiles/ (run here, no GPU).

    python scripts/ncu_summary.py report.ncu-rep [more.ncu-rep ...] > profiles/xxx.md
    python scripts/ncu_summary.py --launches launches.csv > profiles/xxx_launches.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration (ms)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem store bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "smem store wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem load wavefronts"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe % of peak"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe % of peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe % of peak"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global load sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "global load requests"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "global store sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "global store requests"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 sectors read (from L1)"),
    ("lts__t_sectors_srcunit_tex_op_write.sum", "L2 sectors written (from L1)"),
    ("local_load_bytes", "local memory (spill) loads"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def summarize(rep):
    kernels, units = raw(rep)
    print(f"## {rep}\n")
    for k in kernels:
        print(f"### kernel `{k.get('Kernel Name', '?')[:90]}` (launch id {k.get('ID')})\n")
        print("| metric | value | unit |\n|---|---|---|")
        for key, label in KEYS:
            if key in k:
                print(f"| {label} (`{key}`) | {k[key]} | {units.get(key, '')} |")
        stalls = sorted(((key, k[key]) for key in k if key.startswith("smsp__average_warps_issue_stalled")
                         and key.endswith("per_issue_active.ratio")), key=lambda kv: -float(kv[1] or 0))[:6]
        print("\nTop warp stall reasons (warps per issue):\n")
        for key, v in stalls:
            print(f"- {key.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}: {v}")
        print()


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0][-60:]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"].replace(",", ""))
    total = sum(v[1] for v in agg.values())
    print(f"## launch list {path} (ncu --metrics gpu__time_duration.sum, serialised, cold caches)\n")
    print("| kernel | launches | total ms | avg ms | share |\n|---|---|---|---|---|")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{name}` | {n} | {t / 1e6:.3f} | {t / n / 1e6:.3f} | {100 * t / total:.1f}% |")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        for p in sys.argv[2:]:
            launches(p)
    else:
        for p in sys.argv[1:]:
            summarize(p)
