"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total / mean duration and share of GPU time."""
import collections
import csv
import sys


def main(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]  # drop ==PROF== / ==WARNING== lines
    rows = list(csv.DictReader(lines))
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        ns = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns *= {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1)
        a = agg.setdefault(name, [0, 0.0, r["Grid Size"], r["Block Size"]])
        a[0] += 1
        a[1] += ns
    total = sum(a[1] for a in agg.values())
    print(f"## launch list: `{path}` ({len(rows)} launches, {total / 1e6:.2f} ms GPU time, serialised, cold-cache)\n")
    print("| kernel | launches | total ms | mean ms | share | grid | block |")
    print("|---|---|---|---|---|---|---|")
    for name, (cnt, ns, grid, block) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{name}` | {cnt} | {ns / 1e6:.3f} | {ns / cnt / 1e6:.3f} | {100 * ns / total:.1f} % | {grid} | {block} |")


if __name__ == "__main__":
    main(sys.argv[1])
