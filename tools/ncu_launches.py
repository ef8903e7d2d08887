"""Per-kernel summary of an ncu launch list (gpu__time_duration.sum CSV).

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file launches.csv python bench.py ...
    python tools/ncu_launches.py launches.csv [--skip-prefix gen_kernel] > profiles/xxx.md

Launches are grouped by kernel name (template arguments stripped); the
share column is each kernel's fraction of all listed GPU time.  ncu times
are cold-cache and serialised: use them for shares, not absolutes.
"""
import collections
import csv
import re
import sys


def main():
    path = sys.argv[1]
    skip = sys.argv[sys.argv.index("--skip-prefix") + 1] if "--skip-prefix" in sys.argv else None
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    agg = collections.OrderedDict()
    for r in rows:
        if r[12] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"<.*", "", r[4].split("(")[0]).strip()
        name = name.split(" ")[-1]
        if skip and name.startswith(skip):
            continue
        ns = float(r[14].replace(",", ""))
        scale = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(r[13], 1.0)
        n, t, grid, block = agg.get(name, (0, 0.0, r[8], r[7]))
        agg[name] = (n + 1, t + ns * scale, grid, block)
    tot = sum(v[1] for v in agg.values()) or 1.0
    print(f"source: {path}\n")
    print("| kernel | launches | total ms | avg us | share | grid | block |")
    print("|---|---:|---:|---:|---:|---|---|")
    for name, (n, t, grid, block) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {name} | {n} | {t/1e6:.3f} | {t/n/1e3:.1f} | {t/tot*100:.1f}% | {grid} | {block} |")
    print(f"\ntotal listed GPU time: {tot/1e6:.3f} ms")


if __name__ == "__main__":
    main()
