"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel shares.
usage: python tools/launches_summary.py launches.csv TITLE > profiles/<tag>_launches_summary.md"""
import csv
import io
import sys
from collections import defaultdict


def main(path, title):
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0].replace("void ", "").split("<")[0]
        v = float(r["Metric Value"].replace(",", ""))
        tot[k] += v * (1e-3 if r["Metric Unit"] == "ns" else (1.0 if r["Metric Unit"] == "us" else 1e3))
        cnt[k] += 1
    all_us = sum(tot.values())
    print(f"# Launch list shares, {title}\n")
    print("cold-cache, serialised per-launch times: compare SHARES with bench.py's live event times, not absolutes.\n")
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| {k} | {cnt[k]} | {v / 1e3:.2f} | {100 * v / all_us:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
