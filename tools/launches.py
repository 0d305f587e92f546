"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list.
usage: python tools/launches.py gpurun_out/launches.csv [--last-run k_init] [--seq]"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            v = float(d["Metric Value"])
            u = d["Metric Unit"]
            v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "%": None,
                  "ms": 1e3, "second": 1e6, "s": 1e6}[u]
            data.append((d["Kernel Name"].split("(")[0].replace("void ", ""), v, d.get("Grid Size", "")))
    return data


def main():
    path = sys.argv[1]
    data = load(path)
    marker = "k_init"
    idx = [i for i, d in enumerate(data) if marker in d[0]]
    run = data[idx[-1]:] if idx else data
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for k, v, _ in run:
        tot[k] += v
        cnt[k] += 1
    total = sum(tot.values())
    print(f"last run: {len(run)} launches, {total:.1f} us of kernel time")
    for k in sorted(tot, key=lambda x: -tot[x]):
        print(f"{tot[k]:10.1f} us {tot[k] / total * 100:5.1f}%  x{cnt[k]:3d}  {k}")
    if "--seq" in sys.argv:
        for k, v, g in run:
            print(f"{v:9.1f}  {g:>14s}  {k}")


if __name__ == "__main__":
    main()
