"""DRAM traffic of the advance kernel over one SSSP step, for bench.py's
roofline.traffic (compare with the algorithmic bytes B_alg x m_reach).

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:'k_push_range|k_tail' --csv --log-file gpurun_out/traffic.csv \
      python tools/profile_sssp.py --scale 24 --runs 1 --device-loop 0 --relabel on
  python tools/traffic.py gpurun_out/traffic.csv 24 > profiles/advance_traffic.json
(--relabel on: the timed configuration of bench.py from the first call on.
The tail kernel (tail.cuh) runs the last supersteps' advances: counted with
the push launches.)
ncu replays each launch with flushed caches, so this is an upper bound of the
live traffic (the 64 MB distance array stays in L2 across live launches).
"""
import csv
import json
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
per = defaultdict(dict)
names = {}
for r in rows:
    if "Metric Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
                 "us": 1e-6, "ms": 1e-3,
                 "usecond": 1e-6, "msecond": 1e-3}.get(u, 1)
        per[d["ID"]][d["Metric Name"]] = v * scale
        names[d["ID"]] = d["Kernel Name"].split("(")[0]
ids = sorted(per, key=int)
rd = sum(per[i]["dram__bytes_read.sum"] for i in ids)
wr = sum(per[i]["dram__bytes_write.sum"] for i in ids)
t = sum(per[i]["gpu__time_duration.sum"] for i in ids)
kinds = sorted(set(names[i] for i in ids))
print(json.dumps({"scale": int(sys.argv[2]), "kernel": " + ".join(kinds) if ids else None,
                  "launches": len(ids), "dram_read_bytes_total": rd,
                  "dram_bytes_per_step": rd + wr,
                  "dram_write_bytes_total": wr, "dram_bytes_per_launch": (rd + wr) / max(len(ids), 1),
                  "kernel_time_s_total_cold": t,
                  "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                            "gpu__time_duration.sum --clock-control none -k regex:'k_push_range|k_tail' "
                            "python tools/profile_sssp.py --scale %s --runs 1 --device-loop 0 --relabel on "
                            "(flushed caches per launch)"
                            % sys.argv[2]}, indent=1))
