"""Summarize an ncu --csv launch list (gpu__time_duration + dram bytes) per launch."""
import collections
import csv
import sys

for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hdr = None
    data = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", ""))
        data.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    print(f)
    tot = 0.0
    for (i, k), m in data.items():
        t = m.get("gpu__time_duration.sum", 0)
        tot += t
        print(f"  {i:>4} {k:28s} {t / 1e3:10.3f} us  read {m.get('dram__bytes_read.sum', 0) / 1e6:10.1f} MB"
              f"  write {m.get('dram__bytes_write.sum', 0) / 1e6:10.1f} MB")
    print(f"  total {tot / 1e3:.3f} us")
