#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel counts, mean duration and share of the total.  y_L launches of the
e2e pass (dspmv_apply_host: the streamed-x instantiation waits on the x chunk
flags, so it runs longer than a device-resident y_L) are tagged.

    python scripts/launch_summary.py gpurun_out/launches.csv "header line" > profiles/..._summary.txt
"""
import collections
import csv
import re
import sys


def main():
    path, header = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    launches = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = r["Metric Unit"]
        v = float(r["Metric Value"].replace(",", ""))
        us = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[unit]
        launches[r["ID"]] = (re.sub(r"\(.*", "", r["Kernel Name"]).replace("(anonymous namespace)::", ""), us)
    by = collections.defaultdict(list)
    for name, us in launches.values():
        tag = name
        # the streamed-x instantiation (last template argument kCoh = 1) runs only in apply_host
        if "spmv_block_kernel" in name and re.search(r",\s*1>\s*$", name.strip()):
            tag = name + "  [apply_host e2e: waits on the x chunk flags]"
        by[tag].append(us)
    total = sum(sum(v) for v in by.values())
    print(header)
    print("cold-cache serialised launches; compare shares, not absolutes; flush_kernel runs between timed steps, "
          "outside the step events")
    for tag, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):5d} launches  mean {sum(v) / len(v):8.2f} us  share {100 * sum(v) / total:5.1f}%  {tag}")


if __name__ == "__main__":
    main()
