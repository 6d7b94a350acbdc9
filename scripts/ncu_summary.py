#!/usr/bin/env python
"""Summarise an ncu report (.ncu-rep) into profiles/: per-kernel duration,
DRAM bytes, throughputs, occupancy; optionally record the y_L traffic for
bench.py's roofline.traffic.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r1_ncu_yL.json [--traffic-key c2_n1]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed": "l1tex_lsu_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "us": 1e-6,
         "nsecond": 1e-9, "ns": 1e-9, "msecond": 1e-3, "ms": 1e-3, "Ghz": 1e9, "GHz": 1e9,
         "Mhz": 1e6, "hz": 1, "Kbyte/block": 1e3, "byte/block": 1}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    key = sys.argv[sys.argv.index("--traffic-key") + 1] if "--traffic-key" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:160]}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[name] = v * SCALE.get(units[i], 1)
                d[name + "_unit"] = "SI" if units[i] in SCALE else units[i]
        if "dram_read" in d and "dram_write" in d:
            d["dram_bytes"] = d["dram_read"] + d["dram_write"]
        kernels.append(d)
    json.dump({"report": rep, "kernels": kernels}, open(out, "w"), indent=1)
    print(json.dumps(kernels, indent=1)[:3000])
    if key:
        yl = [k for k in kernels if "spmv_block_kernel" in k["kernel"] or "spmv_stream_kernel" in k["kernel"]]
        if yl:
            tp = "profiles/ncu_traffic.json"
            try:
                cur = json.load(open(tp))
            except Exception:
                cur = {}
            cur[key] = {"dram_bytes_per_launch": yl[0]["dram_bytes"], "kernel": yl[0]["kernel"],
                        "duration_s_cold": yl[0]["duration"], "source": rep}
            json.dump(cur, open(tp, "w"), indent=1)


if __name__ == "__main__":
    main()
