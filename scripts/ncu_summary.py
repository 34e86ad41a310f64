#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, no GPU needed).

    python scripts/ncu_summary.py full <report.ncu-rep> <out.json>
    python scripts/ncu_summary.py launches <launches.csv> <out.txt>
    python scripts/ncu_summary.py traffic <report.ncu-rep> <kernel> <out.json> <nnz> <n> <source> <limiter>

`full`: key counters of every kernel in a `--set full` capture (DRAM bytes,
L1/L2 throughput, occupancy, stall summary).  `launches`: per-kernel share of
the device time of a `--metrics gpu__time_duration.sum` launch list.
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.sum", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__cycles_elapsed.avg.per_second",
]


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


def launches(path, out):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        tot[name] += float(r["Metric Value"].replace(",", ""))
        cnt[name] += 1
    all_ns = sum(tot.values())
    txt = [f"{'kernel':40s} {'launches':>8s} {'mean_us':>10s} {'share':>7s}"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        txt.append(f"{k:40s} {cnt[k]:8d} {v / cnt[k] / 1e3:10.2f} {v / all_ns:7.3f}")
    txt.append(f"total {all_ns / 1e3:.1f} us over {sum(cnt.values())} launches (cold-cache, serialised)")
    with open(out, "w") as f:
        f.write("\n".join(txt) + "\n")
    print("\n".join(txt))


def traffic(rep, kernel, out, nnz, n, source, limiter):
    """Per-launch DRAM bytes of `kernel` from a --set full capture: the record
    bench.py reads for roofline.traffic (profiles/<kernel>_dram_bytes_cfg<c>.json)."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--kernel-name", f"regex:{kernel}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def get(k):
        i = hdr.index(k)
        return float(vals[i].replace(",", "")) * scale.get(units[i], 1)
    rec = {"kernel": kernel, "source": source,
           "dram_bytes_per_launch": get("dram__bytes_read.sum") + get("dram__bytes_write.sum"),
           "dram_bytes_read": get("dram__bytes_read.sum"), "dram_bytes_write": get("dram__bytes_write.sum"),
           "nnz": int(nnz), "n": int(n), "limiter": limiter,
           "gpu_time_us_under_ncu": float(vals[hdr.index("gpu__time_duration.sum")].replace(",", "")) *
           {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(units[hdr.index("gpu__time_duration.sum")], 1)}
    with open(out, "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(*sys.argv[2:9])
    else:
        {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
