"""Summarise an ncu report (--set full) or a launch list (--csv --log-file) into
JSON for profiles/.  Usage:
  python tools/ncu_summary.py rep  gpurun_out/prof.ncu-rep  out.json
  python tools/ncu_summary.py list gpurun_out/launches.csv   out.json
"""
import collections
import csv
import io
import json
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
       "launch__shared_mem_per_block_dynamic", "launch__shared_mem_per_block_static",
       "smsp__average_warp_latency_issue_stalled_long_scoreboard", "nvltx__bytes.sum", "nvlrx__bytes.sum",
       "nvltx__bytes_data_user.sum", "nvlrx__bytes_data_user.sum", "l1tex__t_bytes.sum",
       "smsp__pcsamp_warps_issue_stalled_membar", "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio"]


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def to_us(v, unit):
    f = float(v.replace(",", ""))
    return f * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3,
                "second": 1e6, "s": 1e6}.get(unit, 1)


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:120]}
        for m in RAW:
            if m in hdr:
                i = hdr.index(m)
                u = units[i]
                if "bytes" in m:
                    d[m] = to_bytes(vals[i], u)
                elif m == "gpu__time_duration.sum":
                    d["duration_us"] = to_us(vals[i], u)
                else:
                    try:
                        d[m] = float(vals[i].replace(",", ""))
                    except ValueError:
                        d[m] = vals[i]
        if "dram__bytes_read.sum" in d and "dram__bytes_write.sum" in d:
            d["dram_traffic_bytes"] = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        res.append(d)
    return res


def launch_list(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        try:
            us = to_us(r[iv], r[iu])
        except (ValueError, IndexError):
            continue
        k = r[ik].split("(")[0]
        tot[k] += us
        cnt[k] += 1
    T = sum(tot.values())
    return [{"kernel": k, "launches": cnt[k], "total_us": round(tot[k], 2), "avg_us": round(tot[k] / cnt[k], 3),
             "share": round(tot[k] / T, 4)} for k in sorted(tot, key=lambda k: -tot[k])]


if __name__ == "__main__":
    kind, src, dst = sys.argv[1:4]
    data = rep(src) if kind == "rep" else launch_list(src)
    with open(dst, "w") as f:
        json.dump(data, f, indent=1)
    print(json.dumps(data, indent=1)[:3000])
