"""Summaries of ncu captures for profiles/.

  python tools/ncu_summary.py launches <launches.csv>          # per-kernel shares
  python tools/ncu_summary.py full <report.ncu-rep> [name]     # key metrics + stalls
  python tools/ncu_summary.py traffic <report.ncu-rep> <key>   # -> profiles/traffic.json

`launches` reads the CSV of an `ncu --metrics gpu__time_duration.sum` pass;
`full` reads a `--set full` report via `ncu -i ... --page raw --csv`.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEY_METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0][:70]
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(
            d["Metric Unit"], 1e-3)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    tot = sum(a[1] for a in agg.values())
    print(f"{'launches':>8} {'total us':>10} {'share':>6} {'avg us':>9}  kernel")
    for name, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:8d} {us:10.1f} {100 * us / tot:5.1f}% {us / c:9.2f}  {name}")


def full(rep, name=None):
    hdr, units, rows = raw_rows(rep)
    for r in rows:
        kname = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        if name and name not in kname:
            continue
        print(f"kernel: {kname[:120]}")
        for m in KEY_METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"  {m:70s} {r[i]:>16s} {units[i]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith(
                    "_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h))
                except ValueError:
                    pass
        print("  top stall reasons (warps per issue-active cycle):")
        for v, h in sorted(stalls, reverse=True)[:6]:
            print(f"    {h[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:28s} {v:.3f}")


def traffic(rep, key):
    hdr, units, rows = raw_rows(rep)
    r = rows[0]
    def mb(m):
        i = hdr.index(m)
        v = float(r[i])
        return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[units[i]]
    rd, wr = mb("dram__bytes_read.sum"), mb("dram__bytes_write.sum")
    path = os.path.join(ROOT, "profiles", "traffic.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    d[key] = int(round((rd + wr) * 1e6))
    json.dump(d, open(path, "w"), indent=1, sort_keys=True)
    print(key, d[key], "bytes per launch (read", rd, "MB, write", wr, "MB)")


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "launches":
        launches(sys.argv[2])
    elif cmd == "full":
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
    elif cmd == "traffic":
        traffic(sys.argv[2], sys.argv[3])
