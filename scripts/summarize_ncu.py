"""Summarise ncu outputs into profiles/ text files (run here, on the CPU box).

  python scripts/summarize_ncu.py launches gpurun_out/launches.csv > profiles/r01_launches.txt
  python scripts/summarize_ncu.py full gpurun_out/prof_gemm2.ncu-rep > profiles/r01_gemm_full.txt
"""
import collections
import csv
import io
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__grid_size",
    "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def launches(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        ms = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ms
    total = sum(v[1] for v in agg.values())
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)")
    print(f"# source: {path}; {sum(v[0] for v in agg.values())} launches, {total:.1f} ms total")
    print(f"{'kernel':60s} {'launches':>8s} {'total_ms':>12s} {'share':>7s}")
    for name, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:60]:60s} {n:8d} {ms:12.3f} {100 * ms / total:6.2f}%")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary of {path}")
    for r in rows[2:]:
        print(f"## {r[hdr.index('Kernel Name')]}")
        for m in FULL_METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"  {m:95s} {r[i]:>14s} {units[i]}")


def tail(path, count="14"):
    """The last `count` launches of a launch list, in order (one solver iteration's kernels)."""
    rows = list(csv.DictReader(io.StringIO(open(path).read()[open(path).read().find('"ID"'):])))
    seq = [(r["Kernel Name"], float(r["Metric Value"].replace(",", ""))) for r in rows
           if r["Metric Name"] == "gpu__time_duration.sum"]
    print(f"# {path}: last {count} of {len(seq)} launches (us)")
    for name, ns in seq[-int(count):]:
        print(f"{ns / 1e3:9.2f}  {name[:90]}")


if __name__ == "__main__":
    {"launches": launches, "full": full, "tail": tail}[sys.argv[1]](*sys.argv[2:])
