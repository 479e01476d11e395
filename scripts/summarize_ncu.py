"""Key metrics per profiled launch of an ncu --set full report (.ncu-rep)."""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, data = rows[0], rows[2:]
    print(f"# {path}")
    for i, r in enumerate(data):
        d = dict(zip(hdr, r))
        print(f"launch {i}: {d.get('Kernel Name', '')}  grid={d.get('Grid Size')} block={d.get('Block Size')}")
        for k in KEYS:
            if k in d:
                print(f"   {k} = {d[k]}")
        stalls = {k: v for k, v in d.items()
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
        top = sorted(((float(v.replace(",", "")), k) for k, v in stalls.items() if v), reverse=True)[:6]
        print("   top stalls: " + ", ".join(f"{k[34:-27]}={v:.2f}" for v, k in top))


if __name__ == "__main__":
    main(sys.argv[1])
