"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        agg[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"# launch list summary of {path} (ncu gpu__time_duration.sum, cold-cache serialised)")
    print("kernel,launches,total_ms,mean_ms,share")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f'"{k}",{len(v)},{sum(v)/1e6:.3f},{sum(v)/len(v)/1e6:.3f},{sum(v)/tot:.4f}')


if __name__ == "__main__":
    main(sys.argv[1])
