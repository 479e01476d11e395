"""Aggregate an `ncu --page source --csv --print-source sass` dump: stall
samples per opcode class and the hottest instructions."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
tot = Counter()
cnt = Counter()
samples = []
stall_cols = [h for h in hdr if h.startswith("stall_") or "Stall" in h]
seen = set()
for r in data:
    if len(r) < len(hdr) or not r[ix["Instructions Executed"]].strip().isdigit():
        continue
    if "Address" in ix:  # ncu lists each instruction once per view: count it once
        if r[ix["Address"]] in seen:
            continue
        seen.add(r[ix["Address"]])
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else ""
    if op.startswith("@"):
        op = src.split()[1]
    base = op.split(".")[0]
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ex = int(r[ix["Instructions Executed"]] or 0)
    tot[base] += s
    cnt[base] += ex
    samples.append((s, src, r))
T = sum(tot.values())
E = sum(cnt.values())
print(f"total samples {T}, warp instrs {E}")
for k, v in tot.most_common(25):
    print(f"  {k:10s} samples {v:8d} ({100*v/T:5.1f}%)  instrs {cnt[k]:12d} ({100*cnt[k]/E:5.1f}%)")
print("hottest:")
for s, src, r in sorted(samples, reverse=True)[:25]:
    print(f"  {s:6d}  {src}")
