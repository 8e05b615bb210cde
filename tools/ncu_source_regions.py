"""Summarise an ncu --page source --csv --print-source sass export: stall
samples and executed instructions per SASS address range, split where the
kernel's roles live (found by marker instructions).  Usage:
python tools/ncu_source_regions.py source.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ix = {c: h.index(c) for c in cols}
base = int(data[0][0], 16)
# contiguous blocks of >0 executed instructions, reported by top sampled instruction
tot = sum(float(r[iS] or 0) for r in data)
print(f"total samples {tot:.0f}")
top = sorted(data, key=lambda r: -float(r[iS] or 0))[:25]
for r in top:
    st = {c[6:]: int(float(r[ix[c]] or 0)) for c in cols if float(r[ix[c]] or 0) > 0}
    st = dict(sorted(st.items(), key=lambda kv: -kv[1])[:3])
    print(f"{int(r[0], 16) - base:#08x} samples {r[iS]:>6} exec {r[iE]:>9}  {r[1][:60]:60s} {st}")
