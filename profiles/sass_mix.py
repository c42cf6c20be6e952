"""Summarise an `ncu --page source --csv` SASS export: warp instructions and stall samples per opcode.
Usage: python profiles/sass_mix.py file.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
isrc, iex, ismp = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ex, smp = defaultdict(int), defaultdict(int)
for r in rows[2:]:
    if len(r) <= iex:
        continue
    op = r[isrc].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    o = o.split(".")[0]
    try:
        ex[o] += int(r[iex] or 0)
        smp[o] += int(r[ismp] or 0)
    except ValueError:
        pass
T, S = sum(ex.values()), sum(smp.values())
print(f"total warp instr {T:.4g}, samples {S}")
for o, v in sorted(ex.items(), key=lambda t: -t[1])[:top]:
    print(f"  {o:12s} {v:12d} {100 * v / T:5.1f}%  stall samples {100 * smp[o] / max(S, 1):5.1f}%")
