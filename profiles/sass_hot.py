"""Instruction mix of one kernel from an ncu report's SASS page:
   ncu -i rep --page source --csv --print-source sass > x.csv; python profiles/sass_hot.py x.csv
Prints executed warp instructions by opcode class and the stall samples by opcode."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
iS, iI, iSm = h.index("Source"), h.index("Instructions Executed"), h.index("# Samples")
mix, st = collections.Counter(), collections.Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= iI or not r[iI]:
        continue
    op = r[iS].split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0] + ("." + o.split(".")[1] if o.startswith(("LDG", "STG", "LDS", "STS", "LDGSTS")) and "." in o else "")
    n = int(r[iI]); mix[o] += n; tot += n; st[o] += int(r[iSm] or 0)
print("total warp instr", tot)
for o, n in mix.most_common(28):
    print(f"  {o:14s} {n:12d} {100*n/tot:5.1f}%  samples {st[o]}")
