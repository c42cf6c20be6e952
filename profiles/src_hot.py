"""Per-source-line executed instructions and stall samples from an ncu report:
   ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python profiles/src_hot.py x.csv [top]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out, f = [], ""
h = None
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        h = r
        iI, iSm = h.index("Instructions Executed"), h.index("# Samples")
    elif h and r and r[0]:
        try:
            out.append((int(r[iI]), int(r[iSm] or 0), f, r[0], r[1][:100]))
        except (ValueError, IndexError):
            pass
tot, ts = sum(o[0] for o in out), sum(o[1] for o in out)
print("total", tot, "samples", ts)
for n, s, f, l, src in sorted(out, reverse=True)[:top]:
    print(f"{100*n/tot:5.1f}% inst {100*s/ts:5.1f}% smp {f}:{l}: {src}")
