"""Summarise ncu outputs into the committed profile notes.

    python profiles/summarize.py <launches.csv> <full.ncu-rep> <tag>

writes profiles/<tag>_launches.md (per-kernel share of the serialised launch list),
profiles/<tag>_ncu_full.md (key counters of the `--set full` capture) and
profiles/<tag>_traffic.json (DRAM bytes per launch, read by bench.py for roofline.traffic).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

HERE = os.path.dirname(os.path.abspath(__file__))


def short(name):
    return name.split("(")[0].replace("void ", "")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    h = next(r for r in rows if r and r[0] == "ID")
    data = [r for r in rows[rows.index(h) + 1:] if len(r) == len(h)]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in data:
        v = float(r[iv].replace(",", ""))
        v = v / 1e6 if r[iu] == "ns" else (v / 1e3 if r[iu] == "us" else v)
        tot[short(r[ik])] += v
        cnt[short(r[ik])] += 1
    s = sum(tot.values())
    lines = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"| `{k}` | {cnt[k]} | {v:.3f} | {100 * v / s:.1f} % |")
    return "\n".join(lines), s


def full(path):
    # an .ncu-rep, or its `--page raw --csv` export (512^3 captures are exported on the GPU box)
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6, "s": 1e3,
             "second": 1e3, "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3,
             "KB": 1e-6, "MB": 1e-3, "GB": 1.0}

    def g(row, m):
        return row[h.index(m)] if m in h else ""

    def gs(row, m):   # value converted to ms (times) or GB (bytes) using the units row
        v = float(g(row, m).replace(",", ""))
        return v * scale.get(units[h.index(m)], 1.0)

    recs = []
    for row in r[2:]:
        recs.append(dict(
            kernel=short(g(row, "Kernel Name")), ms=gs(row, "gpu__time_duration.sum"),
            dram_GB=gs(row, "dram__bytes_read.sum") + gs(row, "dram__bytes_write.sum"),
            dram_pct=float(g(row, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")),
            l1tex_pct=float(g(row, "l1tex__throughput.avg.pct_of_peak_sustained_active")),
            fp64_pct=float(g(row, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active")),
            warps_pct=float(g(row, "sm__warps_active.avg.pct_of_peak_sustained_active")),
            regs=int(float(g(row, "launch__registers_per_thread"))),
            grid=g(row, "launch__grid_size"), block=g(row, "launch__block_size")))
    lines = ["| kernel | ms | DRAM GB (r+w) | DRAM % | L1/SMEM % | FP64 pipe % | warps % | regs | grid x block |",
             "|---|---|---|---|---|---|---|---|---|"]
    seen = set()
    traffic = {}
    # the LAST capture of each kernel name: the steady launch (e.g. a CG tangent pass after the first,
    # which skips p_old and x)
    # keyed by (name, traffic class): the 6- and 1-component launches of one kernel are separate rows
    for x in reversed(recs):
        key = (x["kernel"], round(x["dram_GB"] / max(x["dram_GB"], 1e-9) * 0 + x["dram_GB"], 0))
        if key in seen:
            continue
        seen.add(key)
        if x["kernel"] not in traffic or x["dram_GB"] * 1e9 > traffic[x["kernel"]]:
            traffic[x["kernel"]] = x["dram_GB"] * 1e9
        lines.append(f"| `{x['kernel']}` | {x['ms']:.3f} | {x['dram_GB']:.3f} | {x['dram_pct']:.1f} | "
                     f"{x['l1tex_pct']:.1f} | {x['fp64_pct']:.1f} | {x['warps_pct']:.1f} | {x['regs']} | "
                     f"{x['grid']} x {x['block']} |")
    return "\n".join(lines), traffic


if __name__ == "__main__":
    lpath, fpath, tag = sys.argv[1:4]
    lt, s = launches(lpath)
    open(os.path.join(HERE, f"{tag}_launches.md"), "w").write(
        f"# {tag}: ncu launch list (cold-cache, serialised; compare shares)\n\n"
        f"`ncu --metrics gpu__time_duration.sum --clock-control none` over the launches of the bench command "
        f"(see profiles/{tag}_profile.sh when present); total {s:.2f} ms.\n\n{lt}\n")
    # several reports (comma-separated) are concatenated in order
    ft, traffic = "", {}
    for k, fp in enumerate(fpath.split(",")):
        t_k, tr_k = full(fp)
        ft = t_k if k == 0 else ft + "\n" + "\n".join(t_k.splitlines()[2:])
        traffic.update({key: val for key, val in tr_k.items() if key not in traffic})
    open(os.path.join(HERE, f"{tag}_ncu_full.md"), "w").write(
        f"# {tag}: `ncu --set full` capture of the hot kernels (last capture of each kernel name)\n\n{ft}\n")
    json.dump(traffic, open(os.path.join(HERE, f"{tag}_traffic.json"), "w"), indent=1)
    print(lt)
    print(ft)
