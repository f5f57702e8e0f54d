"""Summarise ncu outputs into profiles/ (markdown + JSON).

  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py full <prof.ncu-rep> <out.md> [--traffic profiles/gemv_traffic.json --n N --P P]
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("void ", "").replace("unnamed>::", "").replace("ks::", "")
    return name.strip()


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) >= 15 and r[0] != "ID"]
    agg = collections.OrderedDict()
    for r in rows:
        if r[12] != "gpu__time_duration.sum":
            continue
        k = short(r[4])
        t = float(r[14]) * (1e-3 if r[13] == "ns" else 1.0)  # -> us
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += t
    solver = {k: v for k, v in agg.items() if not k.startswith("k_gen") and "at::" not in k
              and "elementwise" not in k and "reduce_kernel" not in k}
    tot = sum(v[1] for v in solver.values())
    lines = ["| kernel | launches | total us | avg us | share of solver kernels |",
             "|---|---|---|---|---|"]
    for k, (c, t) in sorted(solver.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {c} | {t:.1f} | {t / c:.2f} | {100 * t / tot:.2f}% |")
    other = {k: v for k, v in agg.items() if k not in solver}
    if other:
        lines.append("")
        lines.append("Excluded (input generation / torch plumbing): " +
                     ", ".join(f"`{k}` x{v[0]} ({v[1]:.0f} us)" for k, v in other.items()))
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
           "launch__block_size", "launch__occupancy_limit_registers", "sm__cycles_elapsed.avg.per_second",
           "smsp__average_warp_latency_issue_stalled_long_scoreboard", "l1tex__t_bytes.sum",
           "lts__t_sector_hit_rate.pct"]


def full(path, out, traffic=None, n=None, P=None, gemvs=None, persistent=False):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = []
    recs = []
    for r in rows[2:]:
        rec = {"kernel": short(r[hdr.index("Kernel Name")])}
        for m in METRICS:
            if m in hdr:
                rec[m] = f"{r[hdr.index(m)]} {units[hdr.index(m)]}".strip()
        recs.append(rec)
    for rec in recs:
        lines.append(f"### `{rec['kernel']}`")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for m in METRICS:
            if m in rec:
                lines.append(f"| `{m}` | {rec[m]} |")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic:
        def to_bytes(s):
            v, u = s.split()
            v = float(v.replace(",", "")) if v not in ("-nan", "nan") else float("nan")
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u]
        import math
        g_all = gemvs or [1] * len(recs)
        ok = [i for i, r in enumerate(recs) if not math.isnan(to_bytes(r["dram__bytes_read.sum"]))]
        rd = [to_bytes(recs[i]["dram__bytes_read.sum"]) for i in ok]
        wr = [to_bytes(recs[i]["dram__bytes_write.sum"]) for i in ok]
        g = [g_all[i] for i in ok]
        per = sum(a + b for a, b in zip(rd, wr)) / sum(g)
        json.dump({"kernels": [recs[i]["kernel"] for i in ok], "n": n, "P": P, "persistent": persistent,
                   "gemvs_per_launch": g,
                   "dram_bytes_per_launch": per,   # per GEMV when gemvs are given
                   "dram_read_per_gemv": sum(rd) / sum(g), "dram_write_per_gemv": sum(wr) / sum(g),
                   "algorithmic_bytes_per_gemv": 8.0 * n * n / P, "source": path},
                  open(traffic, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        a = sys.argv
        tr = a[a.index("--traffic") + 1] if "--traffic" in a else None
        n = int(a[a.index("--n") + 1]) if "--n" in a else None
        P = int(a[a.index("--P") + 1]) if "--P" in a else None
        gm = [int(v) for v in a[a.index("--gemvs") + 1].split(",")] if "--gemvs" in a else None
        full(a[2], a[3], tr, n, P, gm, "--persistent" in a)
