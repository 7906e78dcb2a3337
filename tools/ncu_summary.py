"""Summarise ncu captures brought back by gpurun into profiles/ (tracked).

  python tools/ncu_summary.py <tag>
reads gpurun_out/launches.csv (gpu__time_duration launch list) and every
gpurun_out/prof_*.ncu-rep (--set full), writes profiles/<tag>_launches.txt and
profiles/<tag>_ncu_full.txt.
"""
import collections
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm clock"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu pipe %"),
    ("smsp__inst_executed.sum", "warp insts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
]


def launches(tag):
    path = os.path.join(OUT, "launches.csv")
    if not os.path.exists(path):
        return
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    seq = []
    for r in rows[hdr + 1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0][:100]
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        tot[name] += v
        cnt[name] += 1
        seq.append((name, v))
    T = sum(tot.values())
    ours = sum(v for k, v in tot.items() if "halo_b200" in k)
    with open(os.path.join(PROF, f"{tag}_launches.txt"), "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
        f.write(f"# command: python tools/prof_step.py 2  (2 HALO-2 INT8 MLP fwd+bwd steps, cfg2 shapes, after setup)\n")
        f.write(f"# total {T:.1f} us over {len(seq)} launches; halo_b200 kernels {ours:.1f} us\n")
        f.write(f"{'total_us':>10} {'n':>4} {'share_of_ours':>13}  kernel\n")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            share = f"{v / ours:.3f}" if "halo_b200" in k else "-"
            f.write(f"{v:10.1f} {cnt[k]:4d} {share:>13}  {k}\n")
        f.write("\n# launch sequence (us)\n")
        for k, v in seq:
            f.write(f"{v:9.1f}  {k}\n")


def full(tag):
    lines = []
    for fn in sorted(os.listdir(OUT)):
        if not (fn.startswith("prof") and fn.endswith(".raw.csv")):
            continue
        raw = open(os.path.join(OUT, fn)).read() if fn.endswith(".csv") else \
            subprocess.run(["ncu", "-i", os.path.join(OUT, fn), "--page", "raw", "--csv"], capture_output=True,
                           text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            continue
        h, units = rows[0], rows[1]
        lines.append(f"## {fn}  (ncu --set full --clock-control none)")
        for r in rows[2:]:
            name = r[h.index("Kernel Name")][:110]
            lines.append(f"- {name}")
            parts = []
            for m, label in METRICS:
                if m in h:
                    i = h.index(m)
                    parts.append(f"{label}={r[i]} {units[i]}".strip())
            lines.append("    " + "; ".join(parts))
        lines.append("")
    if lines:
        with open(os.path.join(PROF, f"{tag}_ncu_full.txt"), "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    launches(tag)
    full(tag)
    print("wrote", [p for p in os.listdir(PROF) if p.startswith(tag)])
