"""Per-class DRAM traffic of the K3 GEMMs in one cfg2 MLP step, from an ncu
CSV (dram__bytes_read.sum, dram__bytes_write.sum, gpu__time_duration.sum over
k_gemm launches of tools/prof_step.py).  The last 9 GEMM launches are one
step, in the layer's order: F gate, F up, F down, E down, G down, E gate,
G gate, E up, G up.  Writes profiles/gemm_traffic_r02.json.
  python tools/gemm_traffic.py gpurun_out/gemm_traffic.csv"""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
T, H, I = 8192, 4096, 14336
# algorithmic bytes: operand codes once + output once (bf16 Y, fp32 E prod / dW)
ALG = {"F_gate": T * H + I * H + 2 * T * I, "F_up": T * H + I * H + 2 * T * I, "F_down": T * I + H * I + 2 * T * H,
       "E_down": H * I + T * H + 4 * T * I, "G_down": T * H + T * I + 4 * H * I,
       "E_gate": I * H + T * I + 4 * T * H, "G_gate": T * I + T * H + 4 * I * H,
       "E_up": I * H + T * I + 4 * T * H, "G_up": T * I + T * H + 4 * I * H}
ORDER = ["F_gate", "F_up", "F_down", "E_down", "G_down", "E_gate", "G_gate", "E_up", "G_up"]

txt = open(sys.argv[1]).read()
txt = txt[txt.index('"ID"'):]
rows = list(csv.DictReader(io.StringIO(txt)))
per = {}
for r in rows:
    if "k_gemm" not in r["Kernel Name"]:
        continue
    per.setdefault(r["ID"], {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
ids = sorted(per, key=int)[-9:]
out = {}
for name, i in zip(ORDER, ids):
    d = per[i]
    dram = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
    out[name] = {"dram_bytes": dram, "algorithmic_bytes": ALG[name], "ratio": round(dram / ALG[name], 3),
                 "ns": d.get("gpu__time_duration.sum")}
cls = {}
for c in "FEG":
    ks = [k for k in out if k.startswith(c + "_")]
    cls[c] = {"dram_bytes_per_launch": sum(out[k]["dram_bytes"] for k in ks) / len(ks),
              "algorithmic_bytes_per_launch": sum(ALG[k] for k in ks) / len(ks)}
    cls[c]["ratio"] = round(cls[c]["dram_bytes_per_launch"] / cls[c]["algorithmic_bytes_per_launch"], 3)
tot = sum(v["dram_bytes"] for v in out.values())
alg = sum(ALG[k] for k in out)
res = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_gemm "
                 "python tools/prof_step.py (cold-cache replay, current kernel)",
       "bytes_per_launch": tot / 9, "algorithmic_bytes_per_launch": alg / 9,
       "dram_over_algorithmic": round(tot / alg, 3), "per_class": cls, "per_launch": out}
with open(os.path.join(ROOT, "profiles", "gemm_traffic_r02.json"), "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "per_launch"}, indent=1))
