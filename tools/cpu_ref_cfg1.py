"""One-off: the unmodified reference (oracle/_ref, headers compiled with the
Release flags + -ffp-contract=off) timed on BASELINE configs[0] -- HALO-2
INT8, 2048 tokens x 4096 -> 4096, Hadamard block 256 -- on ONE host core of
the GPU box, as BASELINE.md §2 planned.  Prints one JSON line."""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402

b, m, n, block = 2048, 4096, 4096, 256
wall = O.ref_time_linear(2, 0, block, b, m, n, 1)
ops = 6.0 * b * m * n
lscpu = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
model = next((l.split(":", 1)[1].strip() for l in lscpu.splitlines() if l.startswith("Model name")), "?")
print(json.dumps({"config": "cfg1 HALO-2 INT8 b=2048 m=4096 n=4096 block 256 fwd+bwd", "impl": "reference (oracle/_ref)",
                  "threads": 1, "nproc": os.cpu_count(), "cpu_model": model, "wall_s": wall,
                  "gops": ops / wall / 1e9, "tokens_per_s": b / wall}), flush=True)
