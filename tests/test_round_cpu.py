"""The device quantizers (paper_2501_02625_b200/csrc/quant_round.cuh) compiled
for the host and checked against the oracle's double-precision round_code
(quantize.hpp:152-180) on random, midpoint-adjacent, exact-tie and
saturation inputs — both the exact and the fast/branch-free paths."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_device_quantizers_match_oracle(orc, tmp_path):
    exe = tmp_path / "round_check"
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-o", str(exe),
                    os.path.join(ROOT, "tests", "cpu", "round_check.cpp"),
                    "-L" + os.path.join(ROOT, "oracle", "_build"), "-lhalo_oracle",
                    "-Wl,-rpath," + os.path.join(ROOT, "oracle", "_build")], check=True)
    r = subprocess.run([str(exe), "400000"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches 0" in r.stdout
