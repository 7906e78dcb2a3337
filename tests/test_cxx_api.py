"""The C++ object API (include/halo_b200.hpp) — the host language of the
reference — compiled against libhalo_b200.so: host checks on CPU, and a
HALO-2 INT8 forward/backward on the GPU checked bit-exactly by the oracle."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2501_02625_b200")


def _build(tmp_path):
    exe = tmp_path / "cxx_api_check"
    subprocess.run(["g++", "-std=c++17", "-O1", "-o", str(exe), os.path.join(ROOT, "tests", "cpu", "cxx_api_check.cpp"),
                    "-I/usr/local/cuda/include", "-L" + PKG, "-lhalo_b200", "-Wl,-rpath," + PKG,
                    "-L/usr/local/cuda/lib64", "-lcudart"], check=True)
    return exe


def test_cxx_api_host(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


@pytest.mark.gpu
def test_cxx_api_layer_on_gpu(orc, tmp_path):
    exe = _build(tmp_path)
    b, m, n, block = 128, 256, 64, 256
    X = orc.bf16_round(orc.randn(b, m, 1))
    X[:, 3] *= 40
    W = orc.bf16_round(orc.randn(n, m, 2, 1 / 16))
    E = orc.bf16_round(orc.randn(b, n, 3, 1e-3))
    for name, a in (("X", X), ("W", W), ("E", E)):
        a.astype(np.float32).tofile(tmp_path / f"{name}.f32")
    r = subprocess.run([str(exe), "gpu", str(tmp_path), str(b), str(m), str(n), str(block)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "counters 1 1 2" in r.stdout  # test_halo_linear.cpp:175-178
    want = orc.linear(2, 0, block, X, W, E)
    assert np.array_equal(np.fromfile(tmp_path / "Y.out", np.float32).reshape(b, n), want["Y"])
    assert np.array_equal(np.fromfile(tmp_path / "EX.out", np.float32).reshape(b, m), want["EX"])
    assert np.array_equal(np.fromfile(tmp_path / "GW.out", np.float32).reshape(n, m), want["GW"])


@pytest.mark.gpu
def test_cxx_fsdp_driver_world1(orc, tmp_path):
    """INTEGRATION.md §3 as a compiled C++ trainer step over the HQ-FSDP NCCL
    data plane (halo_fsdp_*): gather -> forward -> regather -> backward ->
    reduce-scatter, world 1 (NCCL refuses two ranks on one GPU; the protocol
    at world 2/4 is covered on CPU in test_fsdp_cpu.py).  Outputs bit-exact
    with the oracle layer; the stale-scale flag trips after a master write."""
    exe = tmp_path / "fsdp_driver"
    subprocess.run(["g++", "-std=c++17", "-O1", "-o", str(exe), os.path.join(ROOT, "tests", "cpu", "fsdp_driver.cpp"),
                    "-I/usr/local/cuda/include", "-L" + PKG, "-lhalo_b200", "-Wl,-rpath," + PKG,
                    "-L/usr/local/cuda/lib64", "-lcudart"], check=True)
    b, m, n, block = 256, 512, 256, 256
    X = orc.randn(b, m, 1)
    X[:, 3] *= 40
    X = orc.bf16_round(X)  # the driver uploads bf16: inputs must be bf16-exact
    W = orc.bf16_round(orc.randn(n, m, 2, 1 / 16))
    E = orc.bf16_round(orc.randn(b, n, 3, 1e-3))
    for name, a in (("X", X), ("W", W), ("E", E)):
        a.astype(np.float32).tofile(tmp_path / f"{name}.f32")
    r = subprocess.run([str(exe), str(tmp_path), str(b), str(m), str(n), str(block), "1", "0"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "stale-before 0 stale-after 1" in r.stdout, r.stdout
    want = orc.linear(2, 0, block, X, W, E)
    assert np.array_equal(np.fromfile(tmp_path / "Y.out", np.float32).reshape(b, n), want["Y"])
    assert np.array_equal(np.fromfile(tmp_path / "EX.out", np.float32).reshape(b, m), want["EX"])
    assert np.array_equal(np.fromfile(tmp_path / "GW0.out", np.float32).reshape(n, m), want["GW"])


ADAPTER = os.path.join(ROOT, "oracle", "_ref", "integration_adapter")


def test_integration_adapter_host():
    """INTEGRATION.md §1 compiled against the reference headers: the C++ API
    throws the reference's own halo::numeric_error (static_assert + catch)."""
    if not os.path.exists(ADAPTER):
        pytest.skip("adapter not built (needs /root/reference headers at build time)")
    r = subprocess.run([ADAPTER], capture_output=True, text=True)
    assert r.returncode == 0 and "0 failures" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_integration_adapter_matches_reference_layer():
    """The adapter's HaloLinearLayer (device) vs the unmodified reference
    HaloLinearLayer in the same process: Y, E_X, grad_W bit-identical."""
    if not os.path.exists(ADAPTER):
        pytest.skip("adapter not built")
    r = subprocess.run([ADAPTER, "gpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "Y 0 E_X 0 grad_W 0 differing" in r.stdout
