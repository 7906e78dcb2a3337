#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/pcie_probe.py > gpurun_out/pcie.log 2>&1
nvidia-smi topo -m >> gpurun_out/pcie.log 2>&1
