#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/prof_block.py int8 > gpurun_out/prof_block_int8.log 2>&1
timeout 600 python tools/prof_block.py bf16 > gpurun_out/prof_block_bf16.log 2>&1
