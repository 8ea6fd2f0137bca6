#!/bin/bash
# one-shot environment + FP64 probe for a gpurun call
mkdir -p gpurun_out
{ nvidia-smi; free -g; nproc; lscpu | head -20; } > gpurun_out/env.txt 2>&1
tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1
