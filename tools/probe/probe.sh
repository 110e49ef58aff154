#!/bin/bash
mkdir -p gpurun_out
{ nproc; lscpu | grep -E "Model name|Socket|Thread|Core|NUMA node\(s\)"; free -g; nvidia-smi; ./tools/probe/fp64_peak; } > gpurun_out/probe.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv >> gpurun_out/probe.txt
