#!/usr/bin/env bash
# Builds and runs the streaming-read probe (TMA ring vs 256-bit loads).
set -e
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu
./tma_probe
