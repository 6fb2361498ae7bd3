#!/usr/bin/env bash
# Builds and runs the fp64 tensor-core / DFMA peak probe on the GPU box.
set -e
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
./dmma_probe
