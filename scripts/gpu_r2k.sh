#!/bin/bash
# 28-column warp-shuffle K3: GPU parity subset, A/B against the previous K3, K3 ncu
O=gpurun_out/r2k; mkdir -p $O
bash scripts/gpu_variants.sh $O default head
bash scripts/prof_k3.sh ${1:-r02k} > /dev/null 2>&1
