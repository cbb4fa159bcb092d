#!/bin/bash
# ncu --set full of the K3 finest (viewport, full frame) and level-2 kernels only:
#   scripts/prof_k3.sh TAG   -> gpurun_out/prof/
tag=${1:-rXX}
out=gpurun_out/prof; mkdir -p $out
cmd="python bench.py --profile-only --warmup 4 --steps 1 --pipeline 1"
$cmd > /dev/null && $cmd --mode full > /dev/null || exit 1
cap() {
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$2 -s $3 -c 1 -o $out/${tag}_$1 $cmd $4 > $out/${tag}_$1.log 2>&1 || tail -5 $out/${tag}_$1.log
}
cap k3_final "k_level" 11 ""
cap k3_level2 "k_level" 10 ""
cap k3_final_full "k_level" 11 "--mode full"
ls -la $out
