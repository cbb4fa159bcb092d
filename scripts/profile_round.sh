#!/bin/bash
# ncu evidence for one round (run on the GPU box from the repo root):
#   scripts/profile_round.sh TAG
# 1) the profiled command must first exit 0 without ncu; 2) launch list
# (gpu__time_duration per launch, 4 frames); 3) one --set full capture per
# hot kernel (viewport and full-frame).  Output: gpurun_out/prof/.
set -e
tag=${1:-rXX}
out=gpurun_out/prof; mkdir -p $out
cmd="python bench.py --profile-only --warmup 4 --steps 1 --pipeline 1"
$cmd
$cmd --mode full
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_${tag}.csv $cmd > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_full_${tag}.csv $cmd --mode full > /dev/null
cap() {  # name, kernel regex, skip, extra bench args
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$2 -s $3 -c 1 -o $out/${tag}_$1 $cmd $4 > $out/${tag}_$1.log 2>&1 || tail -5 $out/${tag}_$1.log
}
# per frame: k_level x L (levels L..2 are k_level<false>, level 1 k_level<true>)
cap k3_final "k_level" 11 ""
cap k3_level2 "k_level" 10 ""
cap k2 "k_temporal" 1 ""
cap k4 "k_perspective" 1 ""
cap k1_cascade "k_cascade_direct" 1 ""
cap k3_final_full "k_level" 11 "--mode full"
cap k2_full "k_temporal" 1 "--mode full"
ls -la $out
