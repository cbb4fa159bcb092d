#!/bin/bash
O=gpurun_out/r2j; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > $O/tests_all.log 2>&1; echo "all rc=$?"; tail -4 $O/tests_all.log
bash scripts/gpu_variants.sh $O default noskip
cmd="python bench.py --profile-only --warmup 4 --steps 1 --pipeline 1"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_level -s 11 -c 1 -o $O/skip_k3_final $cmd > $O/ncu1.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_level -s 11 -c 1 -o $O/skip_k3_final_full $cmd --mode full > $O/ncu2.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_temporal -s 1 -c 1 -o $O/k2s $cmd > $O/ncu3.log 2>&1
ls $O
