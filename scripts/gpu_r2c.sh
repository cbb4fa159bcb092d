#!/bin/bash
O=gpurun_out/r2c; mkdir -p $O
bash scripts/gpu_variants.sh $O default tma2 tma3 k2staged k1direct
P=$O/prof; mkdir -p $P
cmd="python bench.py --profile-only --warmup 3 --steps 1 --pipeline 1"
WV_LIB=$PWD/paper_2208_10859_b200/variants/tma2.so timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_strip -s 11 -c 1 -o $P/tma2_full $cmd --mode full > $P/tma2_full.log 2>&1
WV_LIB=$PWD/paper_2208_10859_b200/variants/k1direct.so timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_cascade_direct -s 2 -c 1 -o $P/k1direct $cmd > $P/k1direct.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_temporal -s 2 -c 1 -o $P/k2 $cmd > $P/k2.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches_c3.csv $cmd > /dev/null 2>&1
ls -la $P
