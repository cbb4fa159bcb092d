#!/bin/bash
# round-2 K3 A/B: variants + ncu of the strip and per-tile level-1 kernels
O=gpurun_out/r2b; mkdir -p $O
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_decode.py -k "eye_split or blockend" > $O/newtests.log 2>&1; echo "newtests rc=$?"
bash scripts/gpu_variants.sh $O default k3v1 pf pfminb4 hybridpf minb5
P=$O/prof; mkdir -p $P
cmd="python bench.py --profile-only --warmup 3 --steps 1 --pipeline 1 --mode full"
$cmd && timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_strip -s 11 -c 1 -o $P/strip_full $cmd > $P/strip_full.log 2>&1
WV_LIB=$PWD/paper_2208_10859_b200/variants/pf.so timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_strip -s 11 -c 1 -o $P/strippf_full $cmd > $P/strippf_full.log 2>&1
ls -la $P
