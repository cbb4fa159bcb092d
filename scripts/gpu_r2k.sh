#!/bin/bash
O=gpurun_out/r2k; mkdir -p $O
WV_LIB=$PWD/paper_2208_10859_b200/variants/ftz.so timeout 900 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_parity.py -m gpu -q -rf -p no:cacheprovider > $O/ftz_tests.log 2>&1; echo "ftz parity rc=$?"; tail -3 $O/ftz_tests.log
bash scripts/gpu_variants.sh $O default ftz
cmd="python bench.py --profile-only --warmup 4 --steps 1 --pipeline 1"
WV_LIB=$PWD/paper_2208_10859_b200/variants/ftz.so timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_level -s 11 -c 1 -o $O/ftz_k3_final_full $cmd --mode full > $O/ncu1.log 2>&1
