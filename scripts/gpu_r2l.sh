#!/bin/bash
O=gpurun_out/r2l; mkdir -p $O
WV_LIB=$PWD/paper_2208_10859_b200/variants/k4y64.so timeout 900 python -m pytest tests/test_gpu_decode.py -m gpu -q -rf -p no:cacheprovider -k "perspective or eye_split or hundred" > $O/k4y64_tests.log 2>&1; echo "k4y64 tests rc=$?"; tail -3 $O/k4y64_tests.log
bash scripts/gpu_variants.sh $O default noskip k4y64
bash scripts/gpu_variants.sh $O default noskip k4y64
