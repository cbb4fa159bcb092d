#!/bin/bash
O=gpurun_out/r2g; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_decode.py -m gpu -q -rf -p no:cacheprovider -k "span" > $O/tests_span.log 2>&1; echo "span rc=$?"; tail -3 $O/tests_span.log
timeout 1500 bash scripts/profile_round.sh r02a > $O/prof.log 2>&1; echo "prof rc=$?"; tail -15 $O/prof.log
