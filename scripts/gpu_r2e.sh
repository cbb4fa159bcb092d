#!/bin/bash
O=gpurun_out/r2e; mkdir -p $O
python scripts/host_profile.py 400 > $O/host_profile.txt 2>&1; head -1 $O/host_profile.txt
timeout 900 python -m pytest tests -m gpu -q -x -rf -p no:cacheprovider > $O/tests_all.log 2>&1; echo "all rc=$?"; tail -3 $O/tests_all.log
bash scripts/gpu_variants.sh $O default nomerge k1direct k4mb3
