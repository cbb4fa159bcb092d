#!/bin/bash
O=gpurun_out/r2h; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > $O/tests_all.log 2>&1; echo "all rc=$?"; tail -4 $O/tests_all.log
bash scripts/gpu_variants.sh $O default k2inplace
python scripts/host_profile.py 200 > $O/host_profile.txt 2>&1; head -1 $O/host_profile.txt
