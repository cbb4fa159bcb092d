#!/bin/bash
O=gpurun_out/r2d; mkdir -p $O
python scripts/host_profile.py 400 > $O/host_profile.txt 2>&1
bash scripts/gpu_variants.sh $O default k4ty64 k4ty64mb2 k4mb3 k1direct
timeout 900 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > $O/tests_all.log 2>&1; echo "all rc=$?"; tail -3 $O/tests_all.log
