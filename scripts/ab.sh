#!/bin/bash
# A/B of the working build against variants: scripts/ab.sh OUT [pytest -k expr] -- variants...
O=gpurun_out/$1; shift; mkdir -p $O
K=${1:-perspective or render or writeout}; shift
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$K" > $O/tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/tests.log
bash scripts/gpu_variants.sh $O default "$@"
