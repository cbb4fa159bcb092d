#!/bin/bash
# adopted 28-column K3: full GPU suite + smoke, bench lines, K3 ncu
O=gpurun_out/r2l; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "tests exit $?" >> $O/gpu_tests.log
tail -3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?"
timeout 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench exit $?"; cut -c1-300 $O/bench_c3.json
bash scripts/prof_k3.sh ${1:-r02l} > /dev/null 2>&1
