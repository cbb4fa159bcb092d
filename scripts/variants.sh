#!/bin/bash
# Bench each experimental library variant (paper_2208_10859_b200/variants/*.so)
# and the default build; one summary line per variant, after the variant
# passes the reference replay parity tests (a fast variant that is wrong is
# reported as such).  Usage: variants.sh [mode]
mode=${1:-viewport}
shopt -s nullglob
for lib in paper_2208_10859_b200/_wvb200.so paper_2208_10859_b200/variants/*.so; do
  name=$(basename $lib)
  [ "$name" = "checked.so" ] && continue
  [ "$name" = "k1direct.so" ] && [ -z "$WITH_DIRECT" ] && continue
  if ! WV_LIB=$PWD/$lib python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/var_parity.log 2>&1; then
    echo "$name PARITY FAIL"; continue
  fi
  WV_LIB=$PWD/$lib python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --mode $mode \
    > gpurun_out/var.json 2> gpurun_out/var.err
  python -c "import json,sys;d=json.load(open('gpurun_out/var.json'));print(sys.argv[1], d['value'], d['serial_ms_per_frame'], d['stage_ms'])" $name
done
