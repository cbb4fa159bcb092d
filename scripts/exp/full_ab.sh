#!/bin/bash
# full-frame (C5) A/B of wide-tile variants: bench --mode full --tile-strips 2 per variant
O=gpurun_out/$1; shift; mkdir -p $O
for v in "$@"; do
  WV_LIB=$PWD/paper_2208_10859_b200/variants/$v.so timeout 300 python bench.py --steps 40 --warmup 5 --mode full --tile-strips 1 --no-cpu-baseline --no-e2e > $O/$v.json 2>$O/$v.err
  python -c "
import json; d=json.load(open('$O/$v.json')); print('$v', d['value'], d['serial_ms_per_frame'], {k: round(x*1000,1) for k,x in d['stage_ms'].items()})"
done
