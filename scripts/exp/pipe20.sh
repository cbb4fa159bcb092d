#!/bin/bash
# short-run (driver-style 20 steps) C3 rate vs pipeline depth, repeated
O=gpurun_out/pipe20; mkdir -p $O
for r in 1 2; do for p in 2 4 6 8; do
  timeout 300 python bench.py --steps 20 --warmup 5 --pipeline $p --no-cpu-baseline --no-e2e > $O/p$p.$r.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/p$p.$r.json')); print($p, $r, d['value'], d['ms_per_step'])"
done; done
