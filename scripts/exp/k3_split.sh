#!/bin/bash
# timing-only variants (results wrong by design): K3 finest without loads / without compute
O=gpurun_out/k3split; mkdir -p $O
for v in ${VARIANTS:-default noload nocompute}; do
  if [ $v = default ]; then lib=$PWD/paper_2208_10859_b200/_wvb200.so; else lib=$PWD/paper_2208_10859_b200/variants/$v.so; fi
  for m in viewport full; do
    WV_LIB=$lib timeout 300 python bench.py --steps 40 --warmup 5 --mode $m --no-cpu-baseline --no-e2e > $O/$v.$m.json 2>$O/$v.$m.err
    python -c "
import json; d=json.load(open('$O/$v.$m.json')); print('$v', '$m', round(d['stage_ms']['k3_level1_final']*1000,1))" 2>&1 | tail -1
  done
done
