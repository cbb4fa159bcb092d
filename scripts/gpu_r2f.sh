#!/bin/bash
O=gpurun_out/r2f; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > $O/tests_all.log 2>&1; echo "all rc=$?"; tail -5 $O/tests_all.log
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > $O/c3.json 2> $O/c3.err; echo "c3 rc=$?"
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --residency spans > $O/c3_spans.json 2> $O/c3_spans.err; echo "spans rc=$?"
timeout 300 python bench.py --steps 40 --warmup 5 --mode full --no-cpu-baseline > $O/full.json 2> $O/full.err; echo "full rc=$?"
timeout 300 python bench.py --steps 60 --warmup 5 --config c2 --no-cpu-baseline > $O/c2.json 2> $O/c2.err; echo "c2 rc=$?"
timeout 300 python bench.py --steps 100 --warmup 10 --mode foveated --no-cpu-baseline > $O/c4.json 2> $O/c4.err; echo "c4 rc=$?"
python scripts/host_profile.py 200 > $O/host_profile.txt 2>&1; head -1 $O/host_profile.txt
for f in c3 c3_spans full c2 c4; do python -c "
import json,sys
try:
  d=json.load(open('$O/$f.json'))
  print('$f', d['value'], d['serial_ms_per_frame'], d.get('host_enqueue_us'), {k: round(x*1000,1) for k,x in d['stage_ms'].items()}, d['roofline']['frac'], (d.get('e2e') or {}).get('value'), (d.get('e2e') or {}).get('h2d_bytes_per_step'))
except Exception as e: print('$f ERR', e)
"; done
tail -3 $O/c3_spans.err
