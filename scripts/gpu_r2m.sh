#!/bin/bash
# final-state round-2 evidence: tests, smoke, bench lines of every config,
# the reference arm, and the ncu set (tag: first argument)
TAG=${1:-r02b}; O=gpurun_out/r2m_$TAG; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > $O/tests_all.log 2>&1; echo "all rc=$?"; tail -3 $O/tests_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/c3_driver.json 2> $O/c3_driver.err; echo "c3 driver-style rc=$?"
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > $O/c3.json 2> $O/c3.err
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --mode foveated > $O/c4.json 2> $O/c4.err
timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --mode full > $O/full.json 2> $O/full.err
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --config c2 > $O/c2.json 2> $O/c2.err
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --residency spans > $O/spans.json 2> $O/spans.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"
python scripts/host_profile.py 200 > $O/host_profile.txt 2>&1
timeout 1500 bash scripts/profile_round.sh $TAG > $O/prof.log 2>&1; echo "prof rc=$?"
for f in c3_driver c3 c4 full c2 spans ref; do python -c "
import json
try:
  d=json.load(open('$O/$f.json')); print('$f', d['value'], d.get('serial_ms_per_frame'), d.get('host_enqueue_us'), d.get('roofline',{}).get('frac'), (d.get('e2e') or {}).get('value'), d.get('stage_ms'))
except Exception as e: print('$f ERR', e)
"; done
