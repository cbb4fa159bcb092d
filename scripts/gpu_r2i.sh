#!/bin/bash
O=gpurun_out/r2i; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > $O/tests_all.log 2>&1; echo "all rc=$?"; tail -6 $O/tests_all.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --residency spans > $O/c3_spans.json 2> $O/c3_spans.err; echo "spans rc=$?"; tail -2 $O/c3_spans.err
python -c "
import json; d=json.load(open('$O/c3_spans.json')); print(d['value'], d['serial_ms_per_frame'], d['stage_ms'], d['e2e'])"
