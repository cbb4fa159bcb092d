#!/bin/bash
# A/B of library variants (paper_2208_10859_b200/variants/*.so) against the
# default build: a quick bench-clip parity check, then C3 viewport and
# full-frame benches.  Usage: scripts/gpu_variants.sh OUTDIR [variants...]
O=${1:-gpurun_out/var}; shift; mkdir -p $O
vs=${@:-default $(cd paper_2208_10859_b200/variants && ls *.so | sed 's/.so$//')}
for v in $vs; do
  if [ "$v" = default ]; then lib=$PWD/paper_2208_10859_b200/_wvb200.so; else lib=$PWD/paper_2208_10859_b200/variants/$v.so; fi
  WV_LIB=$lib timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_bench_parity.py -k "c3_viewport_step0 or c5_full or c4_foveated_gaze" > $O/$v.parity.log 2>&1 || { echo "$v PARITY FAIL"; tail -5 $O/$v.parity.log; continue; }
  WV_LIB=$lib timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $O/$v.c3.json 2> $O/$v.err
  WV_LIB=$lib timeout 300 python bench.py --steps 40 --warmup 5 --mode full --no-cpu-baseline --no-e2e > $O/$v.full.json 2>> $O/$v.err
  python - $O $v <<'PY'
import json,sys
O,v=sys.argv[1],sys.argv[2]
for m in ("c3","full"):
    try:
        d=json.load(open(f"{O}/{v}.{m}.json"))
        print(v, m, d["value"], d["serial_ms_per_frame"], {k: round(x*1000,1) for k,x in d["stage_ms"].items()}, d["roofline"]["frac"])
    except Exception as e:
        print(v, m, "ERR", e)
PY
done
