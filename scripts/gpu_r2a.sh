set -x
O=gpurun_out/r2a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 900 python -m pytest tests -m gpu -q -rf -x --timeout 600 -p no:cacheprovider tests/test_gpu_bench_parity.py tests/test_gpu_parity.py > $O/tests_parity.log 2>&1; echo "parity rc=$?"
timeout 300 python bench.py --steps 20 --warmup 5 > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench rc=$?"
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $O/bench_c3_200.json 2>> $O/bench_c3.err
WV_LIB=$PWD/paper_2208_10859_b200/variants/k3v1.so timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $O/bench_c3_v1.json 2>> $O/bench_c3.err
WV_LIB=$PWD/paper_2208_10859_b200/variants/segr16.so timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > $O/bench_c3_segr16.json 2>> $O/bench_c3.err
timeout 300 python bench.py --steps 20 --warmup 5 --mode full --no-cpu-baseline > $O/bench_full.json 2>> $O/bench_c3.err
WV_LIB=$PWD/paper_2208_10859_b200/variants/k3v1.so timeout 300 python bench.py --steps 20 --warmup 5 --mode full --no-cpu-baseline --no-e2e > $O/bench_full_v1.json 2>> $O/bench_c3.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 600 -p no:cacheprovider > $O/tests_all.log 2>&1; echo "all rc=$?"
tail -3 $O/tests_parity.log $O/tests_all.log
