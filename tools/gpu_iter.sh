# quick iteration call: a test subset (arg 2, default the parity + split suites), bench C3 (+C5), quick configs
OUT=${1:-gpurun_out/iter}
TESTS=${2:-"tests/test_gpu_parity.py tests/test_split.py"}
mkdir -p $OUT
timeout 1200 python -m pytest $TESTS -x -q -m gpu > $OUT/tests.log 2>&1
tail -3 $OUT/tests.log
timeout 300 python bench.py --no-cpu-baseline > $OUT/bench_C3.json 2> $OUT/bench_C3.log
grep "\[bench\]" $OUT/bench_C3.log
timeout 300 python bench.py --config C5 --steps 5 --no-cpu-baseline > $OUT/bench_C5.json 2> $OUT/bench_C5.log
grep "\[bench\]" $OUT/bench_C5.log
timeout 300 python tools/quick_time.py C1 C2 C4 P3 2>&1 | tee $OUT/quick.txt
