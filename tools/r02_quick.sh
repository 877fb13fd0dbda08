# quick iteration call: tree/split tests, bench C3 (+C5), config timings
set -x
OUT=${1:-gpurun_out/r02q}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_split.py tests/test_shapes.py -x -q > $OUT/tests.log 2>&1
tail -3 $OUT/tests.log
python bench.py --no-cpu-baseline > $OUT/bench_C3.json 2> $OUT/bench_C3.log
grep "\[bench\]" $OUT/bench_C3.log
python bench.py --config C5 --steps 5 --no-cpu-baseline > $OUT/bench_C5.json 2> $OUT/bench_C5.log
grep "\[bench\]" $OUT/bench_C5.log
python tools/quick_time.py C1 C2 C4 2>&1 | tee $OUT/quick.txt
