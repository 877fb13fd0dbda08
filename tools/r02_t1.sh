set -x
OUT=gpurun_out/r02b
mkdir -p $OUT
timeout 900 python -m pytest tests/test_tree.py -x -q > $OUT/tree.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/gputest.log 2>&1
python bench.py --no-cpu-baseline > $OUT/bench_C3.json 2> $OUT/bench_C3.log
python bench.py --config C5 --steps 5 --no-cpu-baseline > $OUT/bench_C5.json 2> $OUT/bench_C5.log
python tools/quick_time.py C1 C2 C4 > $OUT/quick.txt 2>&1
tail -3 $OUT/tree.log $OUT/gputest.log
grep "\[bench\]" $OUT/bench_C3.log $OUT/bench_C5.log
cat $OUT/quick.txt
