OUT=gpurun_out/base
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/host.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 > $OUT/gputest.log 2>&1
tail -3 $OUT/gputest.log
python bench.py --no-cpu-baseline > $OUT/bench_C3.json 2> $OUT/bench_C3.log
grep "\[bench\]" $OUT/bench_C3.log
python bench.py --config C5 --steps 5 --no-cpu-baseline > $OUT/bench_C5.json 2> $OUT/bench_C5.log
grep "\[bench\]" $OUT/bench_C5.log
python tools/quick_time.py C1 C2 C4 P3 2>&1 | tee $OUT/quick.txt
