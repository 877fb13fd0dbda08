mkdir -p gpurun_out/s35
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s35/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s35/tests.log
python tools/dist_sweep.py > gpurun_out/s35/sweep.log 2>&1
for c in C3 C4 C5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/s35/b_$c.json 2>> gpurun_out/s35/b_$c.log
done
