mkdir -p gpurun_out/s30
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s30/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s30/tests.log
for c in C5 C3; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/s30/b_$c.json 2>> gpurun_out/s30/b_$c.log
done
timeout 300 python bench.py --api pairs --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s30/b_pairs.json 2> gpurun_out/s30/b_pairs.log
