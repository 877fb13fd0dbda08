mkdir -p gpurun_out/s12
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s12/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s12/tests.log
for c in C3 C5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/s12/b_$c.json 2>> gpurun_out/s12/b_$c.log
done
