mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/final/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.log
python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.log
for c in C1 C2 C4 C5 P3; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/final/b_$c.json 2>> gpurun_out/final/b_$c.log
done
