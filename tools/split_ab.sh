mkdir -p gpurun_out/s24
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s24/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s24/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s24/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s24/smoke.log
for c in C3 C4 C5 C1; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/s24/b_$c.json 2>> gpurun_out/s24/b_$c.log
done
timeout 300 python bench.py --dist --fused --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s24/b_distf.json 2> gpurun_out/s24/b_distf.log
