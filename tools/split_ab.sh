mkdir -p gpurun_out/s11
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s11/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s11/tests.log
for c in C3 C5 C4; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/s11/b_$c.json 2>> gpurun_out/s11/b_$c.log
done
ncu --set full --clock-control none --import-source on -k regex:"k_scatter" -s 1 -c 1 -o gpurun_out/s11/k3 python tools/one_call.py C3 sort 2 > gpurun_out/s11/ncu.log 2>&1
