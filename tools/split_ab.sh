mkdir -p gpurun_out/s10
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s10/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s10/tests.log
for c in C3 C5 P3 C2; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/s10/b_$c.json 2>> gpurun_out/s10/b_$c.log
done
ncu --set full --clock-control none --import-source on -k regex:"k_tile_sort" -s 1 -c 1 -o gpurun_out/s10/ts python tools/one_call.py C3 sort 2 > gpurun_out/s10/ncu.log 2>&1
