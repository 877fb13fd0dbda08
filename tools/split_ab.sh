mkdir -p gpurun_out/s8
timeout 600 python -m pytest tests/test_split.py tests/test_gpu_parity.py -x -q > gpurun_out/s8/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s8/tests.log
for c in C3 C3 C5 C4; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/s8/b_$c.json 2>> gpurun_out/s8/b_$c.log
done
ncu --set full --clock-control none --import-source on -k regex:"k_split_count|k_split_scatter|k_tile_sort" -s 3 -c 3 -o gpurun_out/s8/split python tools/one_call.py C3 sort 2 > gpurun_out/s8/ncu.log 2>&1
