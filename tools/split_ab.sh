mkdir -p gpurun_out/s9
timeout 600 python -m pytest tests/test_split.py tests/test_gpu_parity.py tests/test_debug_build.py -x -q > gpurun_out/s9/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s9/tests.log
for c in C3 C5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/s9/b_$c.json 2>> gpurun_out/s9/b_$c.log
done
ncu --set full --clock-control none --import-source on -k regex:"k_split_count|k_split_scatter" -s 2 -c 2 -o gpurun_out/s9/split python tools/one_call.py C3 sort 2 > gpurun_out/s9/ncu.log 2>&1
