mkdir -p gpurun_out/s4
timeout 600 python -m pytest tests/test_split.py -x -q > gpurun_out/s4/split_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s4/split_tests.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s4/tests.log
for c in C3 C5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s4/b_$c.json 2> gpurun_out/s4/b_$c.log
done
ncu --set full --clock-control none --import-source on -k regex:"k_split_pass" -s 2 -c 2 -o gpurun_out/s4/split python tools/one_call.py C3 sort 2 > gpurun_out/s4/ncu.log 2>&1
