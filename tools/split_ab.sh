mkdir -p gpurun_out/s38
timeout 600 python -m pytest tests/test_next_rows.py tests/test_split.py -x -q -k "pairs" > gpurun_out/s38/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s38/tests.log
timeout 300 python bench.py --api pairs --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s38/b_pairs.json 2> gpurun_out/s38/b_pairs.log
