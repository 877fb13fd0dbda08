mkdir -p gpurun_out/s16
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pipeline or graph" > gpurun_out/s16/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s16/tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s16/b.json 2> gpurun_out/s16/b.log
