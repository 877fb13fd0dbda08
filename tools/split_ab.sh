mkdir -p gpurun_out/s23
timeout 600 python -m pytest tests/test_split.py tests/test_dist.py -x -q > gpurun_out/s23/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s23/tests.log
timeout 300 python bench.py --dist --fused --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s23/b_distf.json 2> gpurun_out/s23/b_distf.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s23/b.json 2> gpurun_out/s23/b.log
