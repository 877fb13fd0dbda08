mkdir -p gpurun_out/s31
timeout 600 python -m pytest tests/test_split.py -x -q > gpurun_out/s31/split.log 2>&1; echo "rc=$?" >> gpurun_out/s31/split.log
