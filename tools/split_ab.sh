mkdir -p gpurun_out/s37
timeout 900 python -m pytest tests/test_shapes.py -x -q > gpurun_out/s37/tests.log 2>&1; echo "rc=$?" >> gpurun_out/s37/tests.log
