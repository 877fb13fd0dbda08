mkdir -p gpurun_out/e1
python tools/exp.py run main b4c24 b4c20 b8c12 > gpurun_out/e1/exp.log 2>&1
