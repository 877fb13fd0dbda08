mkdir -p gpurun_out/e8
python tools/exp.py run main pdl > gpurun_out/e8/exp.log 2>&1
python tools/exp.py run main pdl >> gpurun_out/e8/exp.log 2>&1
