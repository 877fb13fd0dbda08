mkdir -p gpurun_out/e15
python tools/exp.py run main mpw0 mpw > gpurun_out/e15/exp.log 2>&1
python tools/exp.py run main mpw0 mpw >> gpurun_out/e15/exp.log 2>&1
python tools/exp.py run main mpw --cfg C5 >> gpurun_out/e15/exp.log 2>&1
