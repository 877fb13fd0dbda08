mkdir -p gpurun_out/e21
python tools/exp.py run main tsx > gpurun_out/e21/exp.log 2>&1
python tools/exp.py run main tsx >> gpurun_out/e21/exp.log 2>&1
python tools/exp.py run main tsx --cfg C2 >> gpurun_out/e21/exp.log 2>&1
