mkdir -p gpurun_out/e11
python tools/exp.py run main k3sd > gpurun_out/e11/exp.log 2>&1
python tools/exp.py run main k3sd --cfg C5 >> gpurun_out/e11/exp.log 2>&1
