mkdir -p gpurun_out/e10
python tools/exp.py run main s64v16 --cfg C5 > gpurun_out/e10/exp.log 2>&1
