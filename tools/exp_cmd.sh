mkdir -p gpurun_out/e13
python tools/exp.py run main t64b2c28 t64b2c30 --cfg C5 > gpurun_out/e13/exp.log 2>&1
