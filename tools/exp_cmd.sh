mkdir -p gpurun_out/e4
python tools/exp.py run main pk > gpurun_out/e4/exp.log 2>&1
python tools/exp.py run main pk >> gpurun_out/e4/exp.log 2>&1
