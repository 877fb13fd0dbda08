mkdir -p gpurun_out/e20
python tools/exp.py run main k3n256 > gpurun_out/e20/exp.log 2>&1
python tools/exp.py run main k3n256 --cfg C5 >> gpurun_out/e20/exp.log 2>&1
