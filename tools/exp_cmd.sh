mkdir -p gpurun_out/e7
python tools/exp.py run main spl8 spl12 > gpurun_out/e7/exp.log 2>&1
python tools/exp.py run main spl8 spl12 >> gpurun_out/e7/exp.log 2>&1
