mkdir -p gpurun_out/e14
python tools/exp.py run cp1 cp2 cp4 > gpurun_out/e14/exp.log 2>&1
python tools/exp.py run cp1 cp2 cp4 >> gpurun_out/e14/exp.log 2>&1
