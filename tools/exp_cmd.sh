mkdir -p gpurun_out/e5
python tools/exp.py run main crpf crpf3 > gpurun_out/e5/exp.log 2>&1
python tools/exp.py run main crpf crpf3 >> gpurun_out/e5/exp.log 2>&1
