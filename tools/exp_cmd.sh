mkdir -p gpurun_out/e19
python tools/dist_sweep.py > gpurun_out/e19/sweep.log 2>&1
