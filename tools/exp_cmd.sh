mkdir -p gpurun_out/e2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e2/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/e2/smoke.log
python tools/exp.py run main k3sb > gpurun_out/e2/exp.log 2>&1
python tools/exp.py run main k3sb >> gpurun_out/e2/exp.log 2>&1
