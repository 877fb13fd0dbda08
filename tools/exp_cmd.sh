mkdir -p gpurun_out/e17
python tools/exp.py run main m256 m256v21 m192v33 m128v49 > gpurun_out/e17/exp.log 2>&1
