mkdir -p gpurun_out/e18
python tools/exp.py run main tg93 tg96 > gpurun_out/e18/exp.log 2>&1
python tools/exp.py run main tg93 tg96 --cfg C5 >> gpurun_out/e18/exp.log 2>&1
python tools/exp.py run main tg93 tg96 --cfg C2 >> gpurun_out/e18/exp.log 2>&1
