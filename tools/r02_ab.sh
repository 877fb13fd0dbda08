timeout 900 python -m pytest tests/test_split.py tests/test_shapes.py tests/test_gpu_parity.py -q -x -k "not full_bitexact_large and not full_C3 and not max_size" > gpurun_out/ad.log 2>&1; tail -2 gpurun_out/ad.log
python tools/exp.py run main noadapt --cfg C3 2>&1 | grep -E "^==|tile_sort"
python tools/exp.py run main noadapt --cfg C5 2>&1 | grep -E "^==|tile_sort"
python tools/exp.py run main noadapt --cfg C4 2>&1 | grep -E "^==|tile_sort"
