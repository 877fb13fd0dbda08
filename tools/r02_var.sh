# merge-level variant timing + the merge/parity tests of the default build
set -x
OUT=gpurun_out/${1:-var}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_split.py tests/test_pairs_kv.py -q -x -k "not full_bitexact_large and not full_C3 and not max_size" > $OUT/tests.log 2>&1
tail -3 $OUT/tests.log
python tools/exp.py run ${VARS:-main m128 m128s3 m256 m256s3 m128v49} > $OUT/var.txt 2>&1
grep -E "^==|merge_level|merge_partition" $OUT/var.txt
