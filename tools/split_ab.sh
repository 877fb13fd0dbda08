mkdir -p gpurun_out/s21
python tools/exp.py run main --cfg C4 > gpurun_out/s21/exp.log 2>&1
timeout 600 python -m pytest tests/test_split.py -x -q > gpurun_out/s21/split.log 2>&1; echo "rc=$?" >> gpurun_out/s21/split.log
python - > gpurun_out/s21/plans.log 2>&1 <<'PY'
import torch, workload as W, paper_2003_01216_b200 as hs
for c in ["C3", "C4", "C5", "C2", "P3"]:
    cfg = W.CONFIGS[c]
    d = torch.from_numpy(W.generate(c)).cuda()
    print(c, hs.hs_sort_plan(d, cfg.num_digits, cfg.chunks))
PY
for c in C4 C3 C5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/s21/b_$c.json 2>> gpurun_out/s21/b_$c.log
done
