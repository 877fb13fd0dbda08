mkdir -p gpurun_out/s25
python tools/exp.py run main --cfg C4 > gpurun_out/s25/exp.log 2>&1
python tools/exp.py run main >> gpurun_out/s25/exp.log 2>&1
timeout 600 python -m pytest tests/test_split.py -x -q > gpurun_out/s25/split.log 2>&1; echo "rc=$?" >> gpurun_out/s25/split.log
python - > gpurun_out/s25/plans.log 2>&1 <<'PY'
import torch, workload as W, paper_2003_01216_b200 as hs
for c in ["C3", "C4", "C5", "C2", "P3"]:
    cfg = W.CONFIGS[c]
    d = torch.from_numpy(W.generate(c)).cuda()
    print(c, hs.hs_sort_plan(d, cfg.num_digits, cfg.chunks))
PY
