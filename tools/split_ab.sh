mkdir -p gpurun_out/s36
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s36/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s36/tests.log
python tools/dist_sweep.py > gpurun_out/s36/sweep.log 2>&1
for c in C3 C4 C5 C2; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/s36/b_$c.json 2>> gpurun_out/s36/b_$c.log
done
python - > gpurun_out/s36/plans.log 2>&1 <<'PY'
import torch, workload as W, paper_2003_01216_b200 as hs
for c in ["C3", "C4", "C5", "C2", "P3", "C1"]:
    cfg = W.CONFIGS[c]
    d = torch.from_numpy(W.generate(c)).cuda()
    print(c, hs.hs_sort_plan(d, cfg.num_digits, cfg.chunks))
PY
