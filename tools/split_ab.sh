mkdir -p gpurun_out/s29
timeout 600 python -m pytest tests/test_split.py -x -q > gpurun_out/s29/split.log 2>&1; echo "rc=$?" >> gpurun_out/s29/split.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s29/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s29/tests.log
python - > gpurun_out/s29/plans.log 2>&1 <<'PY'
import torch, numpy as np, workload as W, paper_2003_01216_b200 as hs
for c in ["C3", "C4", "C5", "C2", "P3"]:
    cfg = W.CONFIGS[c]
    d = torch.from_numpy(W.generate(c)).cuda()
    print(c, hs.hs_sort_plan(d, cfg.num_digits, cfg.chunks))
# sorted C3-sized input: before / after timing
import time
k = torch.arange(1 << 28, dtype=torch.int32, device="cuda") * 3
for rep in range(3):
    b = k.clone(); torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); hs.hs_sort(b, 9, 8); e.record(); torch.cuda.synchronize()
    print("sorted 2^28", s.elapsed_time(e), "ms", bool(torch.equal(b, k)))
print(hs.hs_sort_plan(k, 9, 8))
PY
for c in C3 C4 C5; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/s29/b_$c.json 2>> gpurun_out/s29/b_$c.log
done
