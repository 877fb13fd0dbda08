mkdir -p gpurun_out/final2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final2/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/final2/tests.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final2/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final2/smoke.log
python bench.py > gpurun_out/final2/bench.json 2> gpurun_out/final2/bench.log
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final2/ref.json 2> gpurun_out/final2/ref.log
