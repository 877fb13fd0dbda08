# Full evidence call: GPU tests, smoke, bench lines (C3 default + reference arm, C5, pairs, shared),
# per-kernel ncu counters (C3, C5), one full ncu capture of the dominant kernels (C3)
set -x
OUT=${1:-gpurun_out/r02full}
mkdir -p $OUT
{ nproc; lscpu | head -20; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv; } > $OUT/host.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=25 > $OUT/gputest.log 2>&1
tail -3 $OUT/gputest.log
python bench.py > $OUT/bench_C3.json 2> $OUT/bench_C3.log
python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.log
python bench.py --config C5 --steps 5 --no-cpu-baseline > $OUT/bench_C5.json 2> $OUT/bench_C5.log
python bench.py --api pairs --steps 5 --no-cpu-baseline > $OUT/bench_pairs_C3.json 2> $OUT/bench_pairs_C3.log
python bench.py --api pairs --config C5 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_pairs_C5.json 2> $OUT/bench_pairs_C5.log
python bench.py --api shared --steps 5 --no-cpu-baseline > $OUT/bench_shared.json 2> $OUT/bench_shared.log
python tools/quick_time.py C1 C2 C4 P3 > $OUT/quick.txt 2>&1
python tools/pcie_probe.py > $OUT/pcie.txt 2>&1
python tools/dist_sweep.py --kernels > $OUT/dist_sweep.txt 2>&1
grep "\[bench\]" $OUT/*.log | grep "ms/step =" 
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum
for C in C3 C5; do
  python tools/one_call.py $C sort 2 > $OUT/one_$C.log 2>&1 && \
  ncu --metrics $M --clock-control none --csv --log-file $OUT/ncu_$C.csv python tools/one_call.py $C sort 2 > $OUT/ncu_$C.log 2>&1
done
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/b_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $OUT/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
python tools/one_call.py C3 sort 2 > $OUT/one.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_tile_hist|k_scatter|k_split_count|k_split_scatter|k_tile_sort|k_merge_level|k_merge_partition" -s 35 -c 9 -o $OUT/full python tools/one_call.py C3 sort 2 > $OUT/ncu_full.log 2>&1
ls -la $OUT
