# Round-2 GPU call: smoke, GPU tests, bench (C3, C5), quick timings, per-kernel ncu counters (C3, C5)
# usage: bash tools/r02_call.sh OUTDIR [tests|notests] [ncu|noncu]
set -x
OUT=${1:-gpurun_out/r02}
mkdir -p $OUT
{ nproc; lscpu | head -20; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv; } > $OUT/host.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
if [ "${2:-tests}" = "tests" ]; then
  timeout 2400 python -m pytest tests -m gpu -q --durations=20 > $OUT/gputest.log 2>&1
fi
python bench.py > $OUT/bench_C3.json 2> $OUT/bench_C3.log
python bench.py --config C5 --steps 5 --no-cpu-baseline > $OUT/bench_C5.json 2> $OUT/bench_C5.log
python tools/quick_time.py C1 C2 C4 > $OUT/quick.txt 2>&1
if [ "${3:-ncu}" = "ncu" ]; then
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum
for C in C3 C5; do
  python tools/one_call.py $C sort 2 > $OUT/one_$C.log 2>&1 && \
  ncu --metrics $M --clock-control none --csv --log-file $OUT/ncu_$C.csv python tools/one_call.py $C sort 2 > $OUT/ncu_$C.log 2>&1
done
fi
ls -la $OUT
