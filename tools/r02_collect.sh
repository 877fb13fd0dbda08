# Copy one tools/r02_full.sh evidence directory into profiles/r02 and derive the tables
# usage: bash tools/r02_collect.sh gpurun_out/r02fullN
set -e
S=$1; D=profiles/r02; B=$(git rev-parse --short HEAD)
for f in bench_C3.json bench_C3.log bench_C5.json bench_C5.log bench_pairs_C3.json bench_pairs_C3.log bench_pairs_C5.json \
         bench_pairs_C5.log bench_ref.json bench_ref.log bench_shared.json bench_shared.log dist_sweep.txt gputest.log \
         host.txt launches_bench.csv quick.txt pcie.txt; do
  [ -f $S/$f ] && cp $S/$f $D/$f
done
python tools/ncu_table.py $S/launches_bench.csv > $D/launches_bench.txt
{ echo "# C3, build $B: ncu --metrics launch list of tools/one_call.py C3 sort 2 (second hs_sort call), --clock-control none (cold-cache, serialised: compare shares); count-pass bytes only for counted (not padded) buckets (--counted)"; python tools/ncu_kernel_table.py $S/ncu_C3.csv --n 268435456 --ksize 4 --last-call; } > $D/ncu_kernels_C3.txt
{ echo "# C5, build $B, same method"; python tools/ncu_kernel_table.py $S/ncu_C5.csv --n 536870912 --ksize 8 --last-call; } > $D/ncu_kernels_C5.txt
python tools/ncu_summary.py $S/full.ncu-rep > $D/ncu_full_summary_C3.txt
ncu -i $S/full.ncu-rep --page raw --csv > $D/ncu_full_raw_C3.csv
python tools/traffic_from_ncu.py $S/full.ncu-rep C3
