set -x
mkdir -p gpurun_out/p2
python bench.py > gpurun_out/p2/bench.json 2> gpurun_out/p2/bench.log || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/p2/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/p2/ncu_launch.log 2>&1
python tools/one_call.py C3 sort 2 > gpurun_out/p2/one.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_tile_hist|k_scatter|k_tile_sort|k_merge_level|k_merge_partition" -s 31 -c 6 -o gpurun_out/p2/full python tools/one_call.py C3 sort 2 > gpurun_out/p2/ncu_full.log 2>&1
ls -la gpurun_out/p2
