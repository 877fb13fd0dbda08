OUT=gpurun_out/probe; mkdir -p $OUT
python tools/probe_normal.py > $OUT/probe.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_tile_sort" -s 1 -c 1 -o $OUT/ts_normal python tools/probe_normal.py > $OUT/ncu.log 2>&1
ls -la $OUT; cat $OUT/probe.log
