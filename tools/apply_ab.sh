# apply timing of cfg4 under a few environment settings (A/B of kernel routes), then the per-launch list
python tools/apply_timing.py 4 > gpurun_out/at_a.json 2>&1
SGF_GN_ROWS_SPARSE=32 python tools/apply_timing.py 4 > gpurun_out/at_b.json 2>&1
SGF_GN_ROWS_SPARSE=16 python tools/apply_timing.py 4 > gpurun_out/at_c.json 2>&1
SGF_GN_ROWS_SPARSE=16 SGF_SPARSE_BULK_MIN=256 python tools/apply_timing.py 4 > gpurun_out/at_d.json 2>&1
cat gpurun_out/at_a.json gpurun_out/at_b.json gpurun_out/at_c.json gpurun_out/at_d.json
SGF_SPARSE_BULK_MIN=256 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/apply_launches4.csv python tools/apply_ncu.py 4 > gpurun_out/apply_ncu.out 2>&1
