# one GPU call: E-byte granularity probe, per-GEMM rates of one factorization, per-launch list of one apply
python tools/traffic_probe.py 4 > gpurun_out/traffic4.json 2> gpurun_out/traffic4.err
SGF_TRACE=2 python tools/quick_time.py 4 > gpurun_out/trace2.out 2> gpurun_out/trace2.log
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/apply_launches4.csv python tools/apply_ncu.py 4 > gpurun_out/apply_ncu.out 2>&1
