# per-launch lists (ncu, one metric pass) of one apply, one factorization and the whole bench process
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/apply_launches4.csv python tools/apply_ncu.py 4 > gpurun_out/apply_ncu.out 2>&1
ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/factor_launches4.csv python tools/factor_ncu.py 4 > gpurun_out/factor_ncu.out 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 1 --warmup 0 --cpu-baseline none --no-extras > gpurun_out/bench_ncu.out 2>&1
tail -2 gpurun_out/bench_ncu.out | cut -c1-300
