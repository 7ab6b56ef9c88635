# hang diagnosis for tests/test_sharded.py: the two-rank worker with progress notes and a Python stack dump
cases=${1:-p3d30_b3,aniso26_b3,p2d100_b3,p3d30_exact,elast8_b3}
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port=29517 tests/dist_sharded_worker.py --mode solve --backend gloo --cases $cases --free --verbose --dump-after 200 > gpurun_out/sh_all.out 2> gpurun_out/sh_all.err; echo "rc=$?"; grep -c RESULT gpurun_out/sh_all.out; tail -30 gpurun_out/sh_all.err
