# apply timing of cfg4 under a few environment settings (A/B of kernel routes)
for o in 4 5; do SGF_L1_BAND_OCC=$o python tools/apply_timing.py 4 2>&1 | tail -1; done
python -m pytest tests/test_gpu_parity.py tests/test_full_size_golden.py -m gpu -x -q 2>&1 | tail -2
