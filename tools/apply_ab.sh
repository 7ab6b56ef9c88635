# apply / PCG timing of cfg4 (dev tool)
python tools/apply_timing.py 4 2>&1 | tail -1
python tools/apply_timing.py 4 2>&1 | tail -1
