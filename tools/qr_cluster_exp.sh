# A/B of the L2-panel cluster QR variants on cfg5 (SGF_QR_CL = cluster size * 10000 + threads), then the QR variant and cfg5 full-size parity tests
mkdir -p gpurun_out
for v in 161024 81024 160256; do
  echo "== SGF_QR_CL=$v" >> gpurun_out/qr_exp.log
  SGF_QR_CL=$v SGF_TRACE=1 timeout 300 python tools/timeline.py 5 1 2>&1 | grep -E "resident|c-wave|L3 compress|L4 compress|factorize wall" | tail -16 >> gpurun_out/qr_exp.log
done
timeout 900 python -m pytest tests/test_kernel_variants.py -q -m gpu -k "qr" > gpurun_out/qr_variants.log 2>&1
timeout 900 python -m pytest tests/test_full_size_golden.py -q -m gpu -k "cfg5" > gpurun_out/qr_cfg5.log 2>&1
tail -3 gpurun_out/qr_variants.log gpurun_out/qr_cfg5.log
cat gpurun_out/qr_exp.log
