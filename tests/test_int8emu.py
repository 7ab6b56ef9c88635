"""FP64 products on the INT8 tensor cores (ozaki.cu): the batched operand
split + tcgen05 kind::i8 products against a CPU reference within the
scheme's error bound, on partial tiles, transposed operands, several products
per output block, lower-only blocks and triangular B (tools/oz_batch_test.cu,
built here against the in-tree libsgf.so)."""
import json
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"),
                    reason="nvcc not available")
def test_batched_int8_emulated_products(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    lib = os.path.join(ROOT, "paper_1907_03406_b200")
    exe = tmp_path / "oz_batch_test"
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17",
                    "-I", os.path.join(lib, "csrc"), "-I", os.path.join(ROOT, "include"),
                    "-o", str(exe), os.path.join(ROOT, "tools", "oz_batch_test.cu"),
                    "-L", lib, "-lsgf", "-Xlinker", f"-rpath={lib}"], check=True, capture_output=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    cases = [json.loads(l) for l in out.stdout.splitlines() if l.startswith('{"M"')]
    # 6 shape/layout cases + 5 graded-operand cases; "ok" = within the
    # scheme's bound and, for grades 0-2, within FP64's gamma_K sum|a||b|
    # (grade 3, cancellation by opposite column scalings, is gated by the
    # scheme bound only: tools/oz_batch_test.cu)
    assert len(cases) == 11 and all(c["ok"] for c in cases), cases
    assert all(c["err_over_fp64_gamma_K_bound"] <= 1.0 for c in cases if c["grade"] in (0, 1, 2))
    timing = [json.loads(l) for l in out.stdout.splitlines() if l.startswith('{"timing"')]
    assert timing and timing[-1]["fp64_tflops"] > 37.1  # above the DMMA FP64 peak
