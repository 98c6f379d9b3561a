"""Drop-in check: the REFERENCE's own unit tests (test_trellis, test_codec,
test_channel, test_decoder, test_berlab — compiled unmodified against this
repo's include/vitdec headers and linked with libvitdec_b200.so instead of
the reference's trellis.cpp/decoder.cpp; see oracle/Makefile `dropin`) pass
with every framed_decode / serial_decode running on the GPU.

The binary is built where /root/reference exists and travels to the GPU box
as a prebuilt file; it reads nothing from /root/reference at run time.
"""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "oracle" / "_ref" / "dropin_unit_tests"

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not BIN.exists(), reason="drop-in test binary not built (needs /root/reference at build time)")
def test_reference_unit_suite_on_gpu_decoder():
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=900, cwd="/tmp")
    print(r.stdout[-2000:])
    print(r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "Status: SUCCESS!" in r.stdout


WORKERS_BIN = ROOT / "oracle" / "_ref" / "dropin_workers"


@pytest.mark.skipif(not WORKERS_BIN.exists(), reason="drop-in workers check not built (make -C oracle dropin)")
def test_dropin_api_workers_and_native_overload():
    """tests/cpp/dropin_workers.cpp: vitdec::framed_decode(LlrBlock, ..., workers)
    with 1 and 8 host threads and the native int8 overload agree bit for bit
    on a 3 Mi-stage block; real-valued blocks (FP64 kernel) too."""
    r = subprocess.run([str(WORKERS_BIN)], capture_output=True, text=True, timeout=600, cwd="/tmp")
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
