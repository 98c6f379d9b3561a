"""The drop-in API's double -> int8 block conversion (csrc/vd_host_convert.h,
used by vitdec::framed_decode(LlrBlock) to pick the exact int8 kernels, as
the reference's double arithmetic on integer-valued LLRs is exact): compiled
with g++ as the library is, checked on CPU (tests/cpp/host_convert_check.cpp)."""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_int8_block_conversion(tmp_path):
    exe = tmp_path / "host_convert_check"
    subprocess.run(["g++", "-O3", "-std=c++17", "-I", str(ROOT / "paper_2011_09337_b200" / "csrc"),
                    str(ROOT / "tests" / "cpp" / "host_convert_check.cpp"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout + r.stderr
