"""CPU: the glibc-exact log1p used by the sketch's ziggurat tail, compiled for
the host from the same header the kernel uses, against libm on many inputs."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

SRC = r'''
#include "log1p_ieee.cuh"
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
int main() {
  std::mt19937_64 g(12345);
  long bad = 0, n = 0;
  for (long i = 0; i < 4000000; ++i) {
    double u = (g() >> 11) * (1.0 / 9007199254740992.0);
    double a = fpi::log1p_ieee(-u), b = std::log1p(-u);
    ++n; if (std::memcmp(&a, &b, 8)) ++bad;
    double v = std::ldexp((double)(g() >> 11), -53 - (int)(i % 64));
    a = fpi::log1p_ieee(-v); b = std::log1p(-v);
    ++n; if (std::memcmp(&a, &b, 8)) ++bad;
  }
  std::printf("%ld %ld\n", n, bad);
  return bad != 0;
}
'''


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_log1p_matches_libm(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text(SRC)
    exe = tmp_path / "t"
    subprocess.run(["g++", "-O2", "-I", str(ROOT / "paper_2011_04235_b200" / "csrc"), str(src), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    n, bad = map(int, out.stdout.split())
    assert n == 8_000_000 and bad == 0, out.stdout
