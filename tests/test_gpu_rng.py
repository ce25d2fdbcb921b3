"""The device copy of the IP restart generator (csrc/common.cuh Mt19937_64 +
PolarNormal, mix_seed) against libstdc++: the reference perturbs a failed IP
column with std::mt19937_64(mix_seed(seed, i)) + std::normal_distribution
(fastfca.cpp:13-18, 40-41, 66-69), so restart trajectories only match if the
device reproduces those streams.  The libstdc++ side is a few lines of C++
compiled here with the same g++ the reference would use."""
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_2101_08563_b200 import _lib

pytestmark = pytest.mark.gpu

SRC = r"""
#include <cstdint>
#include <cstdio>
#include <random>
static std::uint64_t mix_seed(std::uint64_t seed, int i) {  // the published splitmix64 finaliser
  std::uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (i + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
int main(int argc, char** argv) {
  const std::uint64_t seed = std::strtoull(argv[1], nullptr, 10);
  const int bin = std::atoi(argv[2]), n = std::atoi(argv[3]);
  std::printf("%llu\n", (unsigned long long)mix_seed(seed, bin));
  std::mt19937_64 a(mix_seed(seed, bin));
  for (int k = 0; k < n; ++k) std::printf("%llu\n", (unsigned long long)a());
  std::mt19937_64 b(mix_seed(seed, bin));
  std::normal_distribution<double> gauss(0.0, 1.0);
  for (int k = 0; k < n; ++k) std::printf("%a\n", gauss(b));
}
"""


@pytest.fixture(scope="module")
def stdlib_draws(tmp_path_factory):
    d = tmp_path_factory.mktemp("rng")
    (d / "draws.cpp").write_text(SRC)
    r = subprocess.run(["g++", "-O2", "-std=c++20", "-ffp-contract=off", str(d / "draws.cpp"), "-o", str(d / "draws")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr

    def run(seed, bin_index, n):
        out = subprocess.run([str(d / "draws"), str(seed), str(bin_index), str(n)],
                             capture_output=True, text=True, check=True).stdout.split()
        return int(out[0]), [int(v) for v in out[1:1 + n]], [float.fromhex(v) for v in out[1 + n:]]
    return run


@pytest.mark.parametrize("seed,bin_index", [(0, 0), (7, 1), (12345678901234567, 2048), (2**64 - 1, 512)])
def test_restart_generator_matches_libstdcxx(gpu, stdlib_draws, seed, bin_index):
    n = 700  # crosses the 312-word twist twice
    mixed = np.zeros(1, np.uint64)
    raw = np.zeros(n, np.uint64)
    normals = np.zeros(n)
    _lib.check(_lib.lib().ffca_debug_restart_draws(gpu.handle, seed, bin_index, n, _lib.ptr(mixed),
                                                   _lib.ptr(raw), _lib.ptr(normals)))
    ms, raw_ref, normal_ref = stdlib_draws(seed, bin_index, n)
    assert int(mixed[0]) == ms
    assert [int(v) for v in raw] == raw_ref  # the Mersenne twister, bit for bit
    # the polar method: same accept/reject sequence (r2 is formed without FMA
    # contraction on both sides); the device log may differ from glibc's by an ulp
    np.testing.assert_allclose(normals, np.array(normal_ref), rtol=2e-15, atol=0)
