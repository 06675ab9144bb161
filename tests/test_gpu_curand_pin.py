"""Second, independent pin of the Philox4x32-10 generator:
NVIDIA's cuRAND device API implements the same round function.  Its first
curand4() after curand_init(seed, subsequence, 0) is the Philox block of
counter (0, 0, lo32(subsequence), hi32(subsequence)) under key (lo32(seed),
hi32(seed)); the oracle's philox() must return exactly that block.  (The
Random123 known-answer vectors are the first pin: tests/test_oracle_rng.py.)
The cuRAND program is compiled here with nvcc and run on the GPU; nothing of
this repository's CUDA path is involved."""
import os
import shutil
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SRC = r"""
#include <cstdio>
#include <cstdlib>
#include <curand_kernel.h>
__global__ void k(const unsigned long long *seed, const unsigned long long *sub, uint4 *o, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  curandStatePhilox4_32_10_t s;
  curand_init(seed[i], sub[i], 0, &s);
  o[i] = curand4(&s);
}
int main(int argc, char **argv) {
  const int n = (argc - 1) / 2;
  unsigned long long hs[64], hb[64];
  for (int i = 0; i < n; ++i) {
    hs[i] = strtoull(argv[1 + 2 * i], 0, 0);
    hb[i] = strtoull(argv[2 + 2 * i], 0, 0);
  }
  unsigned long long *ds, *db; uint4 *d;
  cudaMalloc(&ds, 8 * n); cudaMalloc(&db, 8 * n); cudaMalloc(&d, 16 * n);
  cudaMemcpy(ds, hs, 8 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb, 8 * n, cudaMemcpyHostToDevice);
  k<<<1, 64>>>(ds, db, d, n);
  uint4 h[64];
  if (cudaMemcpy(h, d, 16 * n, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  for (int i = 0; i < n; ++i) printf("%u %u %u %u\n", h[i].x, h[i].y, h[i].z, h[i].w);
  return 0;
}
"""

CASES = [(0, 0), (0xffffffffffffffff, 0), (7, 1), (0x5EED0001, 3), (0x29F31D0A4093822, 0x0370734413198A2E),
         (123456789, 0xFFFFFFFF), (2 ** 40 + 17, 2 ** 33 + 5)]


def test_oracle_philox_equals_curand(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    src = tmp_path / "curand_pin.cu"
    exe = tmp_path / "curand_pin"
    src.write_text(SRC)
    subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(exe),
                           str(src)])
    args = [str(x) for s, b in CASES for x in (s, b)]
    out = subprocess.run([str(exe), *args], capture_output=True, text=True, check=True).stdout
    got = np.array([[int(v) for v in line.split()] for line in out.strip().splitlines()],
                   dtype=np.uint64)
    import oracle
    for (seed, sub), row in zip(CASES, got):
        ctr = [0, 0, sub & 0xFFFFFFFF, sub >> 32]
        key = [seed & 0xFFFFFFFF, seed >> 32]
        want = np.asarray(oracle.philox(ctr, key), dtype=np.uint64)
        assert np.array_equal(row, want), (hex(seed), hex(sub), row, want)
