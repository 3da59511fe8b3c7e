// gridgen_dev.cu -- device-side Alg. 13 grid generator (INPUT GENERATOR, test/bench infra).
//
// Same recipe and the same FP operation sequence as synth_grid() in synth.c, so host and
// device outputs are bit-identical (checked by tests/test_synth.py):
//   vertex k = (k div s, k mod s); interior vertices + a*(2u-1) per axis with
//   u = (rng(seed, 2k+axis) >> 11) * 2^-53, rng = splitmix64 finaliser of seed*phi + ctr + 1;
//   triangles (k, k+1, k+s+1), (k, k+s+1, k+s) for k < s*s - s, k mod s != s - 1.
// Used for BASELINE configs 4 (256M vertices) and 5 (64 x 4M-vertex meshes), where a host
// generator + H2D copy would dominate.  Holds none of the Polylla method's arithmetic.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double rng_unit(uint64_t seed, uint64_t ctr) {
  const uint64_t r = mix64(seed * 0x9E3779B97F4A7C15ULL + ctr + 1ULL);
  return __dmul_rn((double)(r >> 11), 1.0 / 9007199254740992.0);
}

__global__ void k_grid_vertices(int64_t s, double a, uint64_t seed, double* __restrict__ xy) {
  const int64_t n = s * s;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = k / s, j = k % s;
    double x = (double)i, y = (double)j;
    if (a != 0.0 && i > 0 && i < s - 1 && j > 0 && j < s - 1) {
      const double ux = rng_unit(seed, 2 * (uint64_t)k), uy = rng_unit(seed, 2 * (uint64_t)k + 1);
      x = __dadd_rn(x, __dmul_rn(a, __dsub_rn(__dmul_rn(2.0, ux), 1.0)));
      y = __dadd_rn(y, __dmul_rn(a, __dsub_rn(__dmul_rn(2.0, uy), 1.0)));
    }
    reinterpret_cast<double2*>(xy)[k] = make_double2(x, y);
  }
}

__global__ void k_grid_triangles(int64_t s, int32_t* __restrict__ tri) {
  const int64_t cells = (s - 1) * (s - 1);
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = c / (s - 1), col = c % (s - 1);
    const int64_t k = row * s + col;  // k < s*s - s and k mod s != s - 1
    int32_t* t = tri + 6 * c;
    t[0] = (int32_t)k; t[1] = (int32_t)(k + 1); t[2] = (int32_t)(k + s + 1);
    t[3] = (int32_t)k; t[4] = (int32_t)(k + s + 1); t[5] = (int32_t)(k + s);
  }
}

}  // namespace

extern "C" __attribute__((visibility("default"))) int synth_grid_dev(int64_t s, double a, uint64_t seed, double* xy,
                                                                     int32_t* tri, void* stream) {
  if (s < 2) return -1;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_grid_vertices<<<148 * 16, 256, 0, st>>>(s, a, seed, xy);
  k_grid_triangles<<<148 * 16, 256, 0, st>>>(s, tri);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
