// Test helper (not product code, not the oracle): cuRAND's own Philox4x32-10 on the device, so
// the GPU test can cross-check K1's draws against NVIDIA's implementation of the generator
// (SURVEY §4 library pins; reading c1).  Built by tests/test_gpu_full_size.py with nvcc.
#include <curand_kernel.h>
#include <stdint.h>

__global__ void k_philox(const uint4* __restrict__ ctr, uint2 key, uint4* __restrict__ out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = curand_Philox4x32_10(ctr[i], key);
}

extern "C" int curand_philox_words(const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out, int n) {
  uint4 *d_c = nullptr, *d_o = nullptr;
  if (cudaMalloc(&d_c, sizeof(uint4) * n) != cudaSuccess) return 1;
  if (cudaMalloc(&d_o, sizeof(uint4) * n) != cudaSuccess) return 1;
  cudaMemcpy(d_c, ctr, sizeof(uint4) * n, cudaMemcpyHostToDevice);
  k_philox<<<(n + 255) / 256, 256>>>(d_c, make_uint2(k0, k1), d_o, n);
  cudaMemcpy(out, d_o, sizeof(uint4) * n, cudaMemcpyDeviceToHost);
  const int bad = cudaGetLastError() != cudaSuccess;
  cudaFree(d_c);
  cudaFree(d_o);
  return bad;
}
