// barrierbench.cu -- cost of the persistent kernels' grid barrier on B200
// (experiment tool, not part of the product): K back-to-back bl_grid_sync
// with (mode 1) or without (mode 0) one cross-CTA store + load per phase.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o barrierbench scripts/barrierbench.cu
#include <cstdio>
#include "../paper_2002_08233_b200/csrc/bl_kernel.cuh"

__global__ void __launch_bounds__(512, 1) bb_kernel(unsigned *bar, float *buf, int K, int mode,
                                                    long long *out) {
  __shared__ int ctr;
  unsigned target = 0;
  const int G = gridDim.x, c = blockIdx.x;
  float acc = 0.f;
  if (threadIdx.x == 0) ctr = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int k = 0; k < K; ++k) {
    if (mode >= 1 && threadIdx.x < 32) buf[c * 32 + threadIdx.x] = (float)k;
    bl_grid_sync(bar, target, &ctr);
    if (mode >= 1 && threadIdx.x < 32) acc += __ldcg(buf + ((c + 1 + k) % G) * 32 + threadIdx.x);
    if (mode >= 2 && threadIdx.x < 32) acc += __ldcg(buf + ((c + 7 + (int)acc % 3) % G) * 32 + threadIdx.x);
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[c] = t1 - t0;
  if (acc == -1.f) buf[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *bar;
  float *buf;
  long long *out;
  cudaMalloc(&bar, 4);
  cudaMalloc(&buf, sms * 32 * 4 * 2);
  cudaMalloc(&out, sms * 8);
  for (int grid : {sms, sms / 2, 16, 8}) {
    for (int mode = 0; mode < 3; ++mode) {
      const int K = 20000;
      cudaMemset(bar, 0, 4);
      void *args[] = {&bar, &buf, (void *)&K, &mode, &out};
      cudaLaunchCooperativeKernel((void *)bb_kernel, grid, 512, args, 0, 0);
      cudaError_t e = cudaDeviceSynchronize();
      long long h = 0;
      cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
      printf("grid %3d mode %d: %s %.3f us per barrier phase\n", grid, mode,
             cudaGetErrorString(e), h / 1965.0 / K);
    }
  }
  return 0;
}
