// bl_microbench.cu -- per-SM issue rates of the instructions that bound the
// repulsion loop: 3-register FFMA, MUFU.RCP, MUFU.RSQ.
// The roofline denominators of DESIGN.md §5 come from these on the box.
#include <cuda_runtime.h>

#include "../../include/bl.h"

#define MB_NT 1024
#define MB_ITERS 4096

template <int OP>
__global__ void __launch_bounds__(MB_NT, 1) bl_mb_kernel(float *sink, long long *cycles, float seed) {
  float a[8], bb[8], cc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    a[k] = seed + threadIdx.x * 1e-6f + k;
    bb[k] = 1.0001f + k * 1e-7f;
    cc[k] = 1e-7f * k;
  }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < MB_ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) {
        a[k] = fmaf(a[k], bb[k], cc[k]);
      } else if (OP == 1) {
        // rcp(x) + c: one MUFU.RCP + one FADD per op (FADD at 128/clk is not
        // the binding pipe); a bare rcp chain is an involution ptxas may fold
        float r;
        asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a[k]));
        a[k] = r + cc[k];
      } else if (OP == 2) {
        float r;
        asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a[k]));
        a[k] = r + cc[k];
      } else if (k < 4) {
        // packed FFMA2 on (a[k], a[k+4]): counts as 2 thread-ops
        unsigned long long v, m, c2;
        asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(a[k]), "f"(a[k + 4]));
        asm("mov.b64 %0, {%1, %2};" : "=l"(m) : "f"(bb[k]), "f"(bb[k + 4]));
        asm("mov.b64 %0, {%1, %2};" : "=l"(c2) : "f"(cc[k]), "f"(cc[k + 4]));
        asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(v) : "l"(v), "l"(m), "l"(c2));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(a[k]), "=f"(a[k + 4]) : "l"(v));
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 123.456f) sink[threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

extern "C" bl_status bl_microbench(double rates[4]) {
  if (!rates) return BL_EINVAL;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return BL_ECUDA;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return BL_ECUDA;
  float *sink = nullptr;
  long long *cyc = nullptr;
  if (cudaMalloc(&sink, MB_NT * sizeof(float)) != cudaSuccess) return BL_ENOMEM;
  if (cudaMalloc(&cyc, sms * sizeof(long long)) != cudaSuccess) {
    cudaFree(sink);
    return BL_ENOMEM;
  }
  long long *h = new long long[sms];
  bl_status st = BL_OK;
  for (int op = 0; op < 4 && st == BL_OK; ++op) {
    for (int rep = 0; rep < 2; ++rep) {  // first pass warms clocks
      if (op == 0) bl_mb_kernel<0><<<sms, MB_NT>>>(sink, cyc, 1.0f);
      if (op == 1) bl_mb_kernel<1><<<sms, MB_NT>>>(sink, cyc, 1.0f);
      if (op == 2) bl_mb_kernel<2><<<sms, MB_NT>>>(sink, cyc, 1.0f);
      if (op == 3) bl_mb_kernel<3><<<sms, MB_NT>>>(sink, cyc, 1.0f);
    }
    if (cudaDeviceSynchronize() != cudaSuccess ||
        cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost) != cudaSuccess) {
      st = BL_ECUDA;
      break;
    }
    double mean = 0;
    for (int i = 0; i < sms; ++i) mean += (double)h[i];
    mean /= sms;
    rates[op] = (double)MB_NT * MB_ITERS * 8 / mean;  // thread-ops per clock per SM
  }
  delete[] h;
  cudaFree(sink);
  cudaFree(cyc);
  return st;
}
