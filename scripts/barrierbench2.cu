// barrierbench2.cu -- grid-barrier alternatives on B200 (experiment tool, not
// part of the product), K back-to-back barriers, mode 1 adds one cross-CTA
// store + load per phase (what a batch hands over):
//   kind 0: the product's barrier (fence.acq_rel.gpu + red.add on ONE counter,
//           one poller per CTA with ld.acquire.gpu)
//   kind 1: flag all-gather: CTA c stores its phase number into flags[c]
//           (st.release.gpu), warp 0 polls all G flags (ld.acquire.gpu, a few
//           per lane) -- no atomic serialisation on one address
//   kind 2: as 1 with the flags read as uint4 (4 CTAs per load)
//   kind 4: as 1 with ld.acquire polls and no fence; kind 5: one flag per thread
//   kind 3: S counters (S = 8): CTA c arrives on counter c % S, the poller
//           warp reads all S (one per lane)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o barrierbench2 scripts/barrierbench2.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint4 ld_relaxed_v4(const uint4 *p) {
  uint4 v;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}

template <int KIND>
__device__ __forceinline__ void grid_sync(unsigned *bar, unsigned *flags, unsigned phase) {
  const int G = gridDim.x, c = blockIdx.x, lane = threadIdx.x & 31;
  __syncthreads();
  if (KIND == 0) {
    if (threadIdx.x == 0) {
      asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
      const unsigned target = phase * (unsigned)G;
      while ((int)(ld_acquire(bar) - target) < 0) {
      }
    }
  } else if (KIND == 1) {
    if (threadIdx.x < 32) {
      if (lane == 0)
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + c), "r"(phase) : "memory");
      for (int i = lane; i < G; i += 32)
        while ((int)(ld_relaxed(flags + i) - phase) < 0) {
        }
      __syncwarp();
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
  } else if (KIND == 2) {
    if (threadIdx.x < 32) {
      if (lane == 0)
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + c), "r"(phase) : "memory");
      const int n4 = (G + 3) / 4;  // flags padded to a multiple of 4, pad = 0xffffffff/2
      for (int i = lane; i < n4; i += 32) {
        for (;;) {
          const uint4 v = ld_relaxed_v4(reinterpret_cast<const uint4 *>(flags) + i);
          if ((int)(v.x - phase) >= 0 && (int)(v.y - phase) >= 0 && (int)(v.z - phase) >= 0 &&
              (int)(v.w - phase) >= 0)
            break;
        }
      }
      __syncwarp();
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
  } else if (KIND == 4) {
    if (threadIdx.x < 32) {
      if (lane == 0)
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + c), "r"(phase) : "memory");
      for (int i = lane; i < G; i += 32)
        while ((int)(ld_acquire(flags + i) - phase) < 0) {
        }
      __syncwarp();
    }
  } else if (KIND == 5) {
    // all 512 threads' lanes < G poll one flag each (one round trip, no loop over flags)
    if (threadIdx.x == 0)
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + c), "r"(phase) : "memory");
    if ((int)threadIdx.x < G)
      while ((int)(ld_acquire(flags + threadIdx.x) - phase) < 0) {
      }
  } else {
    constexpr int S = 8;
    if (threadIdx.x < 32) {
      if (lane == 0)
        asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 32 * (c % S)) : "memory");
      if (lane < S) {
        const unsigned cnt = (unsigned)((G - lane + S - 1) / S);  // CTAs on counter `lane`
        const unsigned target = phase * cnt;
        while ((int)(ld_acquire(bar + 32 * lane) - target) < 0) {
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();
}

template <int KIND>
__global__ void __launch_bounds__(512, 1) bb_kernel(unsigned *bar, unsigned *flags, float *buf, int K,
                                                    int mode, long long *out, int *err) {
  const int G = gridDim.x, c = blockIdx.x;
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int k = 0; k < K; ++k) {
    if (mode >= 1 && threadIdx.x < 32) buf[c * 32 + threadIdx.x] = (float)k;
    grid_sync<KIND>(bar, flags, (unsigned)k + 1u);
    if (mode >= 1 && threadIdx.x < 32) {
      const float v = __ldcg(buf + ((c + 1 + k) % G) * 32 + threadIdx.x);
      if (v != (float)k && v != (float)(k + 1)) atomicAdd(err, 1);  // a neighbour may be one phase ahead
      acc += v;
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[c] = t1 - t0;
  if (acc == -1.f) buf[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *bar, *flags;
  float *buf;
  long long *out;
  int *err;
  cudaMalloc(&bar, 4 * 32 * 8);
  cudaMalloc(&flags, 4 * 256);
  cudaMalloc(&buf, sms * 32 * 4 * 2);
  cudaMalloc(&out, sms * 8);
  cudaMalloc(&err, 4);
  void *fns[6] = {(void *)bb_kernel<0>, (void *)bb_kernel<1>, (void *)bb_kernel<2>, (void *)bb_kernel<3>,
                  (void *)bb_kernel<4>, (void *)bb_kernel<5>};
  for (int kind = 0; kind < 6; ++kind)
    for (int mode = 0; mode < 2; ++mode) {
      const int K = 20000, grid = sms;
      cudaMemset(bar, 0, 4 * 32 * 8);
      cudaMemset(flags, 0x7f, 4 * 256);  // pads: far ahead of every phase
      cudaMemset(flags, 0, 4 * grid);
      cudaMemset(err, 0, 4);
      void *args[] = {&bar, &flags, &buf, (void *)&K, &mode, &out, &err};
      cudaLaunchCooperativeKernel(fns[kind], grid, 512, args, 0, 0);
      cudaError_t e = cudaDeviceSynchronize();
      long long h = 0;
      int herr = 0;
      cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(&herr, err, 4, cudaMemcpyDeviceToHost);
      printf("kind %d grid %3d mode %d: %s %.3f us per barrier phase, stale reads %d\n", kind, grid, mode,
             cudaGetErrorString(e), h / 1965.0 / K, herr);
    }
  return 0;
}
