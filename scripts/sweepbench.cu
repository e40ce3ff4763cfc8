// sweepbench.cu -- isolated repulsion-sweep microbenchmark (experiment tool,
// not part of the product).  Runs the kernel's own bl_sweep<T, TP> (and
// alternative inner loops) over a shared-memory source chunk the size of one
// C5 CTA chunk, on every SM, and prints pairs/clk/SM per variant.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o sweepbench scripts/sweepbench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2002_08233_b200/csrc/bl_kernel.cuh"

// scalar fp32 variant: no packed instructions
template <int T, int TP>
__device__ __forceinline__ void sweep_scalar(const float4 *__restrict__ src4, int s0, int s1,
                                             const float (&tx)[T], const float (&ty)[T],
                                             float (&ax)[T], float (&ay)[T]) {
#pragma unroll 2
  for (int s = s0; s < s1; ++s) {
    const float4 q = src4[s];
#pragma unroll
    for (int k = 0; k < T; ++k) {
      const float dxa = q.x - tx[k], dxb = q.y - tx[k];
      const float dya = q.z - ty[k], dyb = q.w - ty[k];
      const float a = fmaf(dxa, dxa, fmaf(dya, dya, BL_EPS2));
      const float b = fmaf(dxb, dxb, fmaf(dyb, dyb, BL_EPS2));
      float ia, ib;
      if (k < TP) {
        const float r = bl_rcp(a * b);
        ia = b * r;
        ib = a * r;
      } else {
        ia = bl_rcp(a);
        ib = bl_rcp(b);
      }
      ax[k] = fmaf(dxa, ia, fmaf(dxb, ib, ax[k]));
      ay[k] = fmaf(dya, ia, fmaf(dyb, ib, ay[k]));
    }
  }
}

// fp64 targets: sources as double2 in shared memory (one LDS.128 per source),
// D targets per thread computed on the FP64 pipe with rcp.approx.ftz.f64
template <int D>
__device__ __forceinline__ void sweep_f64(const double2 *__restrict__ srcd, int s0, int s1,
                                          const double (&tx)[D], const double (&ty)[D],
                                          double (&ax)[D], double (&ay)[D]) {
#pragma unroll 2
  for (int s = s0; s < s1; ++s) {
    const double2 q = srcd[s];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double dx = q.x - tx[k], dy = q.y - ty[k];
      const double d2 = fma(dx, dx, fma(dy, dy, 1e-19));
      double r;
      asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d2));
      ax[k] = fma(dx, r, ax[k]);
      ay[k] = fma(dy, r, ay[k]);
    }
  }
}

template <int NT, int T, int TP, int MODE, int D>
__global__ void __launch_bounds__(NT, 1) sb_kernel(const float2 *xy, int n4, int reps, float *out,
                                                   long long *cyc) {
  extern __shared__ float4 smem[];
  float4 *src4 = smem;
  double2 *srcd = reinterpret_cast<double2 *>(smem + n4);
  for (int k = threadIdx.x; k < 2 * n4; k += NT) {
    bl_src_set(src4, k, xy[k]);
    if (MODE == 2) srcd[k] = make_double2(xy[k].x, xy[k].y);
  }
  __syncthreads();
  float tx[T], ty[T];
  bl_f2 AX[T], AY[T];
  float ax[T], ay[T];
  double dtx[D > 0 ? D : 1], dty[D > 0 ? D : 1], dax[D > 0 ? D : 1], day[D > 0 ? D : 1];
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const float2 t = xy[(threadIdx.x * T + k + 7) % (2 * n4)];
    tx[k] = t.x + 1e-3f;
    ty[k] = t.y - 1e-3f;
    AX[k] = AY[k] = f2pack(0.f, 0.f);
    ax[k] = ay[k] = 0.f;
  }
#pragma unroll
  for (int k = 0; k < (D > 0 ? D : 1); ++k) {
    const float2 t = xy[(threadIdx.x * 3 + k + 11) % (2 * n4)];
    dtx[k] = t.x + 2e-3;
    dty[k] = t.y - 2e-3;
    dax[k] = day[k] = 0.0;
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (MODE == 0) bl_sweep<T, TP>(src4, 0, n4, tx, ty, AX, AY);
    if (MODE == 1) sweep_scalar<T, TP>(src4, 0, n4, tx, ty, ax, ay);
    if (MODE == 2) {
      // hybrid: the fp32 packed sweep over float4 slots [0, n4) and the fp64
      // sweep over the same sources (2 n4 doubles) interleaved per chunk of 8
      for (int c = 0; c < n4; c += 8) {
        const int e = c + 8 < n4 ? c + 8 : n4;
        bl_sweep<T, TP>(src4, c, e, tx, ty, AX, AY);
        if (D > 0) sweep_f64<(D > 0 ? D : 1)>(srcd, 2 * c, 2 * e, dtx, dty, dax, day);
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < T; ++k) {
    float a, b, c, d;
    f2unpack(AX[k], a, b);
    f2unpack(AY[k], c, d);
    s += a + b + c + d + ax[k] + ay[k];
  }
#pragma unroll
  for (int k = 0; k < (D > 0 ? D : 1); ++k) s += (float)(dax[k] + day[k]);
  out[blockIdx.x * NT + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int NT, int T, int TP, int MODE, int D = 0>
void run(const char *name, const float2 *d_xy, int n4, int sms, float *d_out, long long *d_cyc) {
  auto k = sb_kernel<NT, T, TP, MODE, D>;
  const size_t smem = (size_t)n4 * 16 + (MODE == 2 ? (size_t)2 * n4 * 16 : 0);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int reps = 40;
  for (int w = 0; w < 2; ++w) k<<<sms, NT, smem>>>(d_xy, n4, reps, d_out, d_cyc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    exit(1);
  }
  std::vector<long long> cyc(sms);
  cudaMemcpy(cyc.data(), d_cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (auto c : cyc) mean += (double)c;
  mean /= sms;
  const double pairs = (double)NT * (T * 2.0 * n4 + (MODE == 2 ? D * 2.0 * n4 : 0.0)) * reps;
  printf("%-36s NT=%4d T=%d TP=%d D=%d  %.2f pairs/clk/SM\n", name, NT, T, TP, D, pairs / mean);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int n4 = 886;  // C5: 262,144 / 148 / 2
  std::vector<float2> h(2 * n4);
  srand(1);
  for (auto &v : h) v = make_float2(rand() / (float)RAND_MAX, rand() / (float)RAND_MAX);
  float2 *d_xy;
  float *d_out;
  long long *d_cyc;
  cudaMalloc(&d_xy, h.size() * sizeof(float2));
  cudaMemcpy(d_xy, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice);
  cudaMalloc(&d_out, (size_t)sms * 1024 * sizeof(float));
  cudaMalloc(&d_cyc, sms * sizeof(long long));
  run<512, 8, 0, 0>("packed", d_xy, n4, sms, d_out, d_cyc);
  run<512, 8, 1, 0>("packed", d_xy, n4, sms, d_out, d_cyc);
  run<512, 8, 2, 0>("packed", d_xy, n4, sms, d_out, d_cyc);
  run<512, 8, 3, 0>("packed", d_xy, n4, sms, d_out, d_cyc);
  run<512, 8, 4, 0>("packed", d_xy, n4, sms, d_out, d_cyc);
  run<512, 4, 1, 0>("packed", d_xy, n4, sms, d_out, d_cyc);
  run<1024, 4, 1, 0>("packed", d_xy, n4, sms, d_out, d_cyc);
  run<256, 16, 4, 0>("packed", d_xy, n4, sms, d_out, d_cyc);
  run<256, 16, 5, 0>("packed", d_xy, n4, sms, d_out, d_cyc);
  run<256, 12, 3, 0>("packed", d_xy, n4, sms, d_out, d_cyc);
  run<512, 8, 0, 1>("scalar", d_xy, n4, sms, d_out, d_cyc);
  run<512, 8, 2, 1>("scalar", d_xy, n4, sms, d_out, d_cyc);
  run<512, 8, 3, 1>("scalar", d_xy, n4, sms, d_out, d_cyc);
  run<512, 8, 2, 2, 1>("hybrid fp32 packed + fp64", d_xy, n4, sms, d_out, d_cyc);
  run<512, 8, 3, 2, 1>("hybrid fp32 packed + fp64", d_xy, n4, sms, d_out, d_cyc);
  run<512, 8, 4, 2, 2>("hybrid fp32 packed + fp64", d_xy, n4, sms, d_out, d_cyc);
  run<512, 6, 3, 2, 2>("hybrid fp32 packed + fp64", d_xy, n4, sms, d_out, d_cyc);
  run<512, 8, 8, 2, 2>("hybrid fp32 packed + fp64", d_xy, n4, sms, d_out, d_cyc);
  run<512, 1, 0, 2, 4>("mostly fp64", d_xy, n4, sms, d_out, d_cyc);
  return 0;
}
