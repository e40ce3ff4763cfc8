// pipebench.cu -- issue/pipe rates of the instruction forms the repulsion
// sweep is made of, alone and mixed, plus sweep inner-loop variants that
// split the fp32 work differently between packed (f32x2) and scalar forms.
// Experiment tool (not part of the product); results in profiles/r2/.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o pipebench scripts/pipebench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2002_08233_b200/csrc/bl_kernel.cuh"

#define PB_ITERS 2048

// OP: 0 FFMA (3 regs) | 1 FFMA2 (3 reg pairs) | 2 FADD2 (pair - scalar) |
//     3 FMUL2 | 4 MUFU.RCP | 5 mix 3 FFMA2 : 1 MUFU | 6 mix 6 FFMA2 : 2 MUFU :
//     1 FMUL (sweep TP=0 shape, independent) | 7 FFMA2 with one operand reused
//     (a = a*b + c where b shared by all chains) | 8 FFMA 2-reg + imm
template <int OP>
__global__ void __launch_bounds__(1024, 1) pb_kernel(float *sink, long long *cycles, float seed) {
  bl_f2 a[8], b[8], c[8];
  float s[8], t[8], u[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    s[k] = seed + threadIdx.x * 1e-6f + k;
    t[k] = 1.0001f + k * 1e-7f;
    u[k] = 1e-7f * k;
    a[k] = f2pack(s[k], s[k] + 0.5f);
    b[k] = f2pack(t[k], t[k] * 0.999f);
    c[k] = f2pack(u[k], u[k] * 2.f);
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < PB_ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) {
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(s[k]) : "f"(t[k]), "f"(u[k]));
      } else if (OP == 1) {
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[k]) : "l"(b[k]), "l"(c[k]));
      } else if (OP == 2) {
        bl_f2 tt = f2pack(t[k], t[k]);
        asm volatile("sub.rn.f32x2 %0, %0, %1;" : "+l"(a[k]) : "l"(tt));
      } else if (OP == 3) {
        asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(a[k]) : "l"(b[k]));
      } else if (OP == 4) {
        float r;
        asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(s[k]));
        s[k] = r + u[k];
      } else if (OP == 5) {
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[k]) : "l"(b[k]), "l"(c[k]));
        if (k & 1) {
          asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(c[k]) : "l"(b[k]), "l"(a[k]));
          asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(s[k]));
        } else {
          asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(b[k]) : "l"(a[k]), "l"(c[k]));
        }
      } else if (OP == 6) {
        // 6 FFMA2 + 2 MUFU per k (the TP=0 sweep shape without the data dependencies)
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[k]) : "l"(b[k]), "l"(c[k]));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(b[k]) : "l"(c[k]), "l"(a[k]));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(c[k]) : "l"(a[k]), "l"(b[k]));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[k]) : "l"(c[k]), "l"(b[k]));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(b[k]) : "l"(a[k]), "l"(a[k]));
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(c[k]) : "l"(b[k]), "l"(b[k]));
        asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(s[k]));
        asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(t[k]));
      } else if (OP == 7) {
        asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[k]) : "l"(b[0]), "l"(c[k]));
      } else if (OP == 8) {
        asm volatile("fma.rn.f32 %0, %0, %1, 0f33D6BF95;" : "+f"(s[k]) : "f"(t[k]));
      } else if (OP == 9) {
        // 6 scalar FFMA + 1 MUFU per k
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(s[k]) : "f"(t[k]), "f"(u[k]));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(t[k]) : "f"(u[k]), "f"(s[k]));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(u[k]) : "f"(s[k]), "f"(t[k]));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(s[k]) : "f"(u[k]), "f"(t[k]));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(t[k]) : "f"(s[k]), "f"(s[k]));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(u[k]) : "f"(t[k]), "f"(t[k]));
        float r;
        asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(s[k]));
        asm volatile("add.f32 %0, %0, %1;" : "+f"(u[k]) : "f"(r));
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float z = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float x, y, p, q, w, v;
    f2unpack(a[k], x, y);
    f2unpack(b[k], p, q);
    f2unpack(c[k], w, v);
    z += s[k] + t[k] + u[k] + x + y + p + q + w + v;
  }
  if (z == 123.456f) sink[threadIdx.x] = z;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
void rate(const char *name, double instr_per_k, int sms, float *d_out, long long *d_cyc) {
  for (int w = 0; w < 2; ++w) pb_kernel<OP><<<sms, 1024>>>(d_out, d_cyc, 1.0f);
  cudaDeviceSynchronize();
  std::vector<long long> cyc(sms);
  cudaMemcpy(cyc.data(), d_cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (auto c : cyc) mean += (double)c;
  mean /= sms;
  const double warp_instr = 32.0 * PB_ITERS * 8 * instr_per_k;  // per SM (32 warps)
  printf("%-44s %.3f warp-instr/clk/SM  (%.2f cyc per warp-instr per SMSP)\n", name,
         warp_instr / mean, 4.0 * mean / warp_instr);
}

// ---- sweep variants (T targets / thread, same data flow as bl_sweep) ----
// MODE 0: bl_sweep (all packed) | 1: packed DX/DY/D2, scalar accumulation |
// 2: packed DX/DY + accumulation, scalar D2 | 3: packed DX/DY only
template <int T, int TP, int MODE>
__device__ __forceinline__ void sweep_var(const float4 *__restrict__ src4, int s0, int s1,
                                          const float (&tx)[T], const float (&ty)[T],
                                          bl_f2 (&AX)[T], bl_f2 (&AY)[T], float (&ax)[T],
                                          float (&ay)[T]) {
  const bl_f2 EPS = f2pack(BL_EPS2, BL_EPS2);
  bl_f2 TX[T], TY[T];
#pragma unroll
  for (int k = 0; k < T; ++k) {
    TX[k] = f2pack(tx[k], tx[k]);
    TY[k] = f2pack(ty[k], ty[k]);
  }
#pragma unroll 2
  for (int s = s0; s < s1; ++s) {
    const float4 q = src4[s];
    const bl_f2 X = f2pack(q.x, q.y), Y = f2pack(q.z, q.w);
#pragma unroll
    for (int k = 0; k < T; ++k) {
      const bl_f2 DX = f2sub(X, TX[k]);
      const bl_f2 DY = f2sub(Y, TY[k]);
      float dxa, dxb, dya, dyb;
      f2unpack(DX, dxa, dxb);
      f2unpack(DY, dya, dyb);
      float a, b;
      if (MODE == 2 || MODE == 3) {
        a = fmaf(dxa, dxa, fmaf(dya, dya, BL_EPS2));
        b = fmaf(dxb, dxb, fmaf(dyb, dyb, BL_EPS2));
      } else {
        const bl_f2 D2 = f2fma(DX, DX, f2fma(DY, DY, EPS));
        f2unpack(D2, a, b);
      }
      float ia, ib;
      if (k < TP) {
        const float r = bl_rcp(a * b);
        ia = b * r;
        ib = a * r;
      } else {
        ia = bl_rcp(a);
        ib = bl_rcp(b);
      }
      if (MODE == 1 || MODE == 3) {
        ax[k] = fmaf(dxa, ia, fmaf(dxb, ib, ax[k]));
        ay[k] = fmaf(dya, ia, fmaf(dyb, ib, ay[k]));
      } else {
        const bl_f2 INV = f2pack(ia, ib);
        AX[k] = f2fma(DX, INV, AX[k]);
        AY[k] = f2fma(DY, INV, AY[k]);
      }
    }
  }
}

template <int NT, int T, int TP, int MODE, int UN = 2>
__global__ void __launch_bounds__(NT, 1) sv_kernel(const float2 *xy, int n4, int reps, float *out,
                                                   long long *cyc) {
  extern __shared__ float4 smem[];
  float4 *src4 = smem;
  for (int k = threadIdx.x; k < 2 * n4; k += NT) bl_src_set(src4, k, xy[k]);
  __syncthreads();
  float tx[T], ty[T], ax[T], ay[T];
  bl_f2 AX[T], AY[T];
#pragma unroll
  for (int k = 0; k < T; ++k) {
    const float2 t = xy[(threadIdx.x * T + k + 7) % (2 * n4)];
    tx[k] = t.x + 1e-3f;
    ty[k] = t.y - 1e-3f;
    AX[k] = AY[k] = f2pack(0.f, 0.f);
    ax[k] = ay[k] = 0.f;
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (MODE < 0)
      bl_sweep<T, TP, UN>(src4, 0, n4, tx, ty, AX, AY);
    else
      sweep_var<T, TP, MODE>(src4, 0, n4, tx, ty, AX, AY, ax, ay);
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
  out[blockIdx.x * NT + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int NT, int T, int TP, int MODE, int UN = 2>
void sweep(const char *name, const float2 *d_xy, int n4, int sms, float *d_out, long long *d_cyc) {
  auto k = sv_kernel<NT, T, TP, MODE, UN>;
  const size_t smem = (size_t)n4 * 16;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int reps = 40;
  for (int w = 0; w < 2; ++w) k<<<sms, NT, smem>>>(d_xy, n4, reps, d_out, d_cyc);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("%s failed\n", name);
    exit(1);
  }
  std::vector<long long> cyc(sms);
  cudaMemcpy(cyc.data(), d_cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (auto c : cyc) mean += (double)c;
  mean /= sms;
  const double pairs = (double)NT * T * 2.0 * n4 * reps;
  printf("sweep %-34s NT=%4d T=%2d TP=%d  %.2f pairs/clk/SM\n", name, NT, T, TP, pairs / mean);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *d_out;
  long long *d_cyc;
  cudaMalloc(&d_out, (size_t)sms * 1024 * sizeof(float));
  cudaMalloc(&d_cyc, sms * sizeof(long long));
  rate<0>("FFMA r,r,r", 1, sms, d_out, d_cyc);
  rate<8>("FFMA r,r,imm", 1, sms, d_out, d_cyc);
  rate<1>("FFMA2 rr,rr,rr", 1, sms, d_out, d_cyc);
  rate<7>("FFMA2 rr,rr(shared),rr", 1, sms, d_out, d_cyc);
  rate<2>("FADD2 rr,-r (broadcast)", 1, sms, d_out, d_cyc);
  rate<3>("FMUL2 rr,rr", 1, sms, d_out, d_cyc);
  rate<4>("MUFU.RCP + FADD", 2, sms, d_out, d_cyc);
  rate<5>("mix 1.5 FFMA2 : 0.5 MUFU", 2, sms, d_out, d_cyc);
  rate<6>("mix 6 FFMA2 : 2 MUFU", 8, sms, d_out, d_cyc);
  rate<9>("mix 6 FFMA : 1 MUFU : 1 FADD", 8, sms, d_out, d_cyc);

  const int n4 = 886;  // C5 chunk: 262,144 / 148 / 2
  std::vector<float2> h(2 * n4);
  srand(1);
  for (auto &v : h) v = make_float2(rand() / (float)RAND_MAX, rand() / (float)RAND_MAX);
  float2 *d_xy;
  cudaMalloc(&d_xy, h.size() * sizeof(float2));
  cudaMemcpy(d_xy, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice);
  sweep<512, 8, 2, -1>("bl_sweep", d_xy, n4, sms, d_out, d_cyc);
  if (getenv("PB_UNROLL2")) {
    sweep<512, 8, 2, -1, 4>("bl_sweep unroll 4", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 8, 3, -1, 4>("bl_sweep unroll 4", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 8, 1, -1, 4>("bl_sweep unroll 4", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 8, 4, -1, 4>("bl_sweep unroll 4", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 8, 2, -1, 8>("bl_sweep unroll 8", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 8, 3, -1, 8>("bl_sweep unroll 8", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 8, 2, -1, 6>("bl_sweep unroll 6", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 8, 3, -1, 3>("bl_sweep unroll 3", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 8, 4, -1, 1>("bl_sweep unroll 1", d_xy, n4, sms, d_out, d_cyc);
    sweep<256, 16, 4, -1, 4>("bl_sweep unroll 4", d_xy, n4, sms, d_out, d_cyc);
    sweep<256, 16, 6, -1, 2>("bl_sweep unroll 2", d_xy, n4, sms, d_out, d_cyc);
    sweep<256, 16, 6, -1, 4>("bl_sweep unroll 4", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 8, 2, -1, 4>("bl_sweep unroll 4 (again)", d_xy, n4, sms, d_out, d_cyc);
    return 0;
  }
  if (getenv("PB_UNROLL")) {
    sweep<512, 8, 2, -1, 1>("bl_sweep unroll 1", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 8, 2, -1, 3>("bl_sweep unroll 3", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 8, 2, -1, 4>("bl_sweep unroll 4", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 8, 1, -1, 1>("bl_sweep unroll 1", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 8, 3, -1, 1>("bl_sweep unroll 1", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 8, 1, -1, 2>("bl_sweep unroll 2", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 8, 3, -1, 2>("bl_sweep unroll 2", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 4, 1, -1, 1>("bl_sweep unroll 1", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 4, 1, -1, 2>("bl_sweep unroll 2", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 4, 1, -1, 4>("bl_sweep unroll 4", d_xy, n4, sms, d_out, d_cyc);
    sweep<256, 16, 4, -1, 1>("bl_sweep unroll 1", d_xy, n4, sms, d_out, d_cyc);
    sweep<512, 8, 2, -1, 2>("bl_sweep unroll 2 (again)", d_xy, n4, sms, d_out, d_cyc);
    return 0;
  }
  sweep<512, 8, 0, 0>("all packed", d_xy, n4, sms, d_out, d_cyc);
  sweep<512, 8, 2, 0>("all packed", d_xy, n4, sms, d_out, d_cyc);
  sweep<512, 8, 0, 1>("scalar accumulation", d_xy, n4, sms, d_out, d_cyc);
  sweep<512, 8, 2, 1>("scalar accumulation", d_xy, n4, sms, d_out, d_cyc);
  sweep<512, 8, 4, 1>("scalar accumulation", d_xy, n4, sms, d_out, d_cyc);
  sweep<512, 8, 0, 2>("scalar D2", d_xy, n4, sms, d_out, d_cyc);
  sweep<512, 8, 2, 2>("scalar D2", d_xy, n4, sms, d_out, d_cyc);
  sweep<512, 8, 4, 2>("scalar D2", d_xy, n4, sms, d_out, d_cyc);
  sweep<512, 8, 0, 3>("packed DX/DY only", d_xy, n4, sms, d_out, d_cyc);
  sweep<512, 8, 2, 3>("packed DX/DY only", d_xy, n4, sms, d_out, d_cyc);
  sweep<512, 8, 4, 3>("packed DX/DY only", d_xy, n4, sms, d_out, d_cyc);
  sweep<256, 16, 4, 0>("all packed", d_xy, n4, sms, d_out, d_cyc);
  sweep<256, 16, 4, 1>("scalar accumulation", d_xy, n4, sms, d_out, d_cyc);
  sweep<256, 16, 8, 1>("scalar accumulation", d_xy, n4, sms, d_out, d_cyc);
  sweep<256, 16, 4, 2>("scalar D2", d_xy, n4, sms, d_out, d_cyc);
  return 0;
}
